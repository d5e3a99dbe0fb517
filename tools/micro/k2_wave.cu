// L1 data-pipe wavefront accounting for K2's building blocks (one kernel per pattern; read
// the counters with ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_lgds_cmd_read.sum,
// l1tex__data_pipe_lsu_wavefronts_mem_shared.sum, smsp__inst_executed.sum).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k2_wave k2_wave.cu
// Every kernel handles 32 queries per warp iteration over a 4 MB cell array (64-B cells,
// random cell per query from a hash), so the per-query counts compare directly.
#include <cstdint>
#include <cstdio>

constexpr int kCells = 1 << 16;  // 64 B each: 4 MB (L2-resident, like config 2's 3.8 MB)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void ld128(const double* p, double& a, double& b) {
  asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
}

// current K2 layout: lane pair shares a cell, each lane one 256-bit half, two loads per pair
__global__ void k_pair256(const double* __restrict__ cells, int64_t n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, half = lane & 1;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t cell = hash32(uint32_t(i)) & (kCells - 1);
    const uint32_t cp = __shfl_xor_sync(0xffffffffu, cell, 1);
    const uint32_t c0 = half ? cp : cell, c1 = half ? cell : cp;
    double a, b, c, d, e, f, g, h;
    ld256(cells + int64_t(c0) * 8 + half * 4, a, b, c, d);
    ld256(cells + int64_t(c1) * 8 + half * 4, e, f, g, h);
    __stcs(out + i, a + b + c + d + e + f + g + h);
  }
}

// quad layout: 4 lanes share a cell, each lane one 128-bit quarter, four loads per quad
__global__ void k_quad128(const double* __restrict__ cells, int64_t n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, qd = lane & 3;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t cell = hash32(uint32_t(i)) & (kCells - 1);
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t c = __shfl_sync(0xffffffffu, cell, (lane & ~3) | r);
      double a, b;
      ld128(cells + int64_t(c) * 8 + qd * 2, a, b);
      acc += a + b;
    }
    __stcs(out + i, acc);
  }
}

// lane pair shares a cell, each lane two 128-bit loads of its half
__global__ void k_pair128x2(const double* __restrict__ cells, int64_t n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, half = lane & 1;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t cell = hash32(uint32_t(i)) & (kCells - 1);
    const uint32_t cp = __shfl_xor_sync(0xffffffffu, cell, 1);
    const uint32_t c0 = half ? cp : cell, c1 = half ? cell : cp;
    double a, b, c, d, e, f, g, h;
    ld128(cells + int64_t(c0) * 8 + half * 4, a, b);
    ld128(cells + int64_t(c0) * 8 + half * 4 + 2, c, d);
    ld128(cells + int64_t(c1) * 8 + half * 4, e, f);
    ld128(cells + int64_t(c1) * 8 + half * 4 + 2, g, h);
    __stcs(out + i, a + b + c + d + e + f + g + h);
  }
}

// one lane per cell: two 256-bit loads of its own cell
__global__ void k_lane512(const double* __restrict__ cells, int64_t n, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t cell = hash32(uint32_t(i)) & (kCells - 1);
    double a, b, c, d, e, f, g, h;
    ld256(cells + int64_t(cell) * 8, a, b, c, d);
    ld256(cells + int64_t(cell) * 8 + 4, e, f, g, h);
    __stcs(out + i, a + b + c + d + e + f + g + h);
  }
}

// stores only (baseline for the per-query output write)
__global__ void k_store(int64_t n, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    __stcs(out + i, double(hash32(uint32_t(i))));
}

// 7 shuffles per lane per query (K2's exchange count) + store: do SHFLs count as wavefronts?
__global__ void k_shfl7(int64_t n, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t x = hash32(uint32_t(i));
#pragma unroll
    for (int r = 0; r < 7; ++r) x += __shfl_xor_sync(0xffffffffu, x, 1 + (r & 3));
    __stcs(out + i, double(x));
  }
}

// coordinates straight from global: a warp's 32 rows (768 B) as two coalesced 16-B loads
// (512 B + 256 B), then rows rebuilt with shuffles (each lane ends with its row's 3 doubles)
__global__ void k_coords_direct(const double* __restrict__ coords, int64_t n,
                                double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t w = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 32 < n;
       w += warps) {
    const double* base = coords + w * 96;
    double a0, a1, b0 = 0.0, b1 = 0.0;
    ld128(base + 2 * lane, a0, a1);                   // doubles 0..63
    if (lane < 16) ld128(base + 64 + 2 * lane, b0, b1);  // doubles 64..95
    // row r = lane needs doubles 3r, 3r+1, 3r+2
    double x[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int d = 3 * lane + k;  // 0..95
      const int src = (d & 63) >> 1;
      const double lo = __shfl_sync(0xffffffffu, (d & 1) ? a1 : a0, src);
      const double hi = __shfl_sync(0xffffffffu, (d & 1) ? b1 : b0, src);
      x[k] = d < 64 ? lo : hi;
    }
    __stcs(out + w * 32 + lane, x[0] + x[1] + x[2]);
  }
}

// coordinates via three strided 8-B loads per lane (no staging, no shuffles)
__global__ void k_coords_strided(const double* __restrict__ coords, int64_t n,
                                 double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double x = __ldcs(coords + 3 * i), y = __ldcs(coords + 3 * i + 1),
                 z = __ldcs(coords + 3 * i + 2);
    __stcs(out + i, x + y + z);
  }
}

int main() {
  const int64_t n = 1 << 24;
  double *cells, *coords, *out;
  cudaMalloc(&cells, size_t(kCells) * 64);
  cudaMalloc(&coords, size_t(n) * 24);
  cudaMalloc(&out, size_t(n) * 8);
  cudaMemset(cells, 0, size_t(kCells) * 64);
  cudaMemset(coords, 0, size_t(n) * 24);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4, block = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](const char* name, auto launch) {
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-16s %8.3f us/launch  %6.2f e9 queries/s\n", name, 100.0 * ms, n / (ms / 10) / 1e6);
  };
  time("pair256", [&] { k_pair256<<<grid, block>>>(cells, n, out); });
  time("quad128", [&] { k_quad128<<<grid, block>>>(cells, n, out); });
  time("pair128x2", [&] { k_pair128x2<<<grid, block>>>(cells, n, out); });
  time("lane512", [&] { k_lane512<<<grid, block>>>(cells, n, out); });
  time("store", [&] { k_store<<<grid, block>>>(n, out); });
  time("shfl7", [&] { k_shfl7<<<grid, block>>>(n, out); });
  time("coords_direct", [&] { k_coords_direct<<<grid, block>>>(coords, n, out); });
  time("coords_strided", [&] { k_coords_strided<<<grid, block>>>(coords, n, out); });
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
