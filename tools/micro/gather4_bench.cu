// Microbenchmark (not product code): throughput of TMA tile::gather4 fetching random
// 64-byte rows (the K2 cell records) into shared memory, vs. the LSU path.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

__device__ __forceinline__ void bar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(b), done = 0;
  while (!done) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n" : "=r"(done) : "r"(s), "r"(ph) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}

constexpr int kStages = 16;   // ring stages, each ROWS rows of 64 B
constexpr int kRows = 32;     // rows per stage (8 gather4 ops)

__global__ void __launch_bounds__(64) k_tma(const __grid_constant__ CUtensorMap map, const int* idx, int64_t n, double* sink) {
  __shared__ __align__(128) double buf[kStages][kRows][8];
  __shared__ uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t tiles = n / kRows;
  if (warp == 0) {
    if (lane == 0) {
      int j = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
        const int s = j % kStages;
        if (j >= kStages) bar_wait(&empty[s], ((j / kStages) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])), "r"(kRows * 64) : "memory");
        const int* ix = idx + t * kRows;
        for (int g = 0; g < kRows / 4; ++g) {
          asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"((uint32_t)__cvta_generic_to_shared(&buf[s][4 * g][0])), "l"(&map), "r"(0), "r"(ix[4*g]), "r"(ix[4*g+1]), "r"(ix[4*g+2]), "r"(ix[4*g+3]),
              "r"((uint32_t)__cvta_generic_to_shared(&full[s])) : "memory");
        }
      }
    }
    return;
  }
  double acc = 0.0;
  int j = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
    const int s = j % kStages;
    bar_wait(&full[s], (j / kStages) & 1);
    // lane pair reads one 64-byte row: 32 rows per stage = 32 lanes x 32 B... read 2 doubles
    const double2 v = reinterpret_cast<const double2*>(&buf[s][lane][0])[0];
    acc += v.x + v.y;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[s]);
  }
  if (acc == 1234.5) sink[0] = acc;
}

__global__ void k_lsu(const double* cells, const int* idx, int64_t n, double* sink) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int half = threadIdx.x & 1;
    const int c = idx[i];
    const int cp = __shfl_xor_sync(0xffffffffu, c, 1);
    const double* p0 = cells + (int64_t)(half ? cp : c) * 8 + half * 4;
    const double* p1 = cells + (int64_t)(half ? c : cp) * 8 + half * 4;
    double a0, a1, a2, a3, b0, b1, b2, b3;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3) : "l"(p0));
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(b0), "=d"(b1), "=d"(b2), "=d"(b3) : "l"(p1));
    acc += a0 + a1 + a2 + a3 + b0 + b1 + b2 + b3;
  }
  if (acc == 1234.5) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t ncells = 60000;       // config-2 table: 6 x 100 x 100 cells
  const int64_t n = 64LL << 20;       // gathers
  double* cells; int* idx; double* sink;
  cudaMalloc(&cells, ncells * 64); cudaMalloc(&idx, n * 4); cudaMalloc(&sink, 8);
  cudaMemset(cells, 0, ncells * 64);
  std::vector<int> h(n); std::mt19937 rng(1);
  for (auto& x : h) x = rng() % ncells;
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {8, (cuuint64_t)ncells}, strides[1] = {64};
  cuuint32_t box[2] = {8, 1}, es[2] = {1, 1};
  CUresult r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cells, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocksPerSm : {4, 8, 16}) {
    k_tma<<<sms * blocksPerSm, 64>>>(map, idx, n, sink);
    cudaEventRecord(a);
    for (int k = 0; k < 3; ++k) k_tma<<<sms * blocksPerSm, 64>>>(map, idx, n, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("tma gather4 %d CTAs/SM: %.3f e9 rows/s (%s)\n", blocksPerSm, 3.0 * n / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  k_lsu<<<sms * 8, 512>>>(cells, idx, n, sink);
  cudaEventRecord(a);
  for (int k = 0; k < 3; ++k) k_lsu<<<sms * 8, 512>>>(cells, idx, n, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("lsu pair gather: %.3f e9 rows/s (%s)\n", 3.0 * n / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
