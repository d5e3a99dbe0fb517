// Host side of the e2e stream: (1) PCIe H2D / D2H / both-directions bandwidth from pinned
// memory, (2) how fast T host threads narrow (n,3) float64 coordinates to float32 when every
// value round-trips exactly (the lossless transport check), into pinned staging.
//   nvcc -O3 -Xcompiler -fopenmp,-march=native -o /tmp/pack_bench pack_bench.cu
#include <omp.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// returns false if some value is not exactly representable as float
static bool narrow(const double* __restrict__ in, float* __restrict__ out, int64_t m) {
  bool ok = true;
  for (int64_t i = 0; i < m; ++i) {
    const float f = (float)in[i];
    ok &= ((double)f == in[i]);
    out[i] = f;
  }
  return ok;
}

int main() {
  const int64_t n = 25'000'000;  // queries (one e2e model slice)
  double* h_in;
  double* h_out;
  float* h_f;
  cudaMallocHost(&h_in, n * 24);
  cudaMallocHost(&h_out, n * 8);
  cudaMallocHost(&h_f, n * 12);
  for (int64_t i = 0; i < 3 * n; ++i) h_in[i] = double(1 + (i * 2654435761u) % 100);
  void *d_in, *d_out;
  cudaMalloc(&d_in, n * 24);
  cudaMalloc(&d_out, n * 8);
  cudaStream_t s0, s1;
  cudaStreamCreate(&s0);
  cudaStreamCreate(&s1);
  printf("host threads: %d (hardware_concurrency %u)\n", omp_get_max_threads(),
         std::thread::hardware_concurrency());
  auto bw = [&](const char* what, auto fn, double bytes) {
    fn();
    cudaDeviceSynchronize();
    const double t0 = now();
    for (int r = 0; r < 5; ++r) fn();
    cudaDeviceSynchronize();
    const double dt = (now() - t0) / 5;
    printf("%-28s %8.2f GB/s  (%.2f ms)\n", what, bytes / dt / 1e9, dt * 1e3);
  };
  bw("H2D 24 B/query", [&] { cudaMemcpyAsync(d_in, h_in, n * 24, cudaMemcpyHostToDevice, s0); },
     n * 24.0);
  bw("H2D 12 B/query", [&] { cudaMemcpyAsync(d_in, h_f, n * 12, cudaMemcpyHostToDevice, s0); },
     n * 12.0);
  bw("D2H 8 B/query", [&] { cudaMemcpyAsync(h_out, d_out, n * 8, cudaMemcpyDeviceToHost, s0); },
     n * 8.0);
  bw("H2D 24 + D2H 8 concurrent", [&] {
    cudaMemcpyAsync(d_in, h_in, n * 24, cudaMemcpyHostToDevice, s0);
    cudaMemcpyAsync(h_out, d_out, n * 8, cudaMemcpyDeviceToHost, s1);
  }, n * 32.0);
  bw("H2D 12 + D2H 8 concurrent", [&] {
    cudaMemcpyAsync(d_in, h_f, n * 12, cudaMemcpyHostToDevice, s0);
    cudaMemcpyAsync(h_out, d_out, n * 8, cudaMemcpyDeviceToHost, s1);
  }, n * 20.0);
  const int maxT = omp_get_max_threads();
  for (int T : {1, 2, 4, 8, 12, 16, 24, 32, 48, 64}) {
    if (T > maxT) break;
    omp_set_num_threads(T);
    const int64_t chunk = 1 << 16;
    bool all = true;
    const double t0 = now();
    for (int r = 0; r < 3; ++r) {
#pragma omp parallel for schedule(static) reduction(&& : all)
      for (int64_t c = 0; c < (3 * n + chunk - 1) / chunk; ++c) {
        const int64_t a = c * chunk, m = (3 * n - a) < chunk ? (3 * n - a) : chunk;
        all = narrow(h_in + a, h_f + a, m) && all;
      }
    }
    const double dt = (now() - t0) / 3;
    printf("narrow f64->f32, %2d threads: %6.2f e9 queries/s (%.1f GB/s read), exact=%d\n", T,
           n / dt / 1e9, n * 24.0 / dt / 1e9, (int)all);
  }
  return 0;
}
