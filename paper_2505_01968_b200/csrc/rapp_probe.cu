// Measurement probes (not on the product path): the FP64 instruction rate of this device.
//
// MEASURED_PEAKS.json carries HBM bandwidth and bf16 tensor throughput only; the lattice
// search (K3, rapp_search.cu) executes FP64 adds/multiplies/compares on the CUDA cores, so
// bench.py measures the non-FMA FP64 rate here and reports K3 against it.  Each thread runs
// kChains independent dependency chains of __dadd_rn / __dmul_rn (the library is built with
// --fmad=false, and the _rn intrinsics are never contracted or reassociated), so the loop is
// throughput-bound on the FP64 pipe, not latency-bound.
#include "rapp_internal.h"

namespace rapp {

constexpr int kChains = 8;

template <bool MUL>
__global__ void __launch_bounds__(256) k_probe_fp64(double* __restrict__ sink, int iters,
                                                    double c) {
  double x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = double(threadIdx.x + k) * 1e-3 + 1.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < kChains; ++k) x[k] = MUL ? __dmul_rn(x[k], c) : __dadd_rn(x[k], c);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s = __dadd_rn(s, x[k]);
  if (s == 12345.678) sink[blockIdx.x] = s;  // keeps the chains live; never true
}

template <bool MUL>
static int probe_one(int sm_count, double* sink, double* rate) {
  const int blocks = sm_count * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  RAPP_CUDA(cudaEventCreate(&a));
  RAPP_CUDA(cudaEventCreate(&b));
  const double c = MUL ? 1.0000000001 : 1e-9;
  k_probe_fp64<MUL><<<blocks, threads>>>(sink, 64, c);  // warm-up
  RAPP_CUDA(cudaGetLastError());
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    RAPP_CUDA(cudaEventRecord(a));
    k_probe_fp64<MUL><<<blocks, threads>>>(sink, iters, c);
    RAPP_CUDA(cudaEventRecord(b));
    RAPP_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    RAPP_CUDA(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const double ops = double(blocks) * threads * iters * 8.0 * kChains;
  *rate = ops / (double(best) * 1e-3);
  return RAPP_OK;
}

}  // namespace rapp

using namespace rapp;

extern "C" int rapp_probe_fp64(int device, double* dadd_per_s, double* dmul_per_s) {
  RAPP_CUDA(cudaSetDevice(device));
  int sms = 0;
  RAPP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* sink = nullptr;
  RAPP_CUDA(cudaMalloc(&sink, sizeof(double) * sms * 8));
  double r1 = 0.0, r2 = 0.0;
  int rc = probe_one<false>(sms, sink, &r1);
  if (!rc) rc = probe_one<true>(sms, sink, &r2);
  cudaFree(sink);
  if (rc) return rc;
  if (dadd_per_s) *dadd_per_s = r1;
  if (dmul_per_s) *dmul_per_s = r2;
  return RAPP_OK;
}
