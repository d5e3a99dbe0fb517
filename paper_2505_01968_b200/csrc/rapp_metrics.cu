// Run metrics finalize on the device — SimulationEngine._finalize, hs/sim.py:586-621.
//
// Per function (sorted ids, one CTA each):
//   violation curve  curve[m] = (late_m + rejected + unfinished) / arrived, late_m = number of
//                    latencies > baseline * multiplier[m]  (sim.py:592-598)
//   percentiles      nearest rank: the k-th smallest latency, k = ceil(q / 100.0 * n)
//                    clamped to [1, n]; NaN when there are none (sim.py:599-600, 612-617)
//   cost             sum over the function's cost intervals, in list order, of
//                    (sm/100.0 * quota/100.0) * (max(0, close - start) / 3600000.0) * price,
//                    close = end if end >= 0 else sim_end (compute_cost, sim.py:160-175)
//   cost_per_1k      cost / completed * 1000.0, or 0.0 without completions (sim.py:603-607)
// No sort is needed: late_m is a count (each latency finds how many thresholds lie below it,
// the thresholds being non-decreasing, and a suffix sum over that histogram gives every
// late_m); each order statistic is found by a radix select over the order-preserving bit
// pattern of the doubles (8 passes of 8 bits, all requested ranks at once).  Both give the
// exact values the reference's sorted-list scan gives.  The interval sum is sequential per
// function in the reference's order (one thread), which keeps it bit-identical.
#include <cmath>
#include <cstring>
#include <vector>

#include "rapp_internal.h"

namespace rapp {

constexpr int kMetThreads = 512;
constexpr int kMaxMult = 64;
constexpr int kMaxPct = 8;

__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // total order on the bit patterns
}

__device__ __forceinline__ double key_value(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

struct MetricsDev {
  int32_t F, n_mult, n_pct, slo_sorted;
  const double* baseline;
  const int64_t* counts;  // [F][4] arrived, rejected, unfinished, completed
  const int64_t* lat_off;
  const double* lat;
  const int64_t* iv_off;
  const double* iv;  // [I][4] start, end, sm, quota
  double price, end_ms;
  const double* mult;
  const int32_t* pct_q;
  double* curve;  // [F][n_mult]
  double* pct;    // [F][n_pct]
  double* cost;
  double* cost_per_1k;
};

__global__ void __launch_bounds__(kMetThreads) k_metrics(MetricsDev d) {
  const int f = blockIdx.x;
  __shared__ double s_slo[kMaxMult];
  __shared__ unsigned int s_hist[kMaxPct][256];
  __shared__ unsigned long long s_late[kMaxMult + 1];
  __shared__ unsigned long long s_prefix[kMaxPct];
  __shared__ unsigned long long s_rank[kMaxPct];  // remaining rank inside the prefix bucket
  const int tid = threadIdx.x;
  const int64_t b0 = d.lat_off[f], n = d.lat_off[f + 1] - b0;
  const double* L = d.lat + b0;
  const double base = d.baseline[f];
  for (int m = tid; m < d.n_mult; m += blockDim.x) s_slo[m] = __dmul_rn(base, d.mult[m]);
  for (int m = tid; m <= d.n_mult; m += blockDim.x) s_late[m] = 0;
  __syncthreads();

  // ---- late counts ----------------------------------------------------------------------
  if (d.slo_sorted) {
    // idx = number of thresholds strictly below the latency; late_m = #{idx > m}
    unsigned int local[kMaxMult + 1];
    for (int m = 0; m <= d.n_mult; ++m) local[m] = 0;
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const double x = L[i];
      int lo = 0, hi = d.n_mult;  // first m with !(slo[m] < x)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_slo[mid] < x) lo = mid + 1; else hi = mid;
      }
      local[lo] += 1;
    }
    for (int m = 0; m <= d.n_mult; ++m)
      if (local[m]) atomicAdd(&s_late[m], (unsigned long long)local[m]);
  } else {
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const double x = L[i];
      for (int m = 0; m < d.n_mult; ++m)
        if (x > s_slo[m]) atomicAdd(&s_late[m], 1ull);
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int64_t* c = d.counts + 4 * int64_t(f);
    const int64_t arrived = c[0], other = c[1] + c[2];
    unsigned long long suffix = 0;
    for (int m = d.n_mult - 1; m >= 0; --m) {
      unsigned long long late;
      if (d.slo_sorted) {
        suffix += s_late[m + 1];
        late = suffix;
      } else {
        late = s_late[m];
      }
      const int64_t bad = int64_t(late) + other;
      d.curve[int64_t(f) * d.n_mult + m] =
          arrived ? __ddiv_rn(double(bad), double(arrived)) : 0.0;
    }
    // cost: the function's intervals in list order (compute_cost)
    double cost = 0.0;
    for (int64_t k = d.iv_off[f]; k < d.iv_off[f + 1]; ++k) {
      const double* v = d.iv + 4 * k;
      const double close = v[1] >= 0.0 ? v[1] : d.end_ms;
      const double dur = __dsub_rn(close, v[0]);
      const double hours = __ddiv_rn(dur > 0.0 ? dur : 0.0, 3600000.0);  // max(0.0, dur)
      const double share = __dmul_rn(__ddiv_rn(v[2], 100.0), __ddiv_rn(v[3], 100.0));
      cost = __dadd_rn(cost, __dmul_rn(__dmul_rn(share, hours), d.price));
    }
    d.cost[f] = cost;
    const int64_t done = c[3];
    d.cost_per_1k[f] = done ? __dmul_rn(__ddiv_rn(cost, double(done)), 1000.0) : 0.0;
    // ranks (1-based) of the requested percentiles: ceil(q / 100.0 * n), clamped
    for (int j = 0; j < d.n_pct; ++j) {
      const double r = ceil(__dmul_rn(__ddiv_rn(double(d.pct_q[j]), 100.0), double(n)));
      int64_t rank = r < double(n) ? int64_t(r) : n;  // min(len, rank)
      rank = rank - 1 > 0 ? rank - 1 : 0;              // max(0, . - 1)
      s_rank[j] = (unsigned long long)rank;
      s_prefix[j] = 0;
    }
  }
  __syncthreads();
  if (n == 0) {
    for (int j = tid; j < d.n_pct; j += blockDim.x) d.pct[int64_t(f) * d.n_pct + j] = nan("");
    return;
  }
  // ---- radix select: all requested ranks, most significant byte first -------------------
  for (int pass = 7; pass >= 0; --pass) {
    const int shift = pass * 8;
    for (int i = tid; i < d.n_pct * 256; i += blockDim.x) s_hist[i / 256][i % 256] = 0;
    __syncthreads();
    const unsigned long long hmask = pass == 7 ? 0ull : (~0ull << (shift + 8));
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const unsigned long long k = order_key(L[i]);
      const unsigned int digit = unsigned((k >> shift) & 0xFF);
      for (int j = 0; j < d.n_pct; ++j)
        if ((k & hmask) == s_prefix[j]) atomicAdd(&s_hist[j][digit], 1u);
    }
    __syncthreads();
    if (tid < d.n_pct) {
      const int j = tid;
      unsigned long long r = s_rank[j];
      int digit = 0;
      for (; digit < 255; ++digit) {
        if (r < s_hist[j][digit]) break;
        r -= s_hist[j][digit];
      }
      s_rank[j] = r;
      s_prefix[j] |= (unsigned long long)digit << shift;
    }
    __syncthreads();
  }
  for (int j = tid; j < d.n_pct; j += blockDim.x)
    d.pct[int64_t(f) * d.n_pct + j] = key_value(s_prefix[j]);
}

}  // namespace rapp

using namespace rapp;

extern "C" int rapp_metrics_finalize(rapp_ctx* ctx, int64_t n_fns, const double* baseline_ms,
                                     const int64_t* counts, const int64_t* lat_off,
                                     const double* latencies, const int64_t* iv_off,
                                     const double* intervals, double price_per_gpu_hour,
                                     double end_ms, int32_t n_mult, const double* multipliers,
                                     int32_t n_pct, const int32_t* pct_q, double* curve_out,
                                     double* pct_out, double* cost_out,
                                     double* cost_per_1k_out) {
  if (!ctx || n_fns < 0 || n_mult < 0 || n_mult > kMaxMult || n_pct < 0 || n_pct > kMaxPct ||
      (n_fns > 0 && (!baseline_ms || !counts || !lat_off || !iv_off || !curve_out ||
                     !pct_out || !cost_out || !cost_per_1k_out))) {
    set_error("bad arguments (at most %d multipliers and %d percentiles)", kMaxMult, kMaxPct);
    return RAPP_E_ARG;
  }
  if (n_fns == 0) return RAPP_OK;
  RAPP_CUDA(cudaSetDevice(ctx->device));
  const int64_t nlat = lat_off[n_fns], niv = iv_off[n_fns];
  bool sorted = true;  // thresholds baseline * m non-decreasing for every function
  for (int64_t f = 0; f < n_fns && sorted; ++f)
    for (int m = 1; m < n_mult; ++m)
      if (!(baseline_ms[f] * multipliers[m - 1] <= baseline_ms[f] * multipliers[m])) {
        sorted = false;
        break;
      }
  // one device buffer for inputs and outputs
  const size_t in_b = size_t(n_fns) * 8 + size_t(n_fns) * 32 + size_t(n_fns + 1) * 16 +
                      size_t(nlat) * 8 + size_t(niv) * 32 + size_t(n_mult) * 8 + size_t(n_pct) * 4;
  const size_t out_b = size_t(n_fns) * (size_t(n_mult) + size_t(n_pct) + 2) * 8;
  char* buf = nullptr;
  RAPP_CUDA(cudaMalloc(&buf, in_b + out_b + 256));
  std::vector<char> host(in_b);
  size_t off = 0;
  auto put = [&](const void* src, size_t bytes) {
    const size_t o = off;
    if (bytes) std::memcpy(host.data() + o, src, bytes);
    off += (bytes + 7) & ~size_t(7);
    return o;
  };
  MetricsDev d{};
  d.F = int32_t(n_fns);
  d.n_mult = n_mult;
  d.n_pct = n_pct;
  d.slo_sorted = sorted ? 1 : 0;
  const size_t o_base = put(baseline_ms, size_t(n_fns) * 8);
  const size_t o_cnt = put(counts, size_t(n_fns) * 32);
  const size_t o_loff = put(lat_off, size_t(n_fns + 1) * 8);
  const size_t o_lat = put(latencies, size_t(nlat) * 8);
  const size_t o_ioff = put(iv_off, size_t(n_fns + 1) * 8);
  const size_t o_iv = put(intervals, size_t(niv) * 32);
  const size_t o_mult = put(multipliers, size_t(n_mult) * 8);
  const size_t o_pq = put(pct_q, size_t(n_pct) * 4);
  const size_t used = off;
  cudaError_t e = cudaMemcpy(buf, host.data(), used, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(buf);
    RAPP_CUDA(e);
  }
  d.baseline = reinterpret_cast<const double*>(buf + o_base);
  d.counts = reinterpret_cast<const int64_t*>(buf + o_cnt);
  d.lat_off = reinterpret_cast<const int64_t*>(buf + o_loff);
  d.lat = reinterpret_cast<const double*>(buf + o_lat);
  d.iv_off = reinterpret_cast<const int64_t*>(buf + o_ioff);
  d.iv = reinterpret_cast<const double*>(buf + o_iv);
  d.mult = reinterpret_cast<const double*>(buf + o_mult);
  d.pct_q = reinterpret_cast<const int32_t*>(buf + o_pq);
  d.price = price_per_gpu_hour;
  d.end_ms = end_ms;
  double* out = reinterpret_cast<double*>(buf + ((used + 255) & ~size_t(255)));
  d.curve = out;
  d.pct = out + n_fns * n_mult;
  d.cost = d.pct + n_fns * n_pct;
  d.cost_per_1k = d.cost + n_fns;
  k_metrics<<<(unsigned)n_fns, kMetThreads>>>(d);
  e = cudaGetLastError();
  g_launches.fetch_add(1, std::memory_order_relaxed);
  std::vector<double> h(size_t(n_fns) * (n_mult + n_pct + 2));
  if (e == cudaSuccess)
    e = cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  RAPP_CUDA(e);
  std::memcpy(curve_out, h.data(), size_t(n_fns) * n_mult * 8);
  std::memcpy(pct_out, h.data() + n_fns * n_mult, size_t(n_fns) * n_pct * 8);
  std::memcpy(cost_out, h.data() + n_fns * (n_mult + n_pct), size_t(n_fns) * 8);
  std::memcpy(cost_per_1k_out, h.data() + n_fns * (n_mult + n_pct + 1), size_t(n_fns) * 8);
  return RAPP_OK;
}
