// Device-side building blocks shared by every kernel of the RaPP path.
//
// All FP64 arithmetic goes through the explicit round-to-nearest intrinsics so that no
// multiply-add is ever contracted (the library is also built with --fmad=false as a
// second guard).  The reference evaluates each `a + (b - a) * t` as a separate sub, mul
// and add in IEEE binary64 (hs/_kernels/_grid_cy.pyx:45-51; x86-64 -O2 without FMA), and
// an FMA changes the last bit on ~18% of interior queries (SURVEY.md finding 0.4).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rapp {

// Programmatic dependent launch: a kernel lets its successor launch once all of its CTAs
// are running (griddepcontrol.launch_dependents) and waits for its predecessor's completion
// (griddepcontrol.wait) only before it reads what the predecessor wrote, so launch latency
// and independent set-up overlap the predecessor's tail.  Kernels launched without the
// programmatic attribute see both as no-ops.
#ifndef RAPP_PDL
#define RAPP_PDL 1
#endif
__device__ __forceinline__ void pdl_trigger() {
#if RAPP_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if RAPP_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// a + (b - a) * t with each operation rounded — one lerp of hs/_kernels/_grid_cy.pyx:45-51.
__device__ __forceinline__ double lerp_rn(double a, double b, double t) {
  return __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), t));
}

// Clamped bracket of x on an ascending axis — hs/_kernels/_grid_cy.pyx:9-33.
//   x <= a[0]      -> (0, 0, 0.0)
//   x >= a[n-1]    -> (n-1, n-1, 0.0)
//   binary search with mid = (lo+hi)>>1 and `a[mid] <= x` -> lo
//   node hit       -> (lo, lo, 0.0)
//   otherwise      -> (lo, hi, (x - a[lo]) / (a[hi] - a[lo]))   (IEEE division)
// NaN x fails every comparison and ends at (0, 1, NaN) exactly like the reference.
__device__ __forceinline__ void locate(const double* __restrict__ a, int n, double x,
                                       int& lo, int& hi, double& t) {
  const int last = n - 1;
  if (x <= a[0]) { lo = 0; hi = 0; t = 0.0; return; }
  if (x >= a[last]) { lo = last; hi = last; t = 0.0; return; }
  int l = 0, h = last;
  while (h - l > 1) {
    const int mid = (l + h) >> 1;
    if (a[mid] <= x) l = mid; else h = mid;
  }
  const double al = a[l];
  if (al == x) { lo = l; hi = l; t = 0.0; return; }
  lo = l;
  hi = h;
  t = __ddiv_rn(__dsub_rn(x, al), __dsub_rn(a[h], al));
}

// Trilinear interpolation in the reference's nesting order — _grid_cy.pyx:36-51.
// v is the C-order (nb, ns, nq) grid.
__device__ __forceinline__ double interp3(const double* __restrict__ ba, int nb,
                                          const double* __restrict__ sa, int ns,
                                          const double* __restrict__ qa, int nq,
                                          const double* __restrict__ v,
                                          double b, double s, double q) {
  int i0, i1, j0, j1, k0, k1;
  double tb, ts, tq;
  locate(ba, nb, b, i0, i1, tb);
  locate(sa, ns, s, j0, j1, ts);
  locate(qa, nq, q, k0, k1, tq);
  const int64_t r00 = (int64_t(i0) * ns + j0) * nq, r01 = (int64_t(i0) * ns + j1) * nq;
  const int64_t r10 = (int64_t(i1) * ns + j0) * nq, r11 = (int64_t(i1) * ns + j1) * nq;
  const double c00 = lerp_rn(v[r00 + k0], v[r00 + k1], tq);
  const double c01 = lerp_rn(v[r01 + k0], v[r01 + k1], tq);
  const double c10 = lerp_rn(v[r10 + k0], v[r10 + k1], tq);
  const double c11 = lerp_rn(v[r11 + k0], v[r11 + k1], tq);
  const double c0 = lerp_rn(c00, c01, ts);
  const double c1 = lerp_rn(c10, c11, ts);
  return lerp_rn(c0, c1, tb);
}

// throughput = batch / (latency_ms / 1000.0) — hs/perf.py:95-98 (two IEEE divisions,
// never rewritten as a reciprocal multiply).
__device__ __forceinline__ double throughput(double batch, double latency_ms) {
  return __ddiv_rn(batch, __ddiv_rn(latency_ms, 1000.0));
}

// Largest positive double `lat` with throughput(b, lat) >= target, or 0.0 when none
// (-> no positive latency is feasible).  throughput(b, .) is monotone non-increasing on
// (0, +inf] because both correctly-rounded divisions are monotone, so
//   throughput(b, lat) >= target  <=>  lat <= threshold(b, target)     for lat > 0,
// which lets the lattice search replace two divisions per point with one compare and
// still reproduce the reference's `rps >= target_rps` test (hs/perf.py:132) bit for bit.
// Search over the ordered bit patterns of (0, +inf]: the boundary is bracketed by galloping
// (steps 1, 2, 4, ... ulps) from the estimate RN(RN(b / target) * 1000), which lies within a
// few ulps of it for finite positive operands, then bisected; the predicate is monotone, so
// the result is the one a bisection of the whole range finds (2-8 evaluations instead of 63).
#ifndef RAPP_THRESHOLD_GALLOP
#define RAPP_THRESHOLD_GALLOP 1
#endif
__device__ __forceinline__ double feasibility_threshold(double b, double target) {
  auto ok = [&](uint64_t bits) {
    return throughput(b, __longlong_as_double((long long)bits)) >= target;
  };
  constexpr uint64_t kLo = 1ull;                   // smallest positive denormal
  constexpr uint64_t kHi = 0x7FF0000000000000ull;  // +inf
  uint64_t lo = kLo, hi = kHi;
  if (!ok(lo)) return 0.0;
  if (ok(hi)) return __longlong_as_double((long long)hi);
#if RAPP_THRESHOLD_GALLOP
  const double g = __dmul_rn(__ddiv_rn(b, target), 1000.0);
  if (g > 0.0 && g < __longlong_as_double((long long)kHi)) {  // NaN fails both
    const uint64_t gb = (uint64_t)__double_as_longlong(g);
    if (ok(gb)) {
      lo = gb;
      for (uint64_t step = 1;; step <<= 1) {  // terminates: !ok(kHi)
        const uint64_t c = kHi - lo > step ? lo + step : kHi;
        if (!ok(c)) { hi = c; break; }
        lo = c;
      }
    } else {
      hi = gb;
      for (uint64_t step = 1;; step <<= 1) {  // terminates: ok(kLo)
        const uint64_t c = hi - kLo > step ? hi - step : kLo;
        if (ok(c)) { lo = c; break; }
        hi = c;
      }
    }
  }
#endif
  while (hi - lo > 1) {                 // invariant: ok(lo) && !ok(hi)
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (ok(mid)) lo = mid; else hi = mid;
  }
  return __longlong_as_double((long long)lo);
}

// ---------------------------------------------------------------------------------------
// Bulk (TMA) copy of a table segment into shared memory.  One elected thread arms an
// mbarrier with the byte count and issues cp.async.bulk; every thread waits on the phase.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void bulk_load_table(double* s_dst, const double* g_src,
                                                uint32_t bytes, uint64_t* bar) {
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar),
                 "r"(bytes)
                 : "memory");
    constexpr uint32_t kChunk = 65536;  // keep each bulk op modest
    for (uint32_t off = 0; off < bytes; off += kChunk) {
      const uint32_t n = bytes - off < kChunk ? bytes - off : kChunk;
      const uint32_t sdst = (uint32_t)__cvta_generic_to_shared((char*)s_dst + off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(sdst),
          "l"((const char*)g_src + off), "r"(n), "r"(sbar)
          : "memory");
    }
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(sbar)
        : "memory");
  }
}

// Two regions in one transaction (e.g. axes + bucket tables).  Either size may be 0;
// sizes and addresses must be multiples of 16 bytes.
__device__ __forceinline__ void bulk_load_2(void* d1, const void* s1, uint32_t n1, void* d2,
                                            const void* s2, uint32_t n2, uint64_t* bar) {
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar),
                 "r"(n1 + n2)
                 : "memory");
    constexpr uint32_t kChunk = 65536;
    const void* srcs[2] = {s1, s2};
    void* dsts[2] = {d1, d2};
    const uint32_t ns[2] = {n1, n2};
    for (int r = 0; r < 2; ++r)
      for (uint32_t off = 0; off < ns[r]; off += kChunk) {
        const uint32_t n = ns[r] - off < kChunk ? ns[r] - off : kChunk;
        const uint32_t sdst = (uint32_t)__cvta_generic_to_shared((char*)dsts[r] + off);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
            "%2, [%3];" ::"r"(sdst),
            "l"((const char*)srcs[r] + off), "r"(n), "r"(sbar)
            : "memory");
      }
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(sbar)
        : "memory");
  }
}

}  // namespace rapp
