// K2 fast path: stream interpolation for validated tables.
//
// Used when every axis is strictly ascending and every grid value is finite and > 0 —
// true of every PerfTable, whose loader rejects non-positive latencies (hs/perf.py:239-267).
// Results are bit-identical to the literal kernel (rapp_core.cu) and the reference
// (hs/_kernels/_grid_cy.pyx:9-51).  What changes is the work layout:
//
//  1. locate() without a binary search.  For a strictly ascending axis the binary search
//     returns the unique lo with a[lo] <= x < a[lo+1]; any method that finds that index
//     exactly is equivalent.  Two per-axis modes, chosen at upload:
//       UNIFORM  a[k] == a0 + k*h exactly with h a power of two (sm% / quota% 1..100):
//                lo from the exact quotient RN(x - a0) / h, no memory access.
//       LUT      a bucket table in shared memory gives the interval; buckets that lie
//                (with a one-bucket margin) inside a single interval are flagged exact,
//                the rest are corrected by exact comparisons.
//  2. t = (x - a[lo]) / (a[hi] - a[lo]): for a power-of-two width the quotient is an exact
//     multiply by the (exactly representable) reciprocal: RN(n * 2^-e) == RN(n / 2^e).
//     Other widths use the IEEE division.
//  3. "Cell" layout: the 8 corners of every grid cell (i, j, k) — v[i or i+1, j or j+1,
//     k or k+1], indices clamped to the last node — are stored contiguously (64 B, 64-B
//     aligned), one cell per node on each axis.  Clamps and node hits (the reference's
//     lo == hi brackets) use cell lo with t = 0: c + (d - c) * 0 == c exactly for finite
//     positive c, d, so the result equals the reference's v[lo] + (v[lo] - v[lo]) * 0.
//     NaN coordinates produce NaN exactly as the reference does (cell 0, t = NaN).
//  4. Two lanes cooperate on their two queries: load r of the pair fetches the cell of
//     query r (owned by lane 2p+r), lane h keeping batch row h (4 doubles, one 256-bit
//     load) — both lanes hit the same 64-byte cell in one instruction, so a warp-wide load
//     touches 16 lines.  Each lane does the quota and sm lerps of its row for both
//     queries, and one exchange gives each lane the other row of its own query.
//  5. Coordinates: each warp walks 32-row slices grid-stride and loads the next slice
//     (three strided 8-byte streaming loads per lane) before it interpolates the current
//     one (RAPP_STREAM_DIRECT, the default: measured faster than the alternative kept
//     behind RAPP_STREAM_DIRECT=0, a 4-stage TMA (cp.async.bulk) ring in shared memory fed
//     by a producer warp with full/empty mbarriers); outputs are streaming stores.
#include <cmath>
#include <cstring>
#include <vector>

#include "rapp_device.cuh"
#include "rapp_internal.h"

namespace rapp {

constexpr int kLut = 512;  // buckets per axis (LUT mode)
constexpr uint32_t kExact = 0x80000000u;
enum : int { kModeLut = 0, kModeUniform = 1, kModeGeom2 = 2 };

// GEOM2: a[k] == a0 * 2^k with a0 a normal power of two (batch axes 1, 2, 4, ..., 32).
// For a0 < x < a_last the bracket is read off x's binary exponent exactly.
static bool exact_geom2_grid(const double* a, int64_t n) {
  if (n < 2 || !(a[0] > 0.0) || !std::isnormal(a[0])) return false;
  int e;
  if (std::frexp(a[0], &e) != 0.5) return false;
  for (int64_t k = 0; k < n; ++k)
    if (a[k] != std::ldexp(a[0], (int)k) || std::isinf(a[k])) return false;
  return std::isnormal(1.0 / a[n - 1]);  // every reciprocal 2^-e stays exactly representable
}

static FastLayout fast_layout(int64_t nb, int64_t ns, int64_t nq) {
  FastLayout L{};
  L.o_par = 0;
  L.o_lut = 24;
  L.o_iv_b = L.o_lut + 3 * kLut / 2;
  L.o_iv_s = L.o_iv_b + int32_t(2 * nb);
  L.o_iv_q = L.o_iv_s + int32_t(2 * ns);
  L.o_cells = (L.o_iv_q + int32_t(2 * nq) + 7) & ~7;  // 64-byte aligned cells
  L.small_doubles = L.o_cells;
  L.total_doubles = int32_t(L.o_cells + nb * ns * nq * 8);
  return L;
}

static bool pow2_recip(double d, double* r) {
  if (!(d > 0.0) || std::isinf(d)) return false;
  int e;
  const double m = std::frexp(d, &e);  // d = m * 2^e, m in [0.5, 1)
  if (m != 0.5) return false;
  const double inv = 1.0 / d;
  if (inv == 0.0 || std::isinf(inv) || inv * d != 1.0) return false;
  *r = inv;
  return true;
}

// True when a[k] == a0 + k*h holds exactly in the reals for every k (checked in scaled
// int64 arithmetic).  Then every fma(k, h, a0) is exact and equals a[k], every interval
// width a[k+1] - a[k] is exactly h, and x strictly between a0 + i*h and a0 + (i+1)*h
// can be read off the exact quotient RN(x - a0) / h (see locate_fast<kModeUniform>).
static bool exact_uniform_grid(const double* a, int64_t n, double h) {
  auto scale_of = [](double v) -> int {  // smallest e >= 0 with v * 2^e integral
    if (v == 0.0) return 0;
    for (int e = 0; e <= 1100; ++e) {
      const double w = std::ldexp(v, e);
      if (std::isinf(w)) return -1;
      if (w == std::floor(w)) return e;
    }
    return -1;
  };
  if (scale_of(a[0]) < 0 || scale_of(h) < 0) return false;
  const int e = std::max(scale_of(a[0]), scale_of(h));
  const double A0 = std::ldexp(a[0], e), H = std::ldexp(h, e);
  const double lim = 4.0e18;  // stay well inside int64
  if (std::fabs(A0) + std::fabs(H) * double(n) > lim) return false;
  const int64_t ia0 = (int64_t)A0, ih = (int64_t)H;
  for (int64_t k = 0; k < n; ++k) {
    const double w = std::ldexp(a[k], e);
    if (w != std::floor(w) || std::fabs(w) > lim) return false;
    if ((int64_t)w != ia0 + k * ih) return false;
  }
  return true;
}

// Builds the fast-path extras; RAPP_E_ARG when the table does not qualify.
// params per axis (8 doubles): a0, a_last, lut_scale, mode, h, 1/h, n, 0
int build_fast_extras(int64_t nb, int64_t ns, int64_t nq, const double* b, const double* s,
                      const double* q, const double* v, std::vector<double>& ext,
                      FastLayout& L) {
  const int64_t ncell = nb * ns * nq;
  if (ncell >= (int64_t(1) << 27)) return RAPP_E_ARG;  // int32 cell index * 8 doubles
  for (int64_t i = 0; i < ncell; ++i)
    if (!(v[i] > 0.0) || std::isinf(v[i])) return RAPP_E_ARG;  // finite, positive only
  L = fast_layout(nb, ns, nq);
  ext.assign((size_t)L.total_doubles, 0.0);
  const double* axes[3] = {b, s, q};
  const int64_t lens[3] = {nb, ns, nq};
  const int32_t o_iv[3] = {L.o_iv_b, L.o_iv_s, L.o_iv_q};
  uint32_t* lut = reinterpret_cast<uint32_t*>(ext.data() + L.o_lut);
  for (int a = 0; a < 3; ++a) {
    const double* ax = axes[a];
    const int64_t n = lens[a];
    const double a0 = ax[0], al = ax[n - 1];
    double* par = ext.data() + L.o_par + 8 * a;
    double scale = 0.0;
    if (n > 1 && std::isfinite(al - a0) && (al - a0) > 0.0) scale = double(kLut) / (al - a0);
    par[0] = a0;
    par[1] = al;
    par[2] = scale;
    par[6] = double(n);
    // UNIFORM: power-of-two step h and every node EXACTLY a0 + k*h as a real number
    double h = n > 1 ? ax[1] - ax[0] : 0.0, invh = 0.0;
    const bool uniform = n > 1 && pow2_recip(h, &invh) && exact_uniform_grid(ax, n, h);
    const bool geom2 = !uniform && a == 0 && exact_geom2_grid(ax, n);  // batch axis only
    par[3] = uniform ? kModeUniform : geom2 ? kModeGeom2 : kModeLut;
    if (uniform) L.modes |= 1 << a;
    if (geom2) L.modes |= 8;
    par[4] = uniform ? h : 0.0;
    par[5] = uniform ? invh : 0.0;
    if (geom2) {
      int e0;
      std::frexp(a0, &e0);
      par[4] = double(e0 - 1);  // binary exponent of a0
    }
    // bucket k covers lut-space [k, k+1); its start in x-space:
    auto xs = [&](int64_t k) -> double {
      if (k <= 0) return a0;
      if (k >= kLut) return al;
      return a0 + (al - a0) * (double(k) / kLut);
    };
    auto interval_of = [&](double x) -> int64_t {  // largest i <= n-2 with a[i] <= x
      int64_t i = 0;
      while (i + 1 <= n - 2 && ax[i + 1] <= x) ++i;
      return i;
    };
    for (int64_t k = 0; k < kLut; ++k) {
      const int64_t i = interval_of(xs(k));
      // exact if buckets k-1..k+1 (the computed bucket is off by at most one) lie in
      // (a[i], a[i+1]) with room to spare
      bool exact = n >= 2 && ax[i] < xs(k - 1) && xs(k + 2) < ax[i + 1];
      if (k == 0) exact = n >= 2 && xs(k + 2) < ax[i + 1];  // x > a0 == a[0] is known
      if (k == kLut - 1) exact = n >= 2 && ax[i] < xs(k - 1) && i == n - 2;  // x < a_last
      lut[a * kLut + k] = uint32_t(i) | (exact ? kExact : 0u);
    }
    // intervals: iv[i] = (a[i], exact reciprocal of a[i+1]-a[i] or 0); iv[n-1] = (a_last, 0)
    double* iv = ext.data() + o_iv[a];
    for (int64_t i = 0; i < n; ++i) {
      double r = 0.0;
      if (i + 1 < n && !pow2_recip(ax[i + 1] - ax[i], &r)) r = 0.0;
      iv[2 * i] = ax[i];
      iv[2 * i + 1] = r;
    }
  }
  double* cells = ext.data() + L.o_cells;
  for (int64_t i = 0; i < nb; ++i)
    for (int64_t j = 0; j < ns; ++j)
      for (int64_t k = 0; k < nq; ++k) {
        double* c = cells + ((i * ns + j) * nq + k) * 8;
        for (int d = 0; d < 8; ++d) {  // corner d = (db << 2) | (ds << 1) | dq
          const int64_t ii = std::min(i + ((d >> 2) & 1), nb - 1);
          const int64_t jj = std::min(j + ((d >> 1) & 1), ns - 1);
          const int64_t kk = std::min(k + (d & 1), nq - 1);
          c[d] = v[(ii * ns + jj) * nq + kk];
        }
      }
  return RAPP_OK;
}

#ifndef RAPP_LOCATE_MAGIC
#define RAPP_LOCATE_MAGIC 0  // 1: uniform locate without F2I/I2F (measured 4% slower)
#endif

struct FastAxis {
  const uint32_t* lut;
  const double2* iv;
  int last;
  int e0;  // geom2: binary exponent of a0 (params[4]), converted once per CTA
  double a0, al, scale, h, invh;
  double topd;  // last - 1 as a double (the uniform locate's clamp)
};

__device__ __forceinline__ FastAxis load_axis(const double* ext, int a, const uint32_t* lut,
                                              const double* iv) {
  const double* p = ext + 8 * a;
  FastAxis ax;
  ax.lut = lut + a * kLut;
  ax.iv = reinterpret_cast<const double2*>(iv);
  ax.a0 = p[0];
  ax.al = p[1];
  ax.scale = p[2];
  ax.h = p[4];
  ax.invh = p[5];
  ax.last = int(p[6]) - 1;
  ax.e0 = int(p[4]);
  ax.topd = double(ax.last - 1);
  return ax;
}

// Clamps and NaN (rare).  Cell and t reproduce the reference's (lo, hi, t):
// x <= a0 -> (0,0,0); x >= a_last -> (last,last,0); NaN -> (0, min(1,last), NaN).
__device__ __forceinline__ void locate_edge(const FastAxis& ax, double x, int& c, double& t) {
  if (x <= ax.a0) { c = 0; t = 0.0; return; }
  if (x >= ax.al) { c = ax.last; t = 0.0; return; }
  c = 0;
  const int hi = ax.last > 0 ? 1 : 0;
  t = __ddiv_rn(__dsub_rn(x, ax.a0), __dsub_rn(ax.iv[hi].x, ax.a0));
}

// Cell c (== the reference's lo) and t for x (node hits give t = 0).
template <int MODE>
__device__ __forceinline__ void locate_fast(const FastAxis& ax, double x, int& c, double& t) {
  if (!(x > ax.a0 && x < ax.al)) {  // clamps and NaN all fail this test
    locate_edge(ax, x, c, t);
    return;
  }
  const int top = ax.last - 1;  // a0 < x < a_last: n >= 2 and lo lies in [0, n-2]
  if (MODE == kModeGeom2) {
    // x is normal and a0*2^i <= x < a0*2^(i+1)  <=>  exponent(x) == exponent(a0) + i.
    // lo = 2^ex exactly; width a[i+1] - a[i] = 2^ex, so t = RN((x - lo) * 2^-ex) exactly.
    const int ex = ((__double2hiint(x) >> 20) & 0x7FF) - 1023;
    c = ex - ax.e0;
    const double lo = __hiloint2double((ex + 1023) << 20, 0);
    const double inv = __hiloint2double((1023 - ex) << 20, 0);
    t = __dmul_rn(__dsub_rn(x, lo), inv);
    return;
  }
  if (MODE == kModeUniform) {
    // u = RN(x - a0) / h is exact.  If u is not an integer, i = trunc(u) satisfies
    // i*h < RN(x - a0) < (i+1)*h, and since every a0 + k*h is exact and RN monotone,
    // a[i] < x < a[i+1].  If u is integral, x is within rounding of a node: compare.
    const double u = __dmul_rn(__dsub_rn(x, ax.a0), ax.invh);
#if RAPP_LOCATE_MAGIC
    // trunc(u) without the (reduced-rate) F2I/I2F conversions: 0 <= u < 2^52, so
    // RZ(u + 2^52) = 2^52 + trunc(u) exactly; its low word is trunc(u) and subtracting
    // 2^52 back is exact.  Same (i, fi) as min(int(u), top), double(i).
    const double big = __dadd_rz(u, 0x1p52);
    int i = min(__double2loint(big), top);
    double fi = fmin(__dsub_rn(big, 0x1p52), ax.topd);
#else
    int i = min(int(u), top);
    double fi = double(i);
#endif
    double lo = fma(fi, ax.h, ax.a0);  // exact: == a[i]
    if (fi == u) {
      if (lo > x) {
        --i;
        fi = __dsub_rn(fi, 1.0);
        lo = fma(fi, ax.h, ax.a0);
      } else if (i < top) {
        const double nx = fma(__dadd_rn(fi, 1.0), ax.h, ax.a0);
        if (nx <= x) {
          ++i;
          lo = nx;
        }
      }
    }
    c = i;
    t = __dmul_rn(__dsub_rn(x, lo), ax.invh);  // node hit: x - lo == 0 -> t = 0
    return;
  }
  const int k = min(int(__dmul_rn(__dsub_rn(x, ax.a0), ax.scale)), kLut - 1);
  const uint32_t e = ax.lut[k];
  int i = int(e & ~kExact);
  if (!(e & kExact)) {
    while (i < top && ax.iv[i + 1].x <= x) ++i;
    while (i > 0 && ax.iv[i].x > x) --i;
  }
  const double2 w = ax.iv[i];
  c = i;
  const double num = __dsub_rn(x, w.x);  // node hit: 0 -> t = 0 either way
  t = w.y != 0.0 ? __dmul_rn(num, w.y) : __ddiv_rn(num, __dsub_rn(ax.iv[i + 1].x, w.x));
}

__device__ __forceinline__ void load_row(const double* p, bool smem, double& v0, double& v1,
                                         double& v2, double& v3) {
  if (smem) {
    const double2 a = reinterpret_cast<const double2*>(p)[0];
    const double2 b = reinterpret_cast<const double2*>(p)[1];
    v0 = a.x; v1 = a.y; v2 = b.x; v3 = b.y;
  } else {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3)
        : "l"(p));
  }
}

#ifndef RAPP_STREAM_DIRECT
// 1: every row by direct loads with a one-slice prefetch (no TMA ring): 0.386-0.387 ms vs
// 0.394-0.395 ms per 5e7 config-2 queries for the ring (same box, tools/ab_stream.sh); the
// ring's cp.async.bulk reads and its smem reads/mbarrier polls cost more L1 wavefronts
// than the three strided 8-byte loads per lane
#define RAPP_STREAM_DIRECT 1
#endif
#ifndef RAPP_STREAM_TEX
#define RAPP_STREAM_TEX 0  // 1: the partner query's cell through the texture pipe, 2: both
#endif
#ifndef RAPP_STREAM_MINB
#define RAPP_STREAM_MINB 2
#endif
#ifndef RAPP_STREAM_CONSUMERS
#define RAPP_STREAM_CONSUMERS 16
#endif
#ifndef RAPP_STREAM_ROWS
#define RAPP_STREAM_ROWS 1  // 2 rows per lane (3 stages): same speed, measured
#endif
#ifndef RAPP_STREAM_STAGES
#define RAPP_STREAM_STAGES 4
#endif
#ifndef RAPP_STREAM_SUSPEND_NS
#define RAPP_STREAM_SUSPEND_NS 0
#endif
constexpr int kConsumers = RAPP_STREAM_CONSUMERS;  // consumer warps per CTA
constexpr int kProducer = kConsumers;              // warp index of the TMA producer
constexpr int kFastThreads = (kConsumers + 1) * 32;
// rows per consumer lane per stage: each full/empty barrier round trip (and its
// shared-memory polls) is paid once per kRows rows.  Measured on config 2: 2 rows x 3
// stages runs at the speed of 1 row x 4 stages (0.394 ms per 5e7 queries), 2 x 4 stages is
// 14% slower (one CTA per SM), a try_wait suspend-time hint changes nothing.
constexpr int kRows = RAPP_STREAM_ROWS;
constexpr int kTile = kConsumers * 32 * kRows;  // rows per TMA stage
constexpr int kStages = RAPP_STREAM_STAGES;

// One row per lane (row index i, coordinates x0..x2); see the header comment, item 4.
template <int MB, int MS, int MQ, bool CELLS_SMEM>
__device__ __forceinline__ void interp_row(const FastAxis& ab, const FastAxis& as,
                                           const FastAxis& aq, const double* cells, int CS,
                                           int CQ, double xb, double xs, double xq, int64_t i,
                                           int64_t n, double* __restrict__ out,
                                           double* __restrict__ rps,
                                           cudaTextureObject_t tex, int tcell0) {
  const int half = threadIdx.x & 1;
  int ib, js, kq;
  double tb, ts, tq;
  locate_fast<MB>(ab, xb, ib, tb);
  locate_fast<MS>(as, xs, js, ts);
  locate_fast<MQ>(aq, xq, kq, tq);
  const int cell = (ib * CS + js) * CQ + kq;
  const int cell_p = __shfl_xor_sync(0xffffffffu, cell, 1);
  const double tq_p = __shfl_xor_sync(0xffffffffu, tq, 1);
  const double ts_p = __shfl_xor_sync(0xffffffffu, ts, 1);
  // query r of the pair is owned by lane 2p + r
  const int c0 = half ? cell_p : cell, c1 = half ? cell : cell_p;
  double v[2][4];
#if RAPP_STREAM_TEX
  if (!CELLS_SMEM) {
    // texels are 16 bytes: cell c = texels 4c..4c+3, row `half` = texels 4c + 2 half + {0,1}
    auto tex_row = [&](int c, double& a0, double& a1, double& a2, double& a3) {
      const int t = tcell0 + 4 * c + 2 * half;
      const int4 p = tex1Dfetch<int4>(tex, t), q = tex1Dfetch<int4>(tex, t + 1);
      a0 = __hiloint2double(p.y, p.x); a1 = __hiloint2double(p.w, p.z);
      a2 = __hiloint2double(q.y, q.x); a3 = __hiloint2double(q.w, q.z);
    };
    if (RAPP_STREAM_TEX >= 2) tex_row(c0, v[0][0], v[0][1], v[0][2], v[0][3]);
    else load_row(cells + int64_t(c0) * 8 + half * 4, false, v[0][0], v[0][1], v[0][2], v[0][3]);
    tex_row(c1, v[1][0], v[1][1], v[1][2], v[1][3]);
  } else
#endif
  {
    load_row(cells + int64_t(c0) * 8 + half * 4, CELLS_SMEM, v[0][0], v[0][1], v[0][2], v[0][3]);
    load_row(cells + int64_t(c1) * 8 + half * 4, CELLS_SMEM, v[1][0], v[1][1], v[1][2], v[1][3]);
  }
  // row h of each query: lerp(lerp(v[j0,k0], v[j0,k1], tq), lerp(v[j1,k0], v[j1,k1], tq), ts)
  const double tq0 = half ? tq_p : tq, tq1 = half ? tq : tq_p;
  const double ts0 = half ? ts_p : ts, ts1 = half ? ts : ts_p;
  const double r0 = lerp_rn(lerp_rn(v[0][0], v[0][1], tq0), lerp_rn(v[0][2], v[0][3], tq0), ts0);
  const double r1 = lerp_rn(lerp_rn(v[1][0], v[1][1], tq1), lerp_rn(v[1][2], v[1][3], tq1), ts1);
  const double mine = half ? r1 : r0;   // row h of my query
  const double theirs = half ? r0 : r1;  // row h of my partner's query
  const double other = __shfl_xor_sync(0xffffffffu, theirs, 1);  // row 1-h of my query
  const double lat = half ? lerp_rn(other, mine, tb) : lerp_rn(mine, other, tb);
  if (i < n) {
    __stcs(out + i, lat);
    if (rps != nullptr) __stcs(rps + i, throughput(xb, lat));
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
      (uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
      (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done) {
#if RAPP_STREAM_SUSPEND_NS > 0
    // suspend-time hint: the warp sleeps in the barrier until the phase completes (or the
    // hint expires) instead of re-polling it through the shared-memory pipe
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(sbar), "r"(parity), "n"(RAPP_STREAM_SUSPEND_NS)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(sbar), "r"(parity)
        : "memory");
#endif
  }
}

// One elected thread: bulk-copy `bytes` from global to shared, completing on `bar`.
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"(sbar)
      : "memory");
}

// Persistent CTAs stream full kTile-row tiles of coordinates through a kStages-deep TMA
// ring: one producer warp issues cp.async.bulk into free stages (full/empty mbarriers),
// kConsumers warps each take 32 rows of a stage, release it as soon as the rows are in
// registers, and interpolate.  Rows past the last full tile (or everything, when coords
// is not 16-byte aligned) use direct loads.
template <int MB, int MS, int MQ, bool CELLS_SMEM>
__global__ void __launch_bounds__(kFastThreads, RAPP_STREAM_MINB)
    k_interp_fast(const TableDesc td, const double* __restrict__ pool,
                  const double* __restrict__ coords, int64_t n, int64_t n_tiles,
                  double* __restrict__ out, double* __restrict__ rps,
                  cudaTextureObject_t tex, int tcell0) {
  extern __shared__ __align__(128) double sm[];
  __shared__ uint64_t bar_ext;
  __shared__ uint64_t full[kStages], empty[kStages];
  const double* ext_g = pool + td.xoff;
  const int ext_doubles = CELLS_SMEM ? td.x_total : td.x_small;
  double* buf0 = sm + ((ext_doubles + 15) & ~15);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
  }
  bulk_load_2(sm, ext_g, uint32_t(ext_doubles) * 8u, nullptr, nullptr, 0u, &bar_ext);
  const double* cells = CELLS_SMEM ? sm + td.x_small : ext_g + td.x_small;
  const uint32_t* lut = reinterpret_cast<const uint32_t*>(sm + 24);
  const FastAxis ab = load_axis(sm, 0, lut, sm + td.x_iv_b);
  const FastAxis as = load_axis(sm, 1, lut, sm + td.x_iv_s);
  const FastAxis aq = load_axis(sm, 2, lut, sm + td.x_iv_q);
  const int CS = td.ns, CQ = td.nq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == kProducer) {
    if (lane == 0) {
      int64_t t = blockIdx.x;
      for (int j = 0; t < n_tiles; ++j, t += gridDim.x) {
        const int s = j % kStages;
        if (j >= kStages) mbar_wait(&empty[s], ((j / kStages) - 1) & 1);  // stage released
        tma_load(buf0 + s * 3 * kTile, coords + 3 * t * kTile, kTile * 24u, &full[s]);
      }
    }
    return;  // no CTA-wide barrier follows
  }
  int64_t t = blockIdx.x;
  for (int j = 0; t < n_tiles; ++j, t += gridDim.x) {
    const int s = j % kStages;
    mbar_wait(&full[s], (j / kStages) & 1);
    // this warp's kRows x 32 rows of the stage, row r of lane l at (r * kConsumers + warp)
    // * 32 + l: each LDS.64 and each output store stays a contiguous 32-row slice
    double x[kRows][3];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const double* row = buf0 + s * 3 * kTile + 3 * ((r * kConsumers + warp) * 32 + lane);
      x[r][0] = row[0];
      x[r][1] = row[1];
      x[r][2] = row[2];
    }
    // The next TMA write into this stage is an async-proxy access; order our generic-proxy
    // reads before it (WAR across proxies), then release the stage.
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp's rows are in registers
#pragma unroll
    for (int r = 0; r < kRows; ++r)
      interp_row<MB, MS, MQ, CELLS_SMEM>(ab, as, aq, cells, CS, CQ, x[r][0], x[r][1], x[r][2],
                                         t * kTile + (r * kConsumers + warp) * 32 + lane, n,
                                         out, rps, tex, tcell0);
  }
  // remainder rows (all rows when RAPP_STREAM_DIRECT): direct loads, warp-uniform
  // grid-stride (every lane shuffles); the next slice's coordinates are loaded before this
  // slice is interpolated
  const int64_t warps_total = int64_t(gridDim.x) * kConsumers;
  const int64_t wstride = warps_total * 32;
  int64_t wb = n_tiles * kTile + (int64_t(blockIdx.x) * kConsumers + warp) * 32;
  double nb = ab.a0, ns = as.a0, nq = aq.a0;  // harmless in-range filler past the end
  if (wb + lane < n) {
    nb = __ldcs(coords + 3 * (wb + lane));
    ns = __ldcs(coords + 3 * (wb + lane) + 1);
    nq = __ldcs(coords + 3 * (wb + lane) + 2);
  }
  for (; wb < n; wb += wstride) {
    const int64_t i = wb + lane;
    const double xb = nb, xs = ns, xq = nq;
    const int64_t j = i + wstride;
    if (j < n) {
      nb = __ldcs(coords + 3 * j);
      ns = __ldcs(coords + 3 * j + 1);
      nq = __ldcs(coords + 3 * j + 2);
    } else {
      nb = ab.a0; ns = as.a0; nq = aq.a0;
    }
    interp_row<MB, MS, MQ, CELLS_SMEM>(ab, as, aq, cells, CS, CQ, xb, xs, xq, i, n, out, rps,
                                       tex, tcell0);
  }
}

constexpr int64_t kFastCellsSmem = 96 * 1024;

template <int MB, int MS, int MQ>
static void launch_modes(bool cells_smem, unsigned blocks, size_t smem, cudaStream_t st,
                         const TableDesc& td, const double* pool, const double* coords,
                         int64_t n, int64_t n_tiles, double* out, double* rps,
                         cudaTextureObject_t tex, int tcell0) {
  if (cells_smem) {
    auto k = k_interp_fast<MB, MS, MQ, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    k<<<blocks, kFastThreads, smem, st>>>(td, pool, coords, n, n_tiles, out, rps, tex,
                                          tcell0);
  } else {
    auto k = k_interp_fast<MB, MS, MQ, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    k<<<blocks, kFastThreads, smem, st>>>(td, pool, coords, n, n_tiles, out, rps, tex,
                                          tcell0);
  }
}

#if RAPP_STREAM_TEX
// One int4 texture object over the whole table pool, rebuilt when the pool moves or grows.
static int pool_texture(rapp_ctx* ctx, cudaTextureObject_t* out) {
  static std::mutex mu;
  static const double* ptr = nullptr;
  static int64_t cap = -1;
  static cudaTextureObject_t obj = 0;
  std::lock_guard<std::mutex> g(mu);
  if (ptr != ctx->d_pool || cap != ctx->pool_cap) {
    if (obj) cudaDestroyTextureObject(obj);
    obj = 0;
    if (ctx->pool_cap / 2 >= (int64_t(1) << 27)) {
      set_error("table pool too large for the texture path");
      return RAPP_E_ARG;
    }
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = const_cast<double*>(ctx->d_pool);
    rd.res.linear.desc = cudaCreateChannelDesc<int4>();
    rd.res.linear.sizeInBytes = size_t(ctx->pool_cap) * 8;
    cudaTextureDesc tdsc = {};
    tdsc.readMode = cudaReadModeElementType;
    RAPP_CUDA(cudaCreateTextureObject(&obj, &rd, &tdsc, nullptr));
    ptr = ctx->d_pool;
    cap = ctx->pool_cap;
  }
  *out = obj;
  return RAPP_OK;
}
#endif

int launch_interp_fast(rapp_ctx* ctx, const TableDesc& td, const double* d_coords, int64_t n,
                       double* d_out, double* d_rps, cudaStream_t st) {
  const int64_t cell_bytes = int64_t(td.x_total - td.x_small) * 8;
  const int64_t small_bytes = int64_t(td.x_small) * 8;
  const bool cells_smem = cell_bytes + small_bytes <= kFastCellsSmem;
  const int64_t ext_bytes = cells_smem ? small_bytes + cell_bytes : small_bytes;
  const size_t smem = (size_t)(((ext_bytes + 127) & ~int64_t(127)) +
                               (RAPP_STREAM_DIRECT ? 0 : kStages * 3 * kTile * 8));
  if (smem > 220 * 1024) {
    set_error("fast-path shared-memory footprint %zu too large", smem);
    return RAPP_E_ARG;
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(d_coords) & 15) == 0;
  const int64_t n_tiles = aligned && !RAPP_STREAM_DIRECT ? n / kTile : 0;
  int64_t blocks = n_tiles > 0 ? n_tiles : (n + kTile - 1) / kTile;
  const int64_t per_sm = std::max<int64_t>(
      1, std::min<int64_t>(RAPP_STREAM_MINB, (220 * 1024) / (int64_t)(smem + 1024)));
  const int64_t cap = int64_t(ctx->sm_count) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const unsigned nb = (unsigned)blocks;
  const double* pool = ctx->d_pool;
  cudaTextureObject_t tex = 0;
  int tcell0 = 0;
#if RAPP_STREAM_TEX
  if (!cells_smem) {
    int rc = pool_texture(ctx, &tex);
    if (rc != RAPP_OK) return rc;
    tcell0 = int((td.xoff + td.x_small) / 2);  // 64-byte aligned cells: an even double index
  }
#endif
#define RAPP_LM(B, S, Q) \
  launch_modes<B, S, Q>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps, \
                        tex, tcell0)
  // bit 0: batch axis uniform, bit 1: sm uniform, bit 2: quota uniform, bit 3: batch geom2
  switch (td.modes & 15) {
    case 0: RAPP_LM(0, 0, 0); break;
    case 1: RAPP_LM(1, 0, 0); break;
    case 2: RAPP_LM(0, 1, 0); break;
    case 3: RAPP_LM(1, 1, 0); break;
    case 4: RAPP_LM(0, 0, 1); break;
    case 5: RAPP_LM(1, 0, 1); break;
    case 6: RAPP_LM(0, 1, 1); break;
    case 7: RAPP_LM(1, 1, 1); break;
    case 8: RAPP_LM(2, 0, 0); break;
    case 10: RAPP_LM(2, 1, 0); break;
    case 12: RAPP_LM(2, 0, 1); break;
    case 14: RAPP_LM(2, 1, 1); break;
    default: RAPP_LM(0, 0, 0); break;  // not produced by build_fast_extras
  }
#undef RAPP_LM
  RAPP_LAUNCHED();
  return RAPP_OK;
}

}  // namespace rapp
