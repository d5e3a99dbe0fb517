// K2 fast path: stream interpolation for validated tables (strictly ascending axes).
//
// Same results, bit for bit, as the literal kernel (rapp_core.cu) and the reference
// (hs/_kernels/_grid_cy.pyx:9-51).  What changes is how the work is laid out:
//
//  1. locate() without a binary search.  For a strictly ascending axis the binary search
//     returns the unique lo with a[lo] <= x < a[lo+1]; any method that finds that index
//     exactly is equivalent.  Two per-axis modes, chosen at upload:
//       UNIFORM  a[k] == a0 + k*h exactly with h a power of two (e.g. sm% / quota% 1..100):
//                k = floor((x - a0) / h) corrected by one exact comparison — no memory.
//       LUT      a bucket table in shared memory gives the interval; buckets that lie
//                (with a one-bucket margin) inside a single interval are flagged exact,
//                the rest are corrected by exact comparisons.
//  2. t = (x - a[lo]) / (a[hi] - a[lo]): for a power-of-two width the quotient is an exact
//     multiply by the (exactly representable) reciprocal: RN(n * 2^-e) == RN(n / 2^e).
//     Other widths use the IEEE division.
//  3. "Cell" layout: the 8 corners of each grid cell are stored contiguously (64 B,
//     64-byte aligned).  Two lanes cooperate on one query: each loads one batch row of the
//     cell (4 doubles) with a single 256-bit load and does that row's two quota lerps and
//     its sm lerp; one shuffle exchanges the row values for the batch lerp.  A warp thus
//     touches 16 lines per load instruction instead of 32 x 4.
//     Clamped / node-hit brackets (lo == hi) select the same corner twice, exactly as the
//     reference reads v[lo] twice.
#include <cmath>
#include <cstring>
#include <vector>

#include "rapp_device.cuh"
#include "rapp_internal.h"

namespace rapp {

constexpr int kLut = 512;  // buckets per axis (LUT mode)
constexpr uint32_t kExact = 0x80000000u;
enum : int { kModeLut = 0, kModeUniform = 1 };

static FastLayout fast_layout(int64_t nb, int64_t ns, int64_t nq) {
  FastLayout L{};
  L.o_par = 0;
  L.o_lut = 24;
  L.o_iv_b = L.o_lut + 3 * kLut / 2;
  L.o_iv_s = L.o_iv_b + int32_t(2 * nb);
  L.o_iv_q = L.o_iv_s + int32_t(2 * ns);
  L.o_cells = (L.o_iv_q + int32_t(2 * nq) + 7) & ~7;  // 64-byte aligned cells
  L.small_doubles = L.o_cells;
  const int64_t cb = nb > 1 ? nb - 1 : 1, cs = ns > 1 ? ns - 1 : 1, cq = nq > 1 ? nq - 1 : 1;
  L.total_doubles = int32_t(L.o_cells + cb * cs * cq * 8);
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
// can be read off the exact quotient RN(x - a0) / h (see locate_uniform).
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
  int e = std::max(scale_of(a[0]), scale_of(h));
  if (scale_of(a[0]) < 0 || scale_of(h) < 0) return false;
  const double A0 = std::ldexp(a[0], e), H = std::ldexp(h, e);
  const double lim = 4.0e18;  // stay well inside int64
  if (std::fabs(A0) > lim || std::fabs(H) * double(n) > lim || std::fabs(A0) + std::fabs(H) * double(n) > lim)
    return false;
  const int64_t ia0 = (int64_t)A0, ih = (int64_t)H;
  for (int64_t k = 0; k < n; ++k) {
    const double w = std::ldexp(a[k], e);
    if (w != std::floor(w) || std::fabs(w) > lim) return false;
    if ((int64_t)w != ia0 + k * ih) return false;
  }
  return true;
}

// Builds the fast-path extras for a strictly ascending table.
// params per axis (8 doubles): a0, a_last, lut_scale, mode, h, 1/h, n, 0
int build_fast_extras(int64_t nb, int64_t ns, int64_t nq, const double* b, const double* s,
                      const double* q, const double* v, std::vector<double>& ext,
                      FastLayout& L) {
  // the kernel packs (cell index << 6 | selectors) into one int32
  if ((nb > 1 ? nb - 1 : 1) * (ns > 1 ? ns - 1 : 1) * (nq > 1 ? nq - 1 : 1) >= (int64_t(1) << 25))
    return RAPP_E_ARG;
  L = fast_layout(nb, ns, nq);
  if ((int64_t)L.total_doubles > (int64_t(1) << 30)) return RAPP_E_ARG;
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
    par[3] = uniform ? kModeUniform : kModeLut;
    if (uniform) L.modes |= 1 << a;
    par[4] = uniform ? h : 0.0;
    par[5] = uniform ? invh : 0.0;
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
      // [a[i], a[i+1]) with room to spare
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
  const int64_t cb = nb > 1 ? nb - 1 : 1, cs = ns > 1 ? ns - 1 : 1, cq = nq > 1 ? nq - 1 : 1;
  double* cells = ext.data() + L.o_cells;
  for (int64_t i = 0; i < cb; ++i)
    for (int64_t j = 0; j < cs; ++j)
      for (int64_t k = 0; k < cq; ++k) {
        double* c = cells + ((i * cs + j) * cq + k) * 8;
        for (int d = 0; d < 8; ++d) {  // corner d = (db << 2) | (ds << 1) | dq
          const int64_t ii = std::min(i + ((d >> 2) & 1), nb - 1);
          const int64_t jj = std::min(j + ((d >> 1) & 1), ns - 1);
          const int64_t kk = std::min(k + (d & 1), nq - 1);
          c[d] = v[(ii * ns + jj) * nq + kk];
        }
      }
  return RAPP_OK;
}
struct FastAxis {
  const uint32_t* lut;
  const double2* iv;
  int n;
  double a0, al, scale, h, invh;
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
  ax.n = int(p[6]);
  return ax;
}

// Rare cases of every mode: clamps, NaN.  Returns true if it produced the bracket.
__device__ __forceinline__ bool locate_edges(const FastAxis& ax, double x, int& c, int& s0,
                                             int& s1, double& t) {
  const int last = ax.n - 1;
  if (x <= ax.a0) { c = 0; s0 = 0; s1 = 0; t = 0.0; return true; }
  if (x >= ax.al) {
    c = last > 0 ? last - 1 : 0;
    s0 = s1 = last - c;
    t = 0.0;
    return true;
  }
  if (x != x) {  // NaN: the reference's search ends at (0, min(1, last)), t = NaN
    c = 0;
    s0 = 0;
    s1 = last > 0 ? 1 : 0;
    t = __ddiv_rn(__dsub_rn(x, ax.a0), __dsub_rn(ax.iv[s1].x, ax.a0));
    return true;
  }
  return false;
}

// Bracket of x as (cell c, corner selectors s0/s1, t): identical (lo, hi, t) to
// rapp::locate() for a strictly ascending axis, with lo = c + s0 and hi = c + s1.
template <int MODE>
__device__ __forceinline__ void locate_fast(const FastAxis& ax, double x, int& c, int& s0,
                                            int& s1, double& t) {
  if (!(x > ax.a0 && x < ax.al)) {  // clamps and NaN (all fail the test)
    locate_edges(ax, x, c, s0, s1, t);
    return;
  }
  const int last = ax.n - 1;  // a0 < x < a_last: n >= 2, lo in [0, n-2]
  if (MODE == kModeUniform) {
    // d = RN(x - a0) > 0 and u = d / h exactly.  If u is not an integer, i = trunc(u)
    // satisfies i*h < d < (i+1)*h, and since every a0 + k*h is exact and RN monotone,
    // a[i] < x < a[i+1]: the bracket is (i, i+1) and x is not a node.  Otherwise (u
    // integral: x within rounding of a node) fall back to exact comparisons.
    const double u = __dmul_rn(__dsub_rn(x, ax.a0), ax.invh);
    int i = int(u);
    i = i < last - 1 ? i : last - 1;
    double lo = fma(double(i), ax.h, ax.a0);  // exact: == a[i]
    if (double(i) == u) {
      if (lo > x) {
        --i;
        lo = fma(double(i), ax.h, ax.a0);
      } else if (i < last - 1) {
        const double nx = fma(double(i + 1), ax.h, ax.a0);
        if (nx <= x) {
          ++i;
          lo = nx;
        }
      }
      c = i;
      s0 = 0;
      if (lo == x) { s1 = 0; t = 0.0; return; }
    }
    c = i;
    s0 = 0;
    s1 = 1;
    t = __dmul_rn(__dsub_rn(x, lo), ax.invh);  // == RN((x - a[i]) / (a[i+1] - a[i]))
    return;
  }
  int k = int(__dmul_rn(__dsub_rn(x, ax.a0), ax.scale));
  k = k < kLut - 1 ? k : kLut - 1;
  const uint32_t e = ax.lut[k];
  int i = int(e & ~kExact);
  if (!(e & kExact)) {
    while (i < last - 1 && ax.iv[i + 1].x <= x) ++i;
    while (i > 0 && ax.iv[i].x > x) --i;
  }
  const double2 w = ax.iv[i];
  c = i;
  s0 = 0;
  if (w.x == x) { s1 = 0; t = 0.0; return; }
  s1 = 1;
  const double num = __dsub_rn(x, w.x);
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

__device__ __forceinline__ double shfl_d(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

#ifndef RAPP_STREAM_ILP
#define RAPP_STREAM_ILP 1
#endif
#ifndef RAPP_STREAM_MINB
#define RAPP_STREAM_MINB 2
#endif
#ifndef RAPP_STREAM_CONSUMERS
#define RAPP_STREAM_CONSUMERS 16
#endif
constexpr int kFastIlp = RAPP_STREAM_ILP;         // rows per lane per stage
constexpr int kConsumers = RAPP_STREAM_CONSUMERS;  // consumer warps per CTA
constexpr int kProducer = kConsumers;              // warp index of the TMA producer
constexpr int kFastThreads = (kConsumers + 1) * 32;
constexpr int kTile = kConsumers * 32 * kFastIlp;  // rows per TMA stage
constexpr int kStages = 4;
constexpr int kInterior = 0x2A; // selector bits of an interior query on every axis

// Interpolates ILP rows per lane (row index base + k*32 + lane, coordinates in x).
// Lane pairs cooperate on their two queries, each lane loading one batch row of each cell
// with one 256-bit load (see below).  All 2*ILP loads of a lane are issued before any of
// them is consumed, so their L2 latencies overlap.
template <int ILP, int MB, int MS, int MQ, bool CELLS_SMEM>
__device__ __forceinline__ void interp_rows(const FastAxis& ab, const FastAxis& as,
                                            const FastAxis& aq, const double* cells, int CS,
                                            int CQ, double (&x)[ILP][3], int64_t base,
                                            int64_t n, double* __restrict__ out,
                                            double* __restrict__ rps) {
  const int lane = threadIdx.x & 31;
  const int half = lane & 1;
  int cs[ILP];
  double tb[ILP], ts[ILP], tq[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) {
    int ib, bs0, bs1, js, ss0, ss1, kq, qs0, qs1;
    locate_fast<MB>(ab, x[k][0], ib, bs0, bs1, tb[k]);
    locate_fast<MS>(as, x[k][1], js, ss0, ss1, ts[k]);
    locate_fast<MQ>(aq, x[k][2], kq, qs0, qs1, tq[k]);
    // cell index (< 2^25, checked at upload) and the 6 selector bits in one word
    cs[k] = (((ib * CS + js) * CQ + kq) << 6) | bs0 | (bs1 << 1) | (ss0 << 2) | (ss1 << 3) |
            (qs0 << 4) | (qs1 << 5);
  }
  // Lane h of a pair evaluates batch row h (i0 for h=0, i1 for h=1) of BOTH queries of
  // the pair: its own (o) and its partner's (p).  One exchange then gives each lane the
  // other row of its own query for the batch lerp.
  // Load r of a pair fetches the cell of the pair's query r (owned by lane 2p+r) — both
  // lanes hit the same 64-byte cell in the same instruction, so a warp-wide load touches
  // 16 lines, not 32.  Lane h keeps row h of each cell.
  int c_r[ILP][2];
  double tq_r[ILP][2], ts_r[ILP][2], v[ILP][2][4];
#pragma unroll
  for (int k = 0; k < ILP; ++k) {
    const int csp = __shfl_xor_sync(0xffffffffu, cs[k], 1);
    const double tqp = __shfl_xor_sync(0xffffffffu, tq[k], 1);
    const double tsp = __shfl_xor_sync(0xffffffffu, ts[k], 1);
    c_r[k][0] = half ? csp : cs[k];
    c_r[k][1] = half ? cs[k] : csp;
    tq_r[k][0] = half ? tqp : tq[k];
    tq_r[k][1] = half ? tq[k] : tqp;
    ts_r[k][0] = half ? tsp : ts[k];
    ts_r[k][1] = half ? ts[k] : tsp;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int c = c_r[k][r];
      const int db = half ? (c >> 1) & 1 : c & 1;  // which corner row is "row h"
      load_row(cells + int64_t(c >> 6) * 8 + db * 4, CELLS_SMEM, v[k][r][0], v[k][r][1],
               v[k][r][2], v[k][r][3]);
    }
  }
#pragma unroll
  for (int k = 0; k < ILP; ++k) {
    // row value c_h = lerp(lerp(v[j0,k0], v[j0,k1], tq), lerp(v[j1,k0], v[j1,k1], tq), ts)
    auto row = [&](int sel, double (&v)[4], double t_q, double t_s) -> double {
      double a0 = v[0], a1 = v[1], b0 = v[2], b1 = v[3];
      if ((sel & 63) != kInterior) {  // clamp / node hit: pick the corners the reference reads
        const int s0 = (sel >> 2) & 1, s1 = (sel >> 3) & 1;
        const int q0 = (sel >> 4) & 1, q1 = (sel >> 5) & 1;
        const double r0a = s0 ? b0 : a0, r0b = s0 ? b1 : a1;  // ds = s0 row (dq = 0, 1)
        const double r1a = s1 ? b0 : a0, r1b = s1 ? b1 : a1;  // ds = s1 row
        a0 = q0 ? r0b : r0a;
        a1 = q1 ? r0b : r0a;
        b0 = q0 ? r1b : r1a;
        b1 = q1 ? r1b : r1a;
      }
      return lerp_rn(lerp_rn(a0, a1, t_q), lerp_rn(b0, b1, t_q), t_s);
    };
    const double c0r = row(c_r[k][0], v[k][0], tq_r[k][0], ts_r[k][0]);
    const double c1r = row(c_r[k][1], v[k][1], tq_r[k][1], ts_r[k][1]);
    const double co = half ? c1r : c0r;  // row h of my query
    const double cp = half ? c0r : c1r;  // row h of my partner's query
    const double other = __shfl_xor_sync(0xffffffffu, cp, 1);  // row 1-h of my query
    const double lat = half ? lerp_rn(other, co, tb[k]) : lerp_rn(co, other, tb[k]);
    const int64_t i = base + k * 32 + lane;
    if (i < n) {
      __stcs(out + i, lat);
      if (rps != nullptr) __stcs(rps + i, throughput(x[k][0], lat));
    }
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
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(sbar), "r"(parity)
        : "memory");
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
// kConsumers warps each take 32*ILP rows of a stage, release it as soon as the rows are
// in registers, and interpolate.  Rows past the last full tile (or everything, when coords
// is not 16-byte aligned) use direct loads.
template <int MB, int MS, int MQ, bool CELLS_SMEM>
__global__ void __launch_bounds__(kFastThreads, RAPP_STREAM_MINB)
    k_interp_fast(const TableDesc td, const double* __restrict__ pool,
                  const double* __restrict__ coords, int64_t n, int64_t n_tiles,
                  double* __restrict__ out, double* __restrict__ rps) {
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
  const int CS = td.ns > 1 ? td.ns - 1 : 1, CQ = td.nq > 1 ? td.nq - 1 : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- TMA ring over full tiles: warp kWarps-1 produces, the others consume ----
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
  {
    int64_t t = blockIdx.x;
    for (int j = 0; t < n_tiles; ++j, t += gridDim.x) {
      const int s = j % kStages;
      mbar_wait(&full[s], (j / kStages) & 1);
      const double* tile = buf0 + s * 3 * kTile;
      const int r0 = warp * 32 * kFastIlp;
      double x[kFastIlp][3];
#pragma unroll
      for (int k = 0; k < kFastIlp; ++k) {
        const double* row = tile + 3 * (r0 + k * 32 + lane);
        x[k][0] = row[0];
        x[k][1] = row[1];
        x[k][2] = row[2];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this warp's rows are in registers
      interp_rows<kFastIlp, MB, MS, MQ, CELLS_SMEM>(ab, as, aq, cells, CS, CQ, x,
                                                    t * kTile + r0, n, out, rps);
    }
  }

  // ---- remainder rows: direct loads, warp-uniform grid-stride ----
  const int64_t rem0 = n_tiles * kTile;
  const int64_t per_warp = 32 * kFastIlp;
  const int64_t warps_total = int64_t(gridDim.x) * kConsumers;
  for (int64_t wb = rem0 + (int64_t(blockIdx.x) * kConsumers + warp) * per_warp; wb < n;
       wb += warps_total * per_warp) {
    double x[kFastIlp][3];
#pragma unroll
    for (int k = 0; k < kFastIlp; ++k) {
      const int64_t i = wb + k * 32 + lane;
      if (i < n) {
        x[k][0] = __ldcs(coords + 3 * i);
        x[k][1] = __ldcs(coords + 3 * i + 1);
        x[k][2] = __ldcs(coords + 3 * i + 2);
      } else {
        x[k][0] = ab.a0;  // harmless in-range filler
        x[k][1] = as.a0;
        x[k][2] = aq.a0;
      }
    }
    interp_rows<kFastIlp, MB, MS, MQ, CELLS_SMEM>(ab, as, aq, cells, CS, CQ, x, wb, n, out, rps);
  }
}

constexpr int64_t kFastCellsSmem = 96 * 1024;

template <int MB, int MS, int MQ>
static void launch_modes(bool cells_smem, unsigned blocks, size_t smem, cudaStream_t st,
                         const TableDesc& td, const double* pool, const double* coords,
                         int64_t n, int64_t n_tiles, double* out, double* rps) {
  if (cells_smem) {
    auto k = k_interp_fast<MB, MS, MQ, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    k<<<blocks, kFastThreads, smem, st>>>(td, pool, coords, n, n_tiles, out, rps);
  } else {
    auto k = k_interp_fast<MB, MS, MQ, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    k<<<blocks, kFastThreads, smem, st>>>(td, pool, coords, n, n_tiles, out, rps);
  }
}

int launch_interp_fast(rapp_ctx* ctx, const TableDesc& td, const double* d_coords, int64_t n,
                       double* d_out, double* d_rps, cudaStream_t st) {
  const int64_t cell_bytes = int64_t(td.x_total - td.x_small) * 8;
  const int64_t small_bytes = int64_t(td.x_small) * 8;
  const bool cells_smem = cell_bytes + small_bytes <= kFastCellsSmem;
  const int64_t ext_bytes = cells_smem ? small_bytes + cell_bytes : small_bytes;
  const size_t smem = (size_t)(((ext_bytes + 127) & ~int64_t(127)) + kStages * 3 * kTile * 8);
  if (smem > 220 * 1024) {
    set_error("fast-path shared-memory footprint %zu too large", smem);
    return RAPP_E_ARG;
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(d_coords) & 15) == 0;
  const int64_t n_tiles = aligned ? n / kTile : 0;
  int64_t blocks = n_tiles > 0 ? n_tiles : (n + kTile - 1) / kTile;
  const int64_t per_sm =
      std::max<int64_t>(1, std::min<int64_t>(RAPP_STREAM_MINB, (220 * 1024) / (int64_t)(smem + 1024)));
  const int64_t cap = int64_t(ctx->sm_count) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const unsigned nb = (unsigned)blocks;
  const double* pool = ctx->d_pool;
  switch (td.modes & 7) {  // bit 0: batch axis uniform, bit 1: sm, bit 2: quota
    case 0: launch_modes<0, 0, 0>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps); break;
    case 1: launch_modes<1, 0, 0>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps); break;
    case 2: launch_modes<0, 1, 0>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps); break;
    case 3: launch_modes<1, 1, 0>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps); break;
    case 4: launch_modes<0, 0, 1>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps); break;
    case 5: launch_modes<1, 0, 1>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps); break;
    case 6: launch_modes<0, 1, 1>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps); break;
    default: launch_modes<1, 1, 1>(cells_smem, nb, smem, st, td, pool, d_coords, n, n_tiles, d_out, d_rps); break;
  }
  RAPP_LAUNCHED();
  return RAPP_OK;
}

}  // namespace rapp
