// K3: most_efficient_config batched over functions — fused lattice evaluate ->
// feasibility mask -> lexicographic argmin (hs/perf.py:104-145).
//
// Per function f with table T, batch lattice B_f (the `_batch_lattice` rule applied by
// the caller), table sm axis S and quota lattice Q = range(step, 101, step):
//   meet     = argmin (s*q, s, q, b) over {rps(b,s,q) >= target}
//   fallback = argmin (-rps, s*q, s, q, b) over the whole lattice        (perf.py:123-138)
//
// Exactness recipe (all 0-ulp against the reference):
//  * latency of every lattice point is computed with the reference's nested lerps in the
//    reference's order (rapp_device.cuh).  The lerps of one table row (batch index i) at a
//    given (s,q) do not depend on b, so a thread evaluating one (s,q) pair computes each
//    needed row value once and reuses it for every b bracketed by that row — the same
//    doubles the reference computes, just not recomputed (c0 = row(i0), c1 = row(i1)).
//  * `rps >= target` is decided as `lat <= threshold(b, target)` (rapp_device.cuh), which
//    is exactly equivalent for positive latencies because throughput is a composition of
//    two correctly rounded (monotone) divisions; non-positive / NaN latencies evaluate the
//    division explicitly.
//  * the fallback max-rps point is meet(rps_max): max rps for batch b is
//    throughput(b, min latency over (s,q)), and the min (s*q,s,q,b) point among
//    {rps >= rps_max} = {rps == rps_max} is exactly the fallback key's argmin.
//  * keys are packed into one uint64 in lexicographic order:
//        cost(32) | s_index(12) | q(8) | b_index(12)
//    (s axis strictly ascending -> index order == value order; B_f sorted -> same), so
//    the argmin is an order-independent min-reduction: warp shuffles -> shared memory ->
//    one atomicMin per CTA into the per-function slot.
#include <cmath>
#include <cstring>
#include <memory>
#include <type_traits>

#include "rapp_device.cuh"
#include "rapp_internal.h"

#ifndef RAPP_K3_UNROLL
#define RAPP_K3_UNROLL 8
#endif

namespace rapp {

constexpr int kK3Unroll = RAPP_K3_UNROLL;  // unroll of the per-batch-entry loop
#ifndef RAPP_K3_PAIRS
#define RAPP_K3_PAIRS 3
#endif
constexpr int kK3Pairs = RAPP_K3_PAIRS;  // (s, q) pairs per thread in the meet pass
#ifndef RAPP_K3_RUN_UNROLL
#define RAPP_K3_RUN_UNROLL 1
#endif
constexpr int kK3RunUnroll = RAPP_K3_RUN_UNROLL;  // unroll of the per-run loop

struct FnDesc {
  int32_t table;
  int32_t nB;
  int64_t boff;  // first entry of this function's batch lattice in d_blist / d_thr
};

constexpr int kSearchThreads = 256;
constexpr uint64_t kNoKey = ~0ull;
constexpr int64_t kSearchSmemTable = 64 * 1024;  // table bytes staged in shared memory

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// One warp per function: feasibility thresholds per batch-lattice entry, key reset.
// Opt-in latency SLO (slo != nullptr, slo[f] > 0 or NaN = none): a point is feasible iff
// rps >= target AND lat <= slo[f].  Both are upper bounds on the latency (the first is
// exactly lat <= threshold for positive latencies), so the mask is one threshold,
// min(threshold, slo[f]); latency 0 (rps = inf) satisfies any positive SLO, and the
// fallback pass (k_mec_fallback) recomputes its thresholds without the SLO.
__global__ void k_mec_prepare(const FnDesc* __restrict__ fns, const double* __restrict__ blist,
                              const double* __restrict__ targets, int64_t fn_begin,
                              int64_t fn_end, double* __restrict__ thr,
                              unsigned long long* __restrict__ minlat,
                              unsigned long long* __restrict__ keys,
                              const double* __restrict__ slo) {
  pdl_trigger();
  const int64_t f = fn_begin + (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (f >= fn_end) return;
  const FnDesc fd = fns[f];
  const double target = targets[f];
  const double cap = slo != nullptr ? slo[f] : __longlong_as_double(0x7FF0000000000000ll);
  for (int bi = lane; bi < fd.nB; bi += 32) {
    const double th = feasibility_threshold(blist[fd.boff + bi], target);
    thr[fd.boff + bi] = cap < th ? cap : th;  // NaN cap: no SLO
    minlat[fd.boff + bi] = 0x7FF0000000000000ull;  // +inf
  }
  if (lane == 0) keys[f] = kNoKey;
}

// Fallback targets: rps_max = max_b throughput(b, min latency of b); thresholds for it.
__global__ void k_mec_fallback(const FnDesc* __restrict__ fns, const double* __restrict__ blist,
                               int64_t fn_begin, int64_t fn_end,
                               const unsigned long long* __restrict__ keys,
                               const unsigned long long* __restrict__ minlat,
                               double* __restrict__ thr, double* __restrict__ target2,
                               int32_t* __restrict__ fallback) {
  pdl_trigger();
  pdl_wait();
  const int64_t f = fn_begin + (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (f >= fn_end) return;
  const bool unresolved = keys[f] == kNoKey;
  if (lane == 0) fallback[f] = unresolved ? 1 : 0;
  if (!unresolved) return;
  const FnDesc fd = fns[f];
  double best = -1.0;  // rps >= 0 for positive latencies
  for (int bi = lane; bi < fd.nB; bi += 32) {
    const double r =
        throughput(blist[fd.boff + bi], __longlong_as_double((long long)minlat[fd.boff + bi]));
    best = r > best ? r : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, best, o);
    best = w > best ? w : best;
  }
  for (int bi = lane; bi < fd.nB; bi += 32)
    thr[fd.boff + bi] = feasibility_threshold(blist[fd.boff + bi], best);
  if (lane == 0) target2[f] = best;
}

// The fused lattice pass.  MINLAT=false: meet search (feasibility mask + packed-key
// argmin).  MINLAT=true: per-batch minimum latency for functions with no feasible point.
// GATE: only functions without a feasible point take part (fallback passes): the MINLAT
// pass reads keys[] (not written by it), the second meet pass reads the fallback flags
// (keys[] is being lowered by sibling CTAs of the same function during that pass).
template <bool SMEM, bool MINLAT, bool GATE>
__global__ void __launch_bounds__(kSearchThreads)
    k_mec_lattice(const TableDesc* __restrict__ tds, const double* __restrict__ pool,
                  const FnDesc* __restrict__ fns, const double* __restrict__ blist,
                  const double* __restrict__ thr_g, const double* __restrict__ targets,
                  int64_t fn_begin, int32_t chunks, int32_t step, int32_t nQ,
                  unsigned long long* __restrict__ keys,
                  unsigned long long* __restrict__ minlat_g,
                  const int32_t* __restrict__ fallback) {
  extern __shared__ __align__(16) double smem[];
  __shared__ uint64_t bar;
  __shared__ unsigned long long s_red[kSearchThreads / 32];
  pdl_trigger();
  if (GATE) pdl_wait();  // the gate reads the previous passes' keys / fallback flags
  const int64_t f = fn_begin + blockIdx.x / chunks;
  const int chunk = blockIdx.x % chunks;
  if (GATE && (MINLAT ? keys[f] != kNoKey : fallback[f] == 0)) return;
  const FnDesc fd = fns[f];
  const TableDesc td = tds[fd.table];
  const int nb = td.nb, ns = td.ns, nq = td.nq, nB = fd.nB;

  // shared layout: [table segment (SMEM only)] [S: ts | j0 j1] [Q: tq | k0 k1] [B: tb thr b]
  //                [B: i0 i1] [B: minlat]
  double* p = smem;
  const double* seg = pool + td.off;
  if (SMEM) {
    bulk_load_table(p, seg, uint32_t(td.seg_doubles) * 8u, &bar);
    seg = p;
    p += td.seg_doubles;
  }
  const double* __restrict__ ba = seg + td.ob;
  const double* __restrict__ sa = seg + td.os;
  const double* __restrict__ qa = seg + td.oq;
  const double* __restrict__ v = seg + td.ov;
  double* sTs = p;                 p += ns;
  int2* sJ = (int2*)p;             p += ns;
  double* sTq = p;                 p += nQ;
  int2* sK = (int2*)p;             p += nQ;
  double* sTb = p;                 p += nB;
  double* sThr = p;                p += nB;
  double* sB = p;                  p += nB;
  int2* sI = (int2*)p;             p += nB;
  unsigned long long* sMin = (unsigned long long*)p;  p += nB;
  p += (p - smem) & 1;                           // 16-byte alignment for the vectors below
  double2* sTT = (double2*)p;      p += 2 * nB;  // (tb, threshold) per batch entry
  int4* sSeg = (int4*)p;           p += 2 * nB;  // runs of entries sharing a row bracket
  int4* sLo = (int4*)p;            p += 2 * nB;  // runs of entries sharing a lower row
  uint32_t* sSv = (uint32_t*)p;    p += (ns + 1) / 2;  // sm values as integers (< 2^24)
  __shared__ int s_nseg, s_nlo;

  // per-axis brackets, once per CTA (locate semantics, _grid_cy.pyx:9-33)
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    int lo, hi;
    double t;
    locate(sa, ns, sa[i], lo, hi, t);  // the lattice's sm values are the table's own sms
    sTs[i] = t;
    sJ[i] = make_int2(lo, hi);
    sSv[i] = uint32_t(sa[i]);  // integral and < 2^24 (sm_keyable, checked at plan creation)
  }
  for (int i = threadIdx.x; i < nQ; i += blockDim.x) {
    int lo, hi;
    double t;
    locate(qa, nq, double((i + 1) * step), lo, hi, t);
    sTq[i] = t;
    sK[i] = make_int2(lo, hi);
  }
  if (!GATE) pdl_wait();  // thresholds and key reset of k_mec_prepare (table staging and
                         // the sm / quota brackets above overlap it)
  for (int i = threadIdx.x; i < nB; i += blockDim.x) {
    int lo, hi;
    double t;
    const double b = blist[fd.boff + i];
    locate(ba, nb, b, lo, hi, t);
    sTb[i] = t;
    sI[i] = make_int2(lo, hi);
    sB[i] = b;
    sThr[i] = thr_g[fd.boff + i];
    sTT[i] = make_double2(t, sThr[i]);
    if (MINLAT) sMin[i] = 0x7FF0000000000000ull;
  }
  __syncthreads();
  // batch entries are sorted, so entries bracketed by the same table rows (i0, i1) are
  // consecutive: one segment per bracket, its two row values computed once per (s, q)
  // (warp 0: run heads by ballot, positions by popcount prefix)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int n = 0, m = 0;
    for (int base = 0; base < nB; base += 32) {
      const int i = base + lane;
      const bool in = i < nB;
      const int2 cur = in ? sI[i] : make_int2(0, 0);
      const int2 prv = in && i > 0 ? sI[i - 1] : make_int2(-1, -1);
      const bool hs = in && (cur.x != prv.x || cur.y != prv.y);
      const bool hl = in && cur.x != prv.x;
      const unsigned ms = __ballot_sync(0xffffffffu, hs), ml = __ballot_sync(0xffffffffu, hl);
      const unsigned below = (1u << lane) - 1u;
      if (hs) sSeg[n + __popc(ms & below)] = make_int4(cur.x, cur.y, i, 0);
      if (hl) sLo[m + __popc(ml & below)] = make_int4(cur.x, i, 0, 0);
      n += __popc(ms);
      m += __popc(ml);
    }
    __syncwarp();
    // run ends: the next run's start (or nB)
    for (int k = lane; k < n; k += 32) sSeg[k].w = k + 1 < n ? sSeg[k + 1].z : nB;
    for (int k = lane; k < m; k += 32) sLo[k].z = k + 1 < m ? sLo[k + 1].y : nB;
    if (lane == 0) {
      s_nseg = n;
      s_nlo = m;
    }
  }
  __syncthreads();
  const int nseg = s_nseg, nlo = s_nlo;
  const bool pos_table = td.fast != 0;  // fast-path tables are finite and positive

  const double target = targets[f];
  const int pairs = ns * nQ;
  const int per = (pairs + chunks - 1) / chunks;
  const int p0 = chunk * per, p1 = min(pairs, p0 + per);
  unsigned long long best = kNoKey;
  const int64_t row_stride = int64_t(ns) * nq;

  auto record = [&](int si, int qi, int found) {
    if (found < (1 << 30)) {
      const uint32_t q = uint32_t((qi + 1) * step);
      const uint32_t cost = sSv[si] * q;  // < 2^24 * 100: exact in 32 bits
      const unsigned long long k = (uint64_t(cost) << 32) |
                                   ((uint32_t(si) << 20) | (q << 12) | uint32_t(found));
      best = k < best ? k : best;
    }
  };

  // Any table, any pair: the reference's row values (two-entry cache, rows visited in
  // ascending order) and the batch segments.  Returns the first feasible batch entry.
  auto generic_pair = [&](int si, int qi) -> int {
    const int2 jj = sJ[si], kk = sK[qi];
    const double ts = sTs[si], tq = sTq[qi];
    const int o00 = jj.x * nq + kk.x, o01 = jj.x * nq + kk.y;
    const int o10 = jj.y * nq + kk.x, o11 = jj.y * nq + kk.y;
    int ra = -1, rb = -1;
    double ca = 0.0, cb = 0.0;
    auto row = [&](int i) -> double {
      if (i == rb) return cb;
      if (i == ra) return ca;
      const double* r = v + int64_t(i) * row_stride;
      const double c_j0 = lerp_rn(r[o00], r[o01], tq);
      const double c_j1 = lerp_rn(r[o10], r[o11], tq);
      const double c = lerp_rn(c_j0, c_j1, ts);
      ra = rb;
      ca = cb;
      rb = i;
      cb = c;
      return c;
    };
    int found = 1 << 30;  // first feasible batch entry (entries ascend with b)
    for (int sg = 0; sg < nseg; ++sg) {
      const int4 S = sSeg[sg];
      const double c0 = row(S.x);
      const double c1 = S.y == S.x ? c0 : row(S.y);
      if (MINLAT) {
        for (int bi = S.z; bi < S.w; ++bi) {
          const double lat = lerp_rn(c0, c1, sTT[bi].x);
          if (lat >= 0.0) atomicMin(&sMin[bi], (unsigned long long)__double_as_longlong(lat));
        }
      } else if (pos_table) {
        // finite positive grid: `rps >= target` is exactly `lat <= threshold`
        for (int bi = S.z; bi < S.w; ++bi) {
          const double2 tt = sTT[bi];
          const double lat = lerp_rn(c0, c1, tt.x);  // the reference's final batch lerp
          found = lat <= tt.y && bi < found ? bi : found;
        }
      } else {
        for (int bi = S.z; bi < S.w; ++bi) {
          const double2 tt = sTT[bi];
          const double lat = lerp_rn(c0, c1, tt.x);
          const bool ok = lat > 0.0 ? (lat <= tt.y) : (throughput(sB[bi], lat) >= target);
          found = ok && bi < found ? bi : found;
        }
      }
    }
    return found;
  };

  const int bd = int(blockDim.x);
  if (!MINLAT && pos_table) {
    // Meet pass over a finite positive grid (checked at upload): every interpolated
    // latency is > 0, so `rps >= target` is exactly `lat <= threshold` — no division.
    // Exact shortcuts of the reference's arithmetic for such grids (x + (y - x) * 0 == x
    // for finite positive x and finite y):
    //  * the lattice's sm values are the table's own nodes (j0 == j1, ts == 0), so a row
    //    value is its quota lerp c_j0 — the same double the reference's c0 = c_j0 +
    //    (c_j1 - c_j0) * 0 yields;
    //  * a node hit or clamp (lo == hi, tb == 0) gives row(lo), which is also
    //    row(lo) + (row(lo + 1) - row(lo)) * 0, so it joins the run of entries with lower
    //    row lo; entries with lo == last use d = 0.
    // Runs and entries are walked in descending order (the last feasible entry seen is the
    // first in lattice order); each run needs one new row value.  kK3Pairs (s, q) pairs per
    // thread share the run bookkeeping and every (tb, threshold) load.
    const int last = nb - 1;
    // pair index -> (sm index, quota index) without an integer division: the float quotient
    // is off by at most one for pairs < 2^24, and the remainder test corrects it
    const float inv_nq = 1.0f / float(nQ);
    auto split = [&](int pu, int& s, int& q) {
      int a = int((float(pu) + 0.5f) * inv_nq);
      int r = pu - a * nQ;
      if (r < 0) { --a; r += nQ; } else if (r >= nQ) { ++a; r -= nQ; }
      s = a;
      q = r;
    };
    // table rows: shared-memory tables are read with 32-bit shared addresses (one LDS per
    // corner, the row offset added once per run), global ones through pointers
    using RowRef = typename std::conditional<SMEM, uint32_t, const double*>::type;
    const uint32_t v_sh = SMEM ? (uint32_t)__cvta_generic_to_shared(v) : 0u;
    const uint32_t row_bytes = uint32_t(row_stride) * 8u;
    auto corner = [&](RowRef r, int64_t row) -> double {
      if constexpr (SMEM) {
        double x;
        asm("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(r + uint32_t(row) * row_bytes));
        return x;
      } else {
        return r[row * row_stride];
      }
    };
    // pairs pa, pa + bd, ..., pa + (NP - 1) * bd (all < p1)
    auto fast = [&](int pa, auto np_tag) {
      constexpr int NP = decltype(np_tag)::value;
      int si[NP], qi[NP];
      bool node = true;
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        split(pa + u * bd, si[u], qi[u]);
        const int2 j = sJ[si[u]];
        node = node && j.x == j.y;
      }
      if (!node) {  // not produced by a lattice over table sms
#pragma unroll
        for (int u = 0; u < NP; ++u) record(si[u], qi[u], generic_pair(si[u], qi[u]));
        return;
      }
      RowRef r0[NP], r1[NP];
      double tq[NP], cu[NP], c0[NP], d[NP];
      int fnd[NP];
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int js = sJ[si[u]].x;
        const int2 k = sK[qi[u]];
        if constexpr (SMEM) {
          r0[u] = v_sh + uint32_t(js * nq + k.x) * 8u;
          r1[u] = v_sh + uint32_t(js * nq + k.y) * 8u;
        } else {
          r0[u] = v + (js * nq + k.x);
          r1[u] = v + (js * nq + k.y);
        }
        tq[u] = sTq[qi[u]];
        cu[u] = 0.0;
        fnd[u] = 1 << 30;
      }
      int up = -2;
#pragma unroll (kK3RunUnroll)
      for (int sg = nlo - 1; sg >= 0; --sg) {
        const int4 S = sLo[sg];
        // one branch per run (not per pair): the upper row is the previous run's lower row
        // (runs of consecutive rows, the usual case), the top row (no upper), or fresh
        if (S.x + 1 == up) {
#pragma unroll
          for (int u = 0; u < NP; ++u) {
            c0[u] = lerp_rn(corner(r0[u], S.x), corner(r1[u], S.x), tq[u]);
            d[u] = __dsub_rn(cu[u], c0[u]);
            cu[u] = c0[u];
          }
        } else if (S.x == last) {
#pragma unroll
          for (int u = 0; u < NP; ++u) {
            c0[u] = lerp_rn(corner(r0[u], S.x), corner(r1[u], S.x), tq[u]);
            d[u] = 0.0;
            cu[u] = c0[u];
          }
        } else {
#pragma unroll
          for (int u = 0; u < NP; ++u) {
            c0[u] = lerp_rn(corner(r0[u], S.x), corner(r1[u], S.x), tq[u]);
            const double c1 = lerp_rn(corner(r0[u], S.x + 1), corner(r1[u], S.x + 1), tq[u]);
            d[u] = __dsub_rn(c1, c0[u]);
            cu[u] = c0[u];
          }
        }
        up = S.x;
#pragma unroll (kK3Unroll)
        for (int bi = S.z - 1; bi >= S.y; --bi) {
          const double2 tt = sTT[bi];
#pragma unroll
          for (int u = 0; u < NP; ++u) {
            const double lat = __dadd_rn(c0[u], __dmul_rn(d[u], tt.x));
            fnd[u] = lat <= tt.y ? bi : fnd[u];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < NP; ++u) record(si[u], qi[u], fnd[u]);
    };
    int pa = p0 + int(threadIdx.x);
    for (; pa + (kK3Pairs - 1) * bd < p1; pa += kK3Pairs * bd)
      fast(pa, std::integral_constant<int, kK3Pairs>());
    for (; pa < p1; pa += bd) fast(pa, std::integral_constant<int, 1>());
  } else {
    for (int pr = p0 + int(threadIdx.x); pr < p1; pr += bd) {
      const int si = pr / nQ, qi = pr - si * nQ;
      const int found = generic_pair(si, qi);
      if (!MINLAT) record(si, qi, found);
    }
  }

  if (MINLAT) {
    __syncthreads();
    for (int i = threadIdx.x; i < nB; i += blockDim.x)
      if (sMin[i] != 0x7FF0000000000000ull) atomicMin(&minlat_g[fd.boff + i], sMin[i]);
    return;
  }
  best = warp_min_u64(best);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long k = threadIdx.x < (kSearchThreads / 32) ? s_red[threadIdx.x] : kNoKey;
    k = warp_min_u64(k);
    if (threadIdx.x == 0 && k != kNoKey) atomicMin(&keys[f], k);
  }
}

// key -> (b, s, q)
__global__ void k_mec_decode(const TableDesc* __restrict__ tds, const double* __restrict__ pool,
                             const FnDesc* __restrict__ fns, const double* __restrict__ blist,
                             int64_t fn_begin, int64_t fn_end,
                             const unsigned long long* __restrict__ keys,
                             int32_t* __restrict__ out_bsq, uint64_t* __restrict__ out_key) {
  pdl_trigger();
  pdl_wait();
  const int64_t f = fn_begin + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= fn_end) return;
  const FnDesc fd = fns[f];
  const TableDesc td = tds[fd.table];
  const unsigned long long k = keys[f];
  int32_t b = -1, s = -1, q = -1;
  if (k != kNoKey) {
    b = int32_t(blist[fd.boff + (k & 0xFFF)]);
    q = int32_t((k >> 12) & 0xFF);
    s = int32_t(pool[td.off + td.os + ((k >> 20) & 0xFFF)]);
  }
  out_bsq[3 * (f - fn_begin)] = b;
  out_bsq[3 * (f - fn_begin) + 1] = s;
  out_bsq[3 * (f - fn_begin) + 2] = q;
  if (out_key) out_key[f - fn_begin] = k;
}

}  // namespace rapp

using namespace rapp;

struct rapp_mec_plan {
  rapp_ctx* ctx = nullptr;
  int64_t nfn = 0, total_b = 0, points = 0;
  int32_t step = 10, nQ = 10;
  int max_pairs = 0;
  bool smem_table = true;
  size_t smem_bytes = 0;
  size_t smem_brk_bytes = 0;  // the bracket arrays alone (table read from global memory)
  FnDesc* d_fn = nullptr;
  double* d_blist = nullptr;
  double* d_thr = nullptr;
  unsigned long long* d_minlat = nullptr;
  unsigned long long* d_key = nullptr;
  double* d_slo = nullptr;  // opt-in per-function latency SLO (rapp_mec_plan_set_slo)
  double* d_target2 = nullptr;
  int32_t* d_fb = nullptr;
  // optional per-launch timing of the meet pass (bench.py's roofline): event pairs
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // 2 per timed launch
  size_t ev_used = 0;
  // host-buffer runs (rapp_mec_plan_run): pinned [targets nfn | bsq 3*nfn int32] staging
  // mirrored on the device, one stream — allocated on the first host run, reused after
  cudaStream_t stream = nullptr;
  uint8_t* h_stage = nullptr;
  uint8_t* d_stage = nullptr;
};

#ifndef RAPP_K3_GATED_GLOBAL
#define RAPP_K3_GATED_GLOBAL 1
#endif

namespace rapp {

template <bool SMEM, bool MINLAT, bool GATE>
static int launch_lattice(rapp_mec_plan* pl, const double* targets, int64_t f0, int64_t nf,
                          int chunks, cudaStream_t st) {
  auto kern = k_mec_lattice<SMEM, MINLAT, GATE>;
  const size_t smem = SMEM ? pl->smem_bytes : pl->smem_brk_bytes;
  RAPP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(smem, 1)));
  rapp_ctx* c = pl->ctx;
  RAPP_CUDA(launch_pdl(kern, dim3((unsigned)(nf * chunks)), dim3(kSearchThreads),
                       smem, st, c->d_desc, c->d_pool, pl->d_fn, pl->d_blist, pl->d_thr,
                       targets, f0, chunks, pl->step, pl->nQ, pl->d_key, pl->d_minlat,
                       pl->d_fb));
  RAPP_LAUNCHED();
  return RAPP_OK;
}

static int run_plan(rapp_mec_plan* pl, const double* d_targets, int64_t f0, int64_t f1,
                    int32_t* d_out_bsq, uint64_t* d_out_key, cudaStream_t st) {
  const int64_t nf = f1 - f0;
  if (nf <= 0) return RAPP_OK;
  rapp_ctx* c = pl->ctx;
  const int wpb = 8;  // warps per block for the per-function helpers
  const unsigned hblocks = (unsigned)((nf + wpb - 1) / wpb);
  k_mec_prepare<<<hblocks, 32 * wpb, 0, st>>>(pl->d_fn, pl->d_blist, d_targets, f0, f1,
                                              pl->d_thr, pl->d_minlat, pl->d_key, pl->d_slo);
  RAPP_LAUNCHED();
  // enough CTAs to fill the machine even for a handful of functions
#ifndef RAPP_K3_CTAS_PER_SM
#define RAPP_K3_CTAS_PER_SM 4  // 32 / 64 (2 / 4 CTAs per config-5 function): 3% / 11% slower
#endif
  int chunks = (int)((int64_t(RAPP_K3_CTAS_PER_SM) * c->sm_count + nf - 1) / nf);
  const int max_chunks = (pl->max_pairs + kSearchThreads - 1) / kSearchThreads;
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  int rc;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (pl->timing) {
    if (pl->ev_used + 2 > pl->ev.size()) {
      pl->ev.resize(pl->ev.size() + 64, nullptr);
      for (size_t i = pl->ev_used; i < pl->ev.size(); ++i) RAPP_CUDA(cudaEventCreate(&pl->ev[i]));
    }
    t0 = pl->ev[pl->ev_used++];
    t1 = pl->ev[pl->ev_used++];
    RAPP_CUDA(cudaEventRecord(t0, st));
  }
  if (pl->smem_table) {
    if ((rc = launch_lattice<true, false, false>(pl, d_targets, f0, nf, chunks, st))) return rc;
  } else {
    if ((rc = launch_lattice<false, false, false>(pl, d_targets, f0, nf, chunks, st))) return rc;
  }
  if (t1) RAPP_CUDA(cudaEventRecord(t1, st));
  // the gated passes (functions without a feasible point; usually none) read the table from
  // global memory: their small shared-memory footprint lets 8 CTAs per SM retire the
  // early-exiting ones in a third of the waves
  if (pl->smem_table && !RAPP_K3_GATED_GLOBAL) {
    if ((rc = launch_lattice<true, true, true>(pl, d_targets, f0, nf, chunks, st))) return rc;
  } else {
    if ((rc = launch_lattice<false, true, true>(pl, d_targets, f0, nf, chunks, st))) return rc;
  }
  RAPP_CUDA(launch_pdl(k_mec_fallback, dim3(hblocks), dim3(32 * wpb), 0, st, pl->d_fn,
                       pl->d_blist, f0, f1, pl->d_key, pl->d_minlat, pl->d_thr, pl->d_target2,
                       pl->d_fb));
  RAPP_LAUNCHED();
  if (pl->smem_table && !RAPP_K3_GATED_GLOBAL) {
    if ((rc = launch_lattice<true, false, true>(pl, pl->d_target2, f0, nf, chunks, st))) return rc;
  } else {
    if ((rc = launch_lattice<false, false, true>(pl, pl->d_target2, f0, nf, chunks, st))) return rc;
  }
  RAPP_CUDA(launch_pdl(k_mec_decode, dim3((unsigned)((nf + 127) / 128)), dim3(128), 0, st,
                       c->d_desc, c->d_pool, pl->d_fn, pl->d_blist, f0, f1, pl->d_key,
                       d_out_bsq, d_out_key));
  RAPP_LAUNCHED();
  return RAPP_OK;
}

}  // namespace rapp

extern "C" {

int rapp_mec_plan_create(rapp_ctx* ctx, int64_t nfn, const int32_t* table_of_fn,
                         int32_t quota_step, const int64_t* batch_off,
                         const int64_t* batch_lattice, rapp_mec_plan** out) {
  if (!ctx || !out || nfn < 0 || (nfn > 0 && (!table_of_fn || !batch_off || !batch_lattice))) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  if (quota_step < 1 || quota_step > 100) {
    set_error("quota_step must be in [1, 100]");  // hs/perf.py:116-117
    return RAPP_E_VALUE;
  }
  std::lock_guard<std::mutex> lk(ctx->mu);
  std::unique_ptr<rapp_mec_plan> pl(new rapp_mec_plan());
  pl->ctx = ctx;
  pl->nfn = nfn;
  pl->step = quota_step;
  pl->nQ = 100 / quota_step;
  std::vector<FnDesc> fns((size_t)nfn);
  std::vector<double> blist;
  int64_t max_seg = 0, max_ns = 0, max_nB = 0;
  for (int64_t f = 0; f < nfn; ++f) {
    const int32_t t = table_of_fn[f];
    if (t < 0 || t >= (int32_t)ctx->tables.size()) {
      set_error("unknown table id %d for function %lld", t, (long long)f);
      return RAPP_E_ARG;
    }
    const TableDesc& td = ctx->tables[t];
    const int64_t nB = batch_off[f + 1] - batch_off[f];
    if (nB < 1 || nB > 4096 || td.ns > 4096) {
      set_error("function %lld: batch lattice size %lld / sm axis %d outside [1, 4096]",
                (long long)f, (long long)nB, td.ns);
      return RAPP_E_ARG;
    }
    fns[f].table = t;
    fns[f].nB = (int32_t)nB;
    fns[f].boff = (int64_t)blist.size();
    for (int64_t i = 0; i < nB; ++i) {
      const int64_t b = batch_lattice[batch_off[f] + i];
      if (i && b <= batch_lattice[batch_off[f] + i - 1]) {
        set_error("function %lld: batch lattice must be sorted unique", (long long)f);
        return RAPP_E_ARG;
      }
      blist.push_back((double)b);
    }
    max_seg = std::max<int64_t>(max_seg, td.seg_doubles);
    max_ns = std::max<int64_t>(max_ns, td.ns);
    max_nB = std::max<int64_t>(max_nB, nB);
    pl->max_pairs = std::max<int>(pl->max_pairs, td.ns * pl->nQ);
    pl->points += nB * td.ns * pl->nQ;
  }
  // the packed key needs integral sm values in [0, 2^24) (checked at upload)
  for (int64_t f = 0; f < nfn; ++f)
    if (!ctx->tables[fns[f].table].sm_keyable) {
      set_error("table %d: sm axis unsupported by the lattice search (need integers in "
                "[0, 2^24))", fns[f].table);
      return RAPP_E_ARG;
    }
  pl->total_b = (int64_t)blist.size();
  pl->smem_table = max_seg * 8 <= kSearchSmemTable;
  const int64_t brk = 2 * max_ns + 2 * pl->nQ + 12 * max_nB + 2 + (max_ns + 1) / 2;
  pl->smem_bytes = (size_t)((pl->smem_table ? max_seg : 0) + brk) * 8;
  pl->smem_brk_bytes = (size_t)brk * 8;
  if (pl->smem_bytes > 200 * 1024) {
    set_error("lattice search shared-memory footprint %zu bytes too large", pl->smem_bytes);
    return RAPP_E_ARG;
  }
  RAPP_CUDA(cudaSetDevice(ctx->device));
  const size_t nb_alloc = (size_t)std::max<int64_t>(1, pl->total_b);
  const size_t nf_alloc = (size_t)std::max<int64_t>(1, nfn);
  RAPP_CUDA(cudaMalloc(&pl->d_fn, nf_alloc * sizeof(FnDesc)));
  RAPP_CUDA(cudaMalloc(&pl->d_blist, nb_alloc * 8));
  RAPP_CUDA(cudaMalloc(&pl->d_thr, nb_alloc * 8));
  RAPP_CUDA(cudaMalloc(&pl->d_minlat, nb_alloc * 8));
  RAPP_CUDA(cudaMalloc(&pl->d_key, nf_alloc * 8));
  RAPP_CUDA(cudaMalloc(&pl->d_target2, nf_alloc * 8));
  RAPP_CUDA(cudaMalloc(&pl->d_fb, nf_alloc * 4));
  if (nfn) {
    RAPP_CUDA(cudaMemcpy(pl->d_fn, fns.data(), fns.size() * sizeof(FnDesc),
                         cudaMemcpyHostToDevice));
    RAPP_CUDA(cudaMemcpy(pl->d_blist, blist.data(), blist.size() * 8, cudaMemcpyHostToDevice));
  }
  *out = pl.release();
  return RAPP_OK;
}

int rapp_mec_plan_destroy(rapp_mec_plan* pl) {
  if (!pl) return RAPP_OK;
  cudaSetDevice(pl->ctx->device);
  cudaDeviceSynchronize();
  cudaFree(pl->d_fn);
  cudaFree(pl->d_blist);
  cudaFree(pl->d_thr);
  cudaFree(pl->d_minlat);
  cudaFree(pl->d_key);
  cudaFree(pl->d_target2);
  cudaFree(pl->d_fb);
  cudaFree(pl->d_slo);
  for (cudaEvent_t e : pl->ev) cudaEventDestroy(e);
  if (pl->h_stage) cudaFreeHost(pl->h_stage);
  if (pl->d_stage) cudaFree(pl->d_stage);
  if (pl->stream) cudaStreamDestroy(pl->stream);
  delete pl;
  return RAPP_OK;
}

int rapp_mec_plan_points(rapp_mec_plan* pl, int64_t* points) {
  if (!pl || !points) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  *points = pl->points;
  return RAPP_OK;
}

int rapp_mec_plan_set_slo(rapp_mec_plan* pl, const double* slo_ms) {
  if (!pl) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  std::lock_guard<std::mutex> lk(pl->ctx->mu);
  RAPP_CUDA(cudaSetDevice(pl->ctx->device));
  RAPP_CUDA(cudaDeviceSynchronize());  // no run of this plan may still read the old values
  if (slo_ms == nullptr) {
    cudaFree(pl->d_slo);
    pl->d_slo = nullptr;
    return RAPP_OK;
  }
  for (int64_t f = 0; f < pl->nfn; ++f)
    if (!(slo_ms[f] > 0.0) && !std::isnan(slo_ms[f])) {
      set_error("slo_ms must be positive (NaN: no SLO), got %g for function %lld", slo_ms[f],
                (long long)f);
      return RAPP_E_VALUE;
    }
  if (!pl->d_slo) RAPP_CUDA(cudaMalloc(&pl->d_slo, (size_t)std::max<int64_t>(1, pl->nfn) * 8));
  if (pl->nfn)
    RAPP_CUDA(cudaMemcpy(pl->d_slo, slo_ms, (size_t)pl->nfn * 8, cudaMemcpyHostToDevice));
  return RAPP_OK;
}

int rapp_mec_plan_timing(rapp_mec_plan* pl, int enable) {
  if (!pl) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  pl->timing = enable != 0;
  pl->ev_used = 0;
  return RAPP_OK;
}

int rapp_mec_plan_kernel_time(rapp_mec_plan* pl, double* total_ms, int64_t* launches) {
  if (!pl || !total_ms || !launches) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  double sum = 0.0;
  for (size_t i = 0; i + 1 < pl->ev_used; i += 2) {
    RAPP_CUDA(cudaEventSynchronize(pl->ev[i + 1]));
    float ms = 0.f;
    RAPP_CUDA(cudaEventElapsedTime(&ms, pl->ev[i], pl->ev[i + 1]));
    sum += ms;
  }
  *total_ms = sum;
  *launches = (int64_t)(pl->ev_used / 2);
  return RAPP_OK;
}

int rapp_mec_plan_run_dev(rapp_mec_plan* pl, const double* d_targets, int64_t fn_begin,
                          int64_t fn_end, int32_t* d_out_bsq, uint64_t* d_out_key,
                          void* stream) {
  RAPP_RANGE("rapp_mec_plan_run_dev");
  if (!pl || fn_begin < 0 || fn_end > pl->nfn || fn_begin > fn_end) {
    set_error("bad plan or function range");
    return RAPP_E_ARG;
  }
  RAPP_CUDA(cudaSetDevice(pl->ctx->device));
  return run_plan(pl, d_targets, fn_begin, fn_end, d_out_bsq, d_out_key, (cudaStream_t)stream);
}

int rapp_mec_plan_run(rapp_mec_plan* pl, const double* targets, int64_t fn_begin, int64_t fn_end,
                      int64_t* out_bsq) {
  RAPP_RANGE("rapp_mec_plan_run");
  if (!pl || fn_begin < 0 || fn_end > pl->nfn || fn_begin > fn_end ||
      (fn_end > fn_begin && (!targets || !out_bsq))) {
    set_error("bad plan run arguments");
    return RAPP_E_ARG;
  }
  const int64_t nf = fn_end - fn_begin;
  for (int64_t f = 0; f < nf; ++f)
    if (targets[f] <= 0.0) {
      set_error("target_rps must be positive");  // hs/perf.py:114-115
      return RAPP_E_VALUE;
    }
  if (nf == 0) return RAPP_OK;
  std::lock_guard<std::mutex> lk(pl->ctx->mu);
  RAPP_CUDA(cudaSetDevice(pl->ctx->device));
  const size_t tb = (size_t)pl->nfn * 8, ob = (size_t)pl->nfn * 12;
  if (!pl->stream) {
    RAPP_CUDA(cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking));
    RAPP_CUDA(cudaMallocHost(&pl->h_stage, tb + ob));
    RAPP_CUDA(cudaMalloc(&pl->d_stage, tb + ob));
  }
  // targets are indexed by function id inside the plan: stage them at their slots
  memcpy(pl->h_stage + (size_t)fn_begin * 8, targets, (size_t)nf * 8);
  RAPP_CUDA(cudaMemcpyAsync(pl->d_stage + (size_t)fn_begin * 8, pl->h_stage + (size_t)fn_begin * 8,
                            (size_t)nf * 8, cudaMemcpyHostToDevice, pl->stream));
  int32_t* d_o = reinterpret_cast<int32_t*>(pl->d_stage + tb);
  int rc = run_plan(pl, reinterpret_cast<const double*>(pl->d_stage), fn_begin, fn_end, d_o,
                    nullptr, pl->stream);
  if (rc) return rc;
  int32_t* h_o = reinterpret_cast<int32_t*>(pl->h_stage + tb);
  RAPP_CUDA(cudaMemcpyAsync(h_o, d_o, (size_t)nf * 12, cudaMemcpyDeviceToHost, pl->stream));
  RAPP_CUDA(cudaStreamSynchronize(pl->stream));
  for (int64_t i = 0; i < nf * 3; ++i) out_bsq[i] = h_o[i];
  return RAPP_OK;
}

int rapp_mec_batch(rapp_ctx* ctx, int64_t nfn, const int32_t* table_of_fn, const double* targets,
                   int32_t quota_step, const int64_t* batch_off, const int64_t* batch_lattice,
                   int64_t* out_bsq) {
  for (int64_t f = 0; f < nfn; ++f)
    if (targets[f] <= 0.0) {
      set_error("target_rps must be positive");  // hs/perf.py:114-115
      return RAPP_E_VALUE;
    }
  rapp_mec_plan* pl = nullptr;
  int rc = rapp_mec_plan_create(ctx, nfn, table_of_fn, quota_step, batch_off, batch_lattice, &pl);
  if (rc) return rc;
  std::unique_ptr<rapp_mec_plan, int (*)(rapp_mec_plan*)> guard(pl, rapp_mec_plan_destroy);
  if (nfn == 0) return RAPP_OK;
  double* d_t = nullptr;
  int32_t* d_o = nullptr;
  RAPP_CUDA(cudaMalloc(&d_t, (size_t)nfn * 8));
  RAPP_CUDA(cudaMalloc(&d_o, (size_t)nfn * 12));
  RAPP_CUDA(cudaMemcpy(d_t, targets, (size_t)nfn * 8, cudaMemcpyHostToDevice));
  rc = run_plan(pl, d_t, 0, nfn, d_o, nullptr, 0);
  std::vector<int32_t> h((size_t)nfn * 3);
  cudaError_t e = cudaMemcpy(h.data(), d_o, (size_t)nfn * 12, cudaMemcpyDeviceToHost);
  cudaFree(d_t);
  cudaFree(d_o);
  if (rc) return rc;
  RAPP_CUDA(e);
  for (int64_t i = 0; i < nfn * 3; ++i) out_bsq[i] = h[(size_t)i];
  return RAPP_OK;
}

}  // extern "C"
