// K2 fast path: stream interpolation for validated tables (strictly ascending axes).
//
// Same results, bit for bit, as the literal kernel (rapp_core.cu) and the reference
// (hs/_kernels/_grid_cy.pyx:9-51); three data-layout changes make it cheaper:
//  1. locate() without a binary search: a per-axis bucket table (LUT, in shared memory)
//     gives a starting index that is then corrected by exact comparisons, so the bracket
//     is the unique lo with a[lo] <= x < a[lo+1] — the binary search's answer for a
//     strictly ascending axis — in 1-3 shared-memory reads instead of log2(n) dependent
//     global loads.
//  2. t = (x - a[lo]) / (a[hi] - a[lo]): when the interval width is a power of two the
//     quotient is computed as an exact multiply by its (exactly representable) reciprocal.
//     RN(n * 2^-e) == RN(n / 2^e), so this is still the IEEE-correct quotient.  Other
//     widths use the IEEE division.
//  3. "cell" layout: the 8 corners of every grid cell are stored contiguously (64 B), so a
//     query is 4 x 16-byte loads from 2 sectors instead of 8 scattered 8-byte loads.
//     Clamped / node-hit brackets (lo == hi) select the same corner twice, exactly as the
//     reference reads v[lo] twice.
#include <cmath>
#include <cstring>
#include <vector>

#include "rapp_device.cuh"
#include "rapp_internal.h"

namespace rapp {

constexpr int kLut = 256;  // buckets per axis


static FastLayout fast_layout(int64_t nb, int64_t ns, int64_t nq) {
  FastLayout L{};
  L.o_par = 0;
  L.o_lut = 12;
  L.o_inv_b = L.o_lut + 3 * kLut / 2;
  L.o_inv_s = L.o_inv_b + pad2(nb > 1 ? nb - 1 : 1);
  L.o_inv_q = L.o_inv_s + pad2(ns > 1 ? ns - 1 : 1);
  L.o_cells = L.o_inv_q + pad2(nq > 1 ? nq - 1 : 1);
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

// Builds the fast-path extras for a strictly ascending table.
int build_fast_extras(int64_t nb, int64_t ns, int64_t nq, const double* b, const double* s,
                      const double* q, const double* v, std::vector<double>& ext,
                      FastLayout& L) {
  L = fast_layout(nb, ns, nq);
  if ((int64_t)L.total_doubles > (int64_t(1) << 30)) return RAPP_E_ARG;
  ext.assign((size_t)L.total_doubles, 0.0);
  const double* axes[3] = {b, s, q};
  const int64_t ns_[3] = {nb, ns, nq};
  const int32_t o_inv[3] = {L.o_inv_b, L.o_inv_s, L.o_inv_q};
  int32_t* lut = reinterpret_cast<int32_t*>(ext.data() + L.o_lut);
  for (int a = 0; a < 3; ++a) {
    const double* ax = axes[a];
    const int64_t n = ns_[a];
    const double a0 = ax[0], al = ax[n - 1];
    double invw = 0.0;
    if (n > 1 && std::isfinite(al - a0) && (al - a0) > 0.0) invw = double(kLut) / (al - a0);
    ext[L.o_par + 4 * a + 0] = a0;
    ext[L.o_par + 4 * a + 1] = al;
    ext[L.o_par + 4 * a + 2] = invw;
    ext[L.o_par + 4 * a + 3] = 0.0;
    for (int k = 0; k < kLut; ++k) {
      // largest i <= n-2 with a[i] <= bucket start; the kernel corrects any rounding
      const double xk = a0 + (al - a0) * (double(k) / kLut);
      int64_t i = 0;
      while (i + 1 <= n - 2 && ax[i + 1] <= xk) ++i;
      lut[a * kLut + k] = (int32_t)i;
    }
    for (int64_t i = 0; i + 1 < n; ++i) {
      double r = 0.0;
      if (!pow2_recip(ax[i + 1] - ax[i], &r)) r = 0.0;
      ext[o_inv[a] + i] = r;
    }
  }
  const int64_t cb = nb > 1 ? nb - 1 : 1, cs = ns > 1 ? ns - 1 : 1, cq = nq > 1 ? nq - 1 : 1;
  double* cells = ext.data() + L.o_cells;
  for (int64_t i = 0; i < cb; ++i)
    for (int64_t j = 0; j < cs; ++j)
      for (int64_t k = 0; k < cq; ++k) {
        double* c = cells + ((i * cs + j) * cq + k) * 8;
        for (int d = 0; d < 8; ++d) {
          const int64_t ii = std::min(i + ((d >> 2) & 1), nb - 1);
          const int64_t jj = std::min(j + ((d >> 1) & 1), ns - 1);
          const int64_t kk = std::min(k + (d & 1), nq - 1);
          c[d] = v[(ii * ns + jj) * nq + kk];
        }
      }
  return RAPP_OK;
}

struct FastAxis {
  const double* a;
  const int32_t* lut;
  const double* inv;
  int n;
  double a0, al, invw;
};

// Bracket of x as (cell index c, corner selectors s0/s1 for lo/hi, t).  Identical
// (lo, hi, t) to rapp::locate() for a strictly ascending axis: lo = c + s0, hi = c + s1.
__device__ __forceinline__ void locate_fast(const FastAxis& ax, double x, int& c, int& s0,
                                            int& s1, double& t) {
  const int last = ax.n - 1;
  if (x <= ax.a0) { c = 0; s0 = 0; s1 = 0; t = 0.0; return; }
  if (x >= ax.al) {
    c = last > 0 ? last - 1 : 0;
    s0 = s1 = last - c;
    t = 0.0;
    return;
  }
  if (x != x) {  // NaN: the reference's search ends at (0, min(1, last))
    c = 0;
    s0 = 0;
    s1 = last > 0 ? 1 : 0;
    t = __ddiv_rn(__dsub_rn(x, ax.a0), __dsub_rn(ax.a[s1], ax.a0));
    return;
  }
  // here a0 < x < a_last, so n >= 2 and the answer lies in [0, n-2]
  int k = int(__dmul_rn(__dsub_rn(x, ax.a0), ax.invw));
  k = k < kLut - 1 ? k : kLut - 1;
  k = k > 0 ? k : 0;
  int i = ax.lut[k];
  while (i < last - 1 && ax.a[i + 1] <= x) ++i;
  while (i > 0 && ax.a[i] > x) --i;
  const double lo = ax.a[i];
  c = i;
  s0 = 0;
  if (lo == x) { s1 = 0; t = 0.0; return; }
  s1 = 1;
  const double num = __dsub_rn(x, lo);
  const double r = ax.inv[i];
  t = r != 0.0 ? __dmul_rn(num, r) : __ddiv_rn(num, __dsub_rn(ax.a[i + 1], lo));
}

__device__ __forceinline__ double2 pick2(int sel, double2 a, double2 b) { return sel ? b : a; }
__device__ __forceinline__ double pickq(int sel, double2 w) { return sel ? w.y : w.x; }

constexpr int kFastThreads = 256;
constexpr int kFastIlp = 2;

template <bool CELLS_SMEM>
__global__ void __launch_bounds__(kFastThreads)
    k_interp_fast(const TableDesc td, const double* __restrict__ pool,
                  const double* __restrict__ coords, int64_t n, double* __restrict__ out,
                  double* __restrict__ rps) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint64_t bar;
  const int axes_doubles = td.ov;  // [b | s | q] with padding
  double* s_axes = sm;
  double* s_ext = sm + axes_doubles;
  const double* ext_g = pool + td.xoff;
  const uint32_t small_bytes = uint32_t(td.x_small) * 8u;
  const uint32_t cell_bytes = CELLS_SMEM ? uint32_t(td.x_total - td.x_small) * 8u : 0u;
  bulk_load_2(s_axes, pool + td.off, uint32_t(axes_doubles) * 8u, s_ext, ext_g,
              small_bytes + cell_bytes, &bar);
  const double* cells = CELLS_SMEM ? s_ext + td.x_small : ext_g + td.x_small;
  const int32_t* lut = reinterpret_cast<const int32_t*>(s_ext + 12);
  FastAxis ab{s_axes + td.ob, lut, s_ext + td.x_inv_b, td.nb, s_ext[0], s_ext[1], s_ext[2]};
  FastAxis as{s_axes + td.os, lut + kLut, s_ext + td.x_inv_s, td.ns, s_ext[4], s_ext[5],
              s_ext[6]};
  FastAxis aq{s_axes + td.oq, lut + 2 * kLut, s_ext + td.x_inv_q, td.nq, s_ext[8], s_ext[9],
              s_ext[10]};
  const int CS = td.ns > 1 ? td.ns - 1 : 1, CQ = td.nq > 1 ? td.nq - 1 : 1;

  const int64_t stride = int64_t(gridDim.x) * kFastThreads * kFastIlp;
  for (int64_t base = int64_t(blockIdx.x) * kFastThreads * kFastIlp + threadIdx.x; base < n;
       base += stride) {
    double cb[kFastIlp], cs[kFastIlp], cq[kFastIlp];
#pragma unroll
    for (int k = 0; k < kFastIlp; ++k) {
      const int64_t i = base + int64_t(k) * kFastThreads;
      if (i < n) {
        cb[k] = __ldcs(coords + 3 * i);
        cs[k] = __ldcs(coords + 3 * i + 1);
        cq[k] = __ldcs(coords + 3 * i + 2);
      }
    }
#pragma unroll
    for (int k = 0; k < kFastIlp; ++k) {
      const int64_t i = base + int64_t(k) * kFastThreads;
      if (i >= n) continue;
      int ib, bs0, bs1, js, ss0, ss1, kq, qs0, qs1;
      double tb, ts, tq;
      locate_fast(ab, cb[k], ib, bs0, bs1, tb);
      locate_fast(as, cs[k], js, ss0, ss1, ts);
      locate_fast(aq, cq[k], kq, qs0, qs1, tq);
      const double2* cp =
          reinterpret_cast<const double2*>(cells + ((int64_t(ib) * CS + js) * CQ + kq) * 8);
      double2 w[4];
      if (CELLS_SMEM) {
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = cp[u];
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = __ldg(cp + u);
      }
      // w[db*2 + ds] = (corner dq=0, corner dq=1)
      const double2 b0 = pick2(ss0, w[0], w[1]), b0h = pick2(ss1, w[0], w[1]);
      const double2 b1 = pick2(ss0, w[2], w[3]), b1h = pick2(ss1, w[2], w[3]);
      const double2 w00 = pick2(bs0, b0, b1), w01 = pick2(bs0, b0h, b1h);
      const double2 w10 = pick2(bs1, b0, b1), w11 = pick2(bs1, b0h, b1h);
      const double c00 = lerp_rn(pickq(qs0, w00), pickq(qs1, w00), tq);
      const double c01 = lerp_rn(pickq(qs0, w01), pickq(qs1, w01), tq);
      const double c10 = lerp_rn(pickq(qs0, w10), pickq(qs1, w10), tq);
      const double c11 = lerp_rn(pickq(qs0, w11), pickq(qs1, w11), tq);
      const double c0 = lerp_rn(c00, c01, ts);
      const double c1 = lerp_rn(c10, c11, ts);
      const double lat = lerp_rn(c0, c1, tb);
      __stcs(out + i, lat);
      if (rps != nullptr) __stcs(rps + i, throughput(cb[k], lat));
    }
  }
}

constexpr int64_t kFastCellsSmem = 96 * 1024;

int launch_interp_fast(rapp_ctx* ctx, const TableDesc& td, const double* d_coords, int64_t n,
                       double* d_out, double* d_rps, cudaStream_t st) {
  const int64_t cell_bytes = int64_t(td.x_total - td.x_small) * 8;
  const int64_t small_bytes = (int64_t(td.ov) + td.x_small) * 8;
  const bool cells_smem = cell_bytes + small_bytes <= kFastCellsSmem;
  const size_t smem = (size_t)(small_bytes + (cells_smem ? cell_bytes : 0));
  const int64_t per_block = int64_t(kFastThreads) * kFastIlp;
  int64_t blocks = (n + per_block - 1) / per_block;
  const int64_t cap = int64_t(ctx->sm_count) * (cells_smem ? 2 : 8);
  if (blocks > cap) blocks = cap;
  if (!ctx->fast_attr_set) {
    RAPP_CUDA(cudaFuncSetAttribute(k_interp_fast<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kFastCellsSmem));
    RAPP_CUDA(cudaFuncSetAttribute(k_interp_fast<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kFastCellsSmem));
    ctx->fast_attr_set = true;
  }
  if (cells_smem)
    k_interp_fast<true><<<(unsigned)blocks, kFastThreads, smem, st>>>(td, ctx->d_pool, d_coords,
                                                                      n, d_out, d_rps);
  else
    k_interp_fast<false><<<(unsigned)blocks, kFastThreads, smem, st>>>(td, ctx->d_pool,
                                                                       d_coords, n, d_out, d_rps);
  RAPP_LAUNCHED();
  return RAPP_OK;
}

}  // namespace rapp
