/*
 * rapp_b200.h — C ABI of the B200-native RaPP prediction + configuration-search path.
 *
 * Drop-in boundary for the reference package `hybridscale` (HAS-GPU).  Paths are
 * relative to /root/reference; hs/ = pkg/src/hybridscale/.  The reference binds its
 * table kernel from Python (Cython module hs/_kernels/_grid_cy.pyx, selected by
 * hs/_kernels/__init__.py:8-15); a Python host binds this library with ctypes the same
 * way.  No torch types appear here: plain pointers and sizes.
 *
 * Conventions
 *   - Every entry point returns RAPP_OK (0) or an error code; rapp_last_error() gives a
 *     thread-local message whose prefix matches the reference exception text.
 *   - "_dev" entry points take DEVICE pointers and a cudaStream_t passed as void*; they
 *     are stream-ordered and do not synchronise.  Other entry points take HOST pointers
 *     and return when results are in host memory.
 *   - Arithmetic is IEEE binary64 with every operation individually rounded (no FMA
 *     contraction), so results are bit-identical to the reference's CPU kernel.
 *   - One context per device; the library keeps a default context per device for the
 *     stateless reference-shaped entry points.
 */
#ifndef RAPP_B200_H
#define RAPP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    RAPP_OK = 0,
    RAPP_E_VALUE = 1,       /* -> ValueError (hs/perf.py:88-91, :114-117)            */
    RAPP_E_TABLE = 2,       /* -> TableFormatError (hs/perf.py:73-76, hs/errors.py:29) */
    RAPP_E_ARG = 3,         /* bad handle / id / size                                  */
    RAPP_E_CUDA = 4,        /* CUDA runtime failure (no device, launch error, OOM)     */
    RAPP_E_PLACEMENT = 5,   /* -> PlacementError (hs/allocator.py:96-99,116-123)       */
    RAPP_E_INVARIANT = 6,   /* -> InvariantViolation (hs/core.py:160-197)              */
    RAPP_E_DEGENERATE = 7   /* -> FilterDegenerateError (hs/kalman.py:56-57)           */
};

const char *rapp_last_error(void);
/* Library version string and the compile target ("sm_100a"). */
const char *rapp_version(void);

/* ---- reference-shaped stateless kernels (hs/_kernels/_grid_cy.pyx) ------------------ */

/* Replaces `locate(axis, x)` — hs/_kernels/_grid_cy.pyx:54-58 (logic :9-33). */
int rapp_locate(const double *axis, int64_t n, double x,
                int64_t *lo, int64_t *hi, double *t);

/* Replaces `interp3(b_axis, s_axis, q_axis, values, b, s, q)` — _grid_cy.pyx:61-64. */
int rapp_interp3(const double *b_axis, int64_t nb, const double *s_axis, int64_t ns,
                 const double *q_axis, int64_t nq, const double *values,
                 double b, double s, double q, double *out);

/* Replaces `interp3_many(b_axis, s_axis, q_axis, values, coords, out)` —
 * _grid_cy.pyx:67-74.  coords is (n,3) row-major (batch, sm%, quota%); out is (n).
 * Host buffers; page-locked buffers are DMA'd directly, pageable ones are staged.
 * The copy-in, kernel and copy-out of successive chunks overlap on several streams. */
int rapp_interp3_many(const double *b_axis, int64_t nb, const double *s_axis, int64_t ns,
                      const double *q_axis, int64_t nq, const double *values,
                      const double *coords, int64_t n, double *out);

/* ---- contexts and device-resident tables (PerfTable, hs/perf.py:56-76) --------------- */

typedef struct rapp_ctx rapp_ctx;

int rapp_ctx_create(int device, rapp_ctx **out);
int rapp_ctx_destroy(rapp_ctx *ctx);
/* Device the context lives on and the number of SMs. */
int rapp_ctx_info(rapp_ctx *ctx, int *device, int *sm_count);

/* Uploads one immutable (nb,ns,nq) C-order float64 grid plus its axes.  Axes must be
 * strictly ascending (the reference's CSV loader builds them sorted-unique,
 * hs/perf.py:214-217).  Returns a table id >= 0. */
int rapp_table_create(rapp_ctx *ctx, int64_t nb, int64_t ns, int64_t nq,
                      const double *b_axis, const double *s_axis, const double *q_axis,
                      const double *values, int32_t *table_id);
int rapp_table_count(rapp_ctx *ctx, int32_t *count);

/* Stream interpolation on device buffers: d_out[i] = interp3(table, d_coords[i,:]).
 * If d_rps != NULL also writes throughput d_coords[i,0] / (d_out[i] / 1000.0)
 * (hs/perf.py:95-98). */
int rapp_interp3_many_dev(rapp_ctx *ctx, int32_t table_id, const double *d_coords,
                          int64_t n, double *d_out, double *d_rps, void *stream);

/* Same over host buffers (the PerfTable-level drop-in with copies inside). */
int rapp_interp3_many_host(rapp_ctx *ctx, int32_t table_id, const double *coords,
                           int64_t n, double *out);

/* ---- configuration search: most_efficient_config batched over functions --------------
 * hs/perf.py:104-145.  Function f searches table_of_fn[f] over the lattice
 *   B_f x table.sms x range(quota_step, 101, quota_step)
 * where B_f = batch_lattice[batch_off[f] .. batch_off[f+1]) (the caller has applied the
 * `_batch_lattice` rule, hs/perf.py:140-145: sorted-unique allowed batches inside the
 * table's batch range, else all table batches).  Result: out_bsq[3f..3f+2] = (b,s,q) of
 * the min (s*q, s, q, b) point with throughput >= targets[f], else of the
 * min (-throughput, s*q, s, q, b) point.
 * Host arrays; evaluated on the context's device.  targets must be > 0 (RAPP_E_VALUE
 * otherwise, as perf.py:114-115) and 1 <= quota_step <= 100 (perf.py:116-117). */
int rapp_mec_batch(rapp_ctx *ctx, int64_t nfn, const int32_t *table_of_fn,
                   const double *targets, int32_t quota_step, const int64_t *batch_off,
                   const int64_t *batch_lattice, int64_t *out_bsq);

/* Device-resident plan for repeated searches over a fixed function set (the per-tick
 * path): the batch lattices are uploaded once. */
typedef struct rapp_mec_plan rapp_mec_plan;
int rapp_mec_plan_create(rapp_ctx *ctx, int64_t nfn, const int32_t *table_of_fn,
                         int32_t quota_step, const int64_t *batch_off,
                         const int64_t *batch_lattice, rapp_mec_plan **out);
int rapp_mec_plan_destroy(rapp_mec_plan *plan);
/* Number of lattice points (predictions) one run of the plan evaluates. */
int rapp_mec_plan_points(rapp_mec_plan *plan, int64_t *points);
/* d_targets: nfn doubles on device; d_out_bsq: 3*nfn int32 on device; d_out_key: nfn
 * uint64 packed meet keys (or NULL).  Functions [fn_begin, fn_end) only (sharding). */
int rapp_mec_plan_run_dev(rapp_mec_plan *plan, const double *d_targets, int64_t fn_begin,
                          int64_t fn_end, int32_t *d_out_bsq, uint64_t *d_out_key,
                          void *stream);

/* ---- kernel-launch accounting (evidence for bench.py's gpu_launches) ----------------- */
int64_t rapp_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RAPP_B200_H */
