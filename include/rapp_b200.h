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
/* Destroys the internal per-device contexts of the stateless entry points
 * (rapp_interp3_many & co.).  For a clean process shutdown only (leak checks). */
int rapp_shutdown(void);
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

/* Small-batch evaluation for the scalar API (PerfTable.predict_latency / throughput,
 * hs/perf.py:80-102): latency[i] and, if rps != NULL, throughput of coords[i,:] (host
 * buffers, n rows of (batch, sm%, quota%)).  Persistent pinned staging: one H2D copy, one
 * launch and one D2H copy per call, no allocation after the first. */
int rapp_table_points(rapp_ctx *ctx, int32_t table_id, int64_t n, const double *coords,
                      double *latency, double *rps);

/* ---- perf-table ingest (load_table / validate_table_file, hs/perf.py:155-267) ----------
 * Native row reader for the strict common CSV form: the exact header line, then
 * `fid,int,int,int,float` rows with one function id, no quoting, padding, blank lines or
 * non-ASCII bytes.  *regular = 1 and n_rows rows are written (cap >= rows) when the whole
 * file has that form; otherwise *regular = 0 and the caller reads it with a full CSV reader
 * (which also produces the reference's format-error messages). */
int rapp_csv_parse(const char *buf, int64_t len, int64_t cap, int64_t *batch, int64_t *sm,
                   int64_t *quota, double *latency, int64_t *n_rows, char *function_id,
                   int64_t function_id_cap, int32_t *regular);

/* Grid assembly and validation on the device.  Rows are (batch, sm, quota, latency) in file
 * order.  Axes = sorted distinct values per column (hs/perf.py:209-211); a row whose cell
 * already has an earlier row is a duplicate (perf.py:200-205); every empty cell is
 * missing (perf.py:216-221); when none is missing every cell is checked for v <= 0 and for
 * monotonicity along batch / sm / quota (perf.py:239-267).  Cell flag bits: 1 missing,
 * 2 non_positive, 4 batch decreases, 8 sm increases, 16 quota increases. */
typedef struct rapp_ingest rapp_ingest;
int rapp_ingest_create(rapp_ctx *ctx, int64_t n_rows, const int64_t *batch, const int64_t *sm,
                       const int64_t *quota, const double *latency, rapp_ingest **out);
int rapp_ingest_shape(rapp_ingest *ing, int64_t *nb, int64_t *ns, int64_t *nq,
                      int32_t *n_missing, int32_t *n_flagged, int32_t *n_duplicates);
/* Host copies (any pointer may be NULL): axes (int64), grid (nb*ns*nq doubles, C order,
 * 0.0 at missing cells), cell flags (nb*ns*nq bytes), per-row duplicate flags (n_rows). */
int rapp_ingest_read(rapp_ingest *ing, int64_t *b_axis, int64_t *s_axis, int64_t *q_axis,
                     double *grid, uint8_t *cell_flags, uint8_t *row_duplicate);
int rapp_ingest_destroy(rapp_ingest *ing);

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

/* Same over host buffers (the scalar most_efficient_config and PerfTableSet.search):
 * targets[0 .. fn_end-fn_begin) for functions [fn_begin, fn_end) -> out_bsq (b,s,q) per
 * function.  The plan keeps pinned staging and a stream: one H2D, the search launches, one
 * D2H per call.  RAPP_E_VALUE when a target is <= 0 (hs/perf.py:114-115). */
int rapp_mec_plan_run(rapp_mec_plan *plan, const double *targets, int64_t fn_begin,
                      int64_t fn_end, int64_t *out_bsq);

/* Opt-in latency SLO (north_star: feasibility "latency <= SLO"; the reference reads
 * FunctionSpec.slo_ms nowhere, hs/core.py:96-98, hs/perf.py:132): slo_ms[f] > 0 makes a
 * lattice point feasible for function f only if rps >= target AND latency <= slo_ms[f];
 * NaN means no SLO for that function; slo_ms == NULL (the default) restores the reference
 * rule for every function.  When no point is feasible the fallback is the reference's
 * unchanged max-throughput rule over the whole lattice.  RAPP_E_VALUE for slo <= 0. */
int rapp_mec_plan_set_slo(rapp_mec_plan *plan, const double *slo_ms);

/* Measurement: when enabled (which also resets the record), every run brackets its meet
 * pass — the fused lattice kernel K3 — with CUDA events on the run's stream;
 * rapp_mec_plan_kernel_time synchronises them and returns the summed kernel time and the
 * number of timed launches. */
int rapp_mec_plan_timing(rapp_mec_plan *plan, int enable);
int rapp_mec_plan_kernel_time(rapp_mec_plan *plan, double *total_ms, int64_t *launches);

/* ---- batched scaler tick (hs/sim.py:470-491 driving hs/autoscaler.py:73-234) ---------
 * A device-resident scaler world: functions (in sorted-id order), their tables, the
 * cluster (GPUs in sorted-id order with their partition lists in insertion order, pods),
 * per-function Kalman state and scale-down stamps.  rapp_tick_run evaluates one scaler
 * tick for every function — Kalman update, Autoscaler.scale, and the apply step — with
 * the reference's sequential-commit semantics: function k decides against the cluster as
 * left by functions 0..k-1 of the same tick. */

typedef struct {
    double alpha, beta;        /* ScalerConfig (hs/autoscaler.py:28-43) */
    double cooldown_ms, r_min;
    int32_t delta_iq;
    int32_t policy;            /* 0 hybrid (HybridPolicy), 1 replica-count baseline
                                  (_ReplicaPolicy: horizontal-only / exclusive-gpu,
                                  hs/policies.py:49-160) */
    double interval_s;         /* scaler_interval_ms / 1000.0, computed by the caller */
    double cold_start_ms;      /* SimConfig.cold_start_ms (new pods become RUNNING then) */
    double kal_A, kal_Q, kal_H, kal_D, kal_P0;  /* Kalman defaults (hs/kalman.py:15-19) */
    int32_t sum_mode;          /* the caller's float sum() (hs/autoscaler.py:86-87): 0 CPython
                                  >= 3.12 (Neumaier-compensated), 1 older (left to right) */
    int32_t _pad;
} rapp_scaler_config;

typedef struct {
    int32_t table_id;          /* rapp_table_create id of perf_table_ref or function_id */
    int32_t _pad;
    double min_rps;            /* NaN: None (the scaler-wide r_min applies) */
    int64_t lattice_off;       /* its most_efficient_config batch lattice (after the   */
    int64_t lattice_len;       /*   _batch_lattice rule) inside `batch_lattice`        */
    int32_t kal_init;          /* 1: R/P below hold state; 0: first tick initialises  */
    int32_t _pad2;
    double kal_R, kal_P;
    double last_down_ms;       /* -inf when the function never scaled down */
    int32_t shape_batch;       /* replica policy: the fixed pod shape (initial_config) */
    int32_t shape_sm, shape_quota, _pad3;
} rapp_fn_desc;

typedef struct {
    int32_t fn;                /* function index, or -1 for pods of unmanaged functions */
    int32_t batch, sm, quota;
    int32_t gpu;               /* GPU rank (position in sorted GPU ids) */
    int32_t part;              /* position of its partition in the GPU's list */
    int32_t state;             /* 0 COLD_STARTING, 1 RUNNING, 2 DRAINING */
    int32_t _pad;
    double ready_at_ms;
    char id[32];               /* pod id, NUL-padded (string order decides ties) */
} rapp_pod_desc;

typedef struct {
    int32_t fn;                /* function index */
    int32_t kind;              /* 0 VERTICAL_UP 1 VERTICAL_DOWN 2 HORIZONTAL_UP 3 HORIZONTAL_DOWN */
    int32_t batch, sm, quota;
    int32_t pod;               /* pod index (new pods: the index created by the apply) */
    int32_t gpu;               /* GPU rank */
    int32_t released;          /* HORIZONTAL_DOWN: 1 if the idle pod was released */
} rapp_action;

typedef struct rapp_tick rapp_tick;

/* part_off has n_gpus+1 entries; partitions are (sm, quota_allocated) pairs in list order.
 * pod_counter is the next `pod-%06d` counter value for pods the ticks create. */
int rapp_tick_create(rapp_ctx *ctx, const rapp_scaler_config *cfg, int64_t n_fns,
                     const rapp_fn_desc *fns, const int64_t *batch_lattice, int64_t n_gpus,
                     const int64_t *part_off, const int32_t *part_sm,
                     const int32_t *part_alloc, int64_t n_pods, const rapp_pod_desc *pods,
                     int64_t pod_counter, rapp_tick **out);
int rapp_tick_destroy(rapp_tick *t);

/* One tick at time now_ms.  arrivals[n_fns] are the tick's request counts; idle[i] (for
 * every pod index < rapp_tick_pod_count) marks pods with no queued or in-service work, so
 * that a HORIZONTAL_DOWN releases them at once.  If predicted != NULL the Kalman step is
 * skipped and predicted[f] is used as the rate (Autoscaler.scale semantics).  Outputs:
 * actions (capacity max_actions), n_actions, observed/predicted rates per function (either
 * may be NULL).  The device world is updated in place. */
int rapp_tick_run(rapp_tick *t, double now_ms, const int64_t *arrivals, const uint8_t *idle,
                  const double *predicted_in, rapp_action *actions, int64_t max_actions,
                  int64_t *n_actions, double *observed_out, double *predicted_out);

/* rapp_tick_run in two halves, so the caller can work while the tick runs on the device:
 * submit copies the inputs and enqueues the tick and its output copy (no synchronisation);
 * collect waits for it and returns what rapp_tick_run returns (same arguments, same
 * errors).  Exactly one collect follows each successful submit, with no other call on the
 * handle in between (RAPP_E_ARG otherwise). */
int rapp_tick_submit(rapp_tick *t, double now_ms, const int64_t *arrivals, const uint8_t *idle,
                     const double *predicted_in, int64_t max_actions);
int rapp_tick_collect(rapp_tick *t, rapp_action *actions, int64_t max_actions,
                      int64_t *n_actions, double *observed_out, double *predicted_out);

/* Host events between ticks: pods the simulator released (a DRAINING pod whose last
 * request completed, hs/sim.py:424-438), applied in order before the next tick. */
int rapp_tick_release(rapp_tick *t, const int64_t *pods, int64_t n);

/* Same with device buffers and no host synchronisation (for timing / graphs). */
int rapp_tick_run_dev(rapp_tick *t, double now_ms, const int64_t *d_arrivals,
                      const uint8_t *d_idle, void *stream);
/* Device views of the last tick's outputs (valid until the next run). */
int rapp_tick_outputs_dev(rapp_tick *t, const rapp_action **d_actions, const int32_t **d_count,
                          const double **d_observed, const double **d_predicted);

int rapp_tick_pod_count(rapp_tick *t, int64_t *n_pods);
/* Host copy of the world (after any number of ticks): pods (alive flag via state -1 for
 * released pods), per-function Kalman / stamp state, partitions per GPU, pod counter. */
int rapp_tick_read_pods(rapp_tick *t, rapp_pod_desc *pods, int64_t cap, int64_t *n);
/* Opt-in latency SLO for the fresh-GPU configuration search of the tick
 * (hs/autoscaler.py:155-165 calls most_efficient_config; see rapp_mec_plan_set_slo for the
 * rule): slo_ms[f] > 0 per function (NaN: none); NULL restores the reference rule.  Rebuilds
 * the tick's search index (synchronous).  RAPP_E_VALUE for slo <= 0. */
int rapp_tick_set_slo(rapp_tick *t, const double *slo_ms);
int rapp_tick_read_fns(rapp_tick *t, rapp_fn_desc *fns);
int rapp_tick_read_parts(rapp_tick *t, int64_t *part_off, int32_t *part_sm,
                         int32_t *part_alloc, int32_t *part_npods, int64_t cap);
int rapp_tick_counter(rapp_tick *t, int64_t *pod_counter);

/* ---- learned RaPP predictor (§8(f) row 4, PerfModel protocol hs/perf.py:23-31) -------
 * No reference counterpart exists (the paper's GNN/MLP predictor is out of the reference's
 * scope), so this path has no parity target: it is checked against a PyTorch
 * fp32 forward of the same BF16 operands.  Model: x = [graph features (40) | 16 config
 * features of (batch, sm%, quota%), the last the constant 1 | 0 pad] (64) -> relu(W1 x + b1)
 * (127 units + a constant unit) -> relu(W2 . + b2) (127 + 1) -> exp(min(w3 . + b3, 80)) =
 * latency ms.  The biases ride on the constant feature / units (b1 replaces W1 column 55,
 * b2 W2 column 127, b3 w3[127]), so all three layers are BF16 tensor-core GEMMs.  Weights
 * are fp32 row-major (W1 [128][64], W2 [128][128], w3 [128]); graph_features [n][40]. */
typedef struct rapp_mlp rapp_mlp;
int rapp_mlp_create(rapp_ctx *ctx, int32_t n_models, const float *graph_features,
                    const float *w1, const float *b1, const float *w2, const float *b2,
                    const float *w3, float b3, rapp_mlp **out);
int rapp_mlp_destroy(rapp_mlp *mlp);
/* d_coords (n,3) float64 rows of one model -> d_out (n) float64 latency; tcgen05 GEMMs. */
int rapp_mlp_predict_dev(rapp_mlp *mlp, int32_t model, const double *d_coords, int64_t n,
                         double *d_out, void *stream);
/* Same over host buffers through the chunked copy-in / kernel / copy-out pipeline. */
int rapp_mlp_predict_host(rapp_mlp *mlp, int32_t model, const double *coords, int64_t n,
                          double *out);
/* most_efficient_config over the learned predictions (hs/perf.py:104-145 semantics): for
 * function f (model d_model_of_fn[f]) the lattice batches x sms x range(step, 101, step);
 * rps = b / (latency / 1000.0) in FP64; d_keys[f] = the packed min (s*q, s_idx, q, b_idx) key
 * over rps >= d_targets[f], else over rps == max rps (the reference's fallback order);
 * key bits: cost << 32 | s_idx << 20 | q << 12 | b_idx.  d_scratch: 2 * n_fn uint64.
 * sms must be integral in [0, 2^24); both axes sorted, at most 4096 values. */
int rapp_mlp_search_dev(rapp_mlp *mlp, int64_t n_fn, const int32_t *d_model_of_fn,
                        const double *d_targets, int32_t n_batches, const double *d_batches,
                        int32_t n_sms, const double *d_sms, int32_t quota_step,
                        uint64_t *d_keys, uint64_t *d_scratch, void *stream);
/* Diagnostics: same, and the first tile's raw FP32 accumulators (before bias) of both
 * layers into d_acc[2][128][128]. */
int rapp_mlp_debug_dev(rapp_mlp *mlp, int32_t model, const double *d_coords, int64_t n,
                       double *d_out, float *d_acc, void *stream);

/* ---- run metrics finalize (SimulationEngine._finalize, hs/sim.py:586-621) ------------
 * Functions in sorted-id order.  counts[f] = {arrived, rejected, unfinished, completed};
 * latencies of f = latencies[lat_off[f] .. lat_off[f+1]) (any order); cost intervals of f =
 * intervals[iv_off[f] .. iv_off[f+1]) rows {start_ms, end_ms (<0: open), sm, quota} in the
 * reference's list order.  Outputs: violation curve [F][n_mult] over the SLO multipliers
 * (baseline * m), nearest-rank percentiles [F][n_pct] for pct_q (NaN without latencies),
 * cost [F] (compute_cost, sim.py:160-175, open intervals priced to end_ms) and cost per
 * 1k completed requests [F].  n_mult <= 64, n_pct <= 8.  Host buffers. */
int rapp_metrics_finalize(rapp_ctx *ctx, int64_t n_fns, const double *baseline_ms,
                          const int64_t *counts, const int64_t *lat_off,
                          const double *latencies, const int64_t *iv_off,
                          const double *intervals, double price_per_gpu_hour, double end_ms,
                          int32_t n_mult, const double *multipliers, int32_t n_pct,
                          const int32_t *pct_q, double *curve_out, double *pct_out,
                          double *cost_out, double *cost_per_1k_out);

/* ---- measurement probes (bench.py; not on the product path) --------------------------
 * Non-FMA FP64 instruction rate of `device` (independent __dadd_rn / __dmul_rn chains on
 * every SM): the denominator of the lattice search's FP64 roofline. */
int rapp_probe_fp64(int device, double *dadd_per_s, double *dmul_per_s);

/* ---- kernel-launch accounting (evidence for bench.py's gpu_launches) ----------------- */
int64_t rapp_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RAPP_B200_H */
