// Batched scaler tick: every function's Kalman update + Autoscaler.scale + apply, in one
// sequence of launches, with the reference's sequential-commit semantics.
//
// Reference (paths relative to /root/reference/pkg/src/hybridscale):
//   tick driver        sim.py:470-491   (sorted functions; decide; apply; next function)
//   apply              sim.py:493-525   (change_quota / place new COLD_STARTING pod /
//                                        DRAINING + immediate release when idle)
//   decision           autoscaler.py:73-234
//   allocator          allocator.py:17-139
//   Kalman             kalman.py:45-62
//
// Decomposition (exact):
//  phase A (k_tick_phase_a, one warp per function, all functions in parallel) computes
//    everything a function's decision reads from its OWN state only: the Kalman step, the
//    non-draining pods sorted by (-sm, pod_id), capability (CPython 3.12 sum(): Neumaier
//    compensated), the up / down / no-op classification, the whole scale-down walk (it
//    never reads shared state), and for scale-up the throughput of every pod at every
//    quota step.  No other function can change these inputs within a tick.
//  phase A2 (k_tick_grid) tabulates throughput(batch_ref, sm, q) for sm, q in 1..100 of
//    every scale-up function: the used-GPU branch reads only this table once the GPU and
//    its best slot are known.
//  phase B (k_tick_commit, one warp) walks the functions in order and performs the parts
//    that read shared state — partition headroom for the vertical walk, the lowest
//    (occupancy, gpu id) used GPU, its best slot, the covering quota, the first free GPU
//    and the fresh-GPU configuration search (prefix-max index, see below) — applying each
//    action to the device cluster before the next function decides.  Consecutive
//    functions whose commit phase A already knows up to a validation (FastRec: a vertical
//    walk that closes the gap, or one followed by the horizontal branch, or vertical
//    scale-down steps) are committed one per lane in a single step (Commit::fast_run),
//    under exactly the conditions in which the sequential walk would repeat phase A's.
//
// Every floating-point expression is evaluated in the reference's order with individually
// rounded operations (interp3 / throughput from rapp_device.cuh; explicit _rn intrinsics).
#include <array>
#include <climits>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <algorithm>
#include <vector>

#include "rapp_device.cuh"
#include "rapp_internal.h"

namespace rapp {

constexpr int kMaxPods = 128;  // pods per managed function (RAPP_E_ARG beyond)
constexpr int kMaxGpus = 1 << 18;  // GPUs per world (rank field of the argmin keys)
constexpr int kMaxFns = 1 << 20;   // managed functions per world
constexpr int kPartCap = 100;  // partitions per GPU (each >= 1 SM%, sum <= 100)
constexpr int kRow = 101;      // quota steps per pod row
constexpr int kCold = 0, kRunning = 1, kDraining = 2, kDead = -1;
constexpr int kNone = 0, kUp = 1, kDown = 2;
enum : int { kVUp = 0, kVDown = 1, kHUp = 2, kHDown = 3 };

struct PodId {
  uint64_t w[4];  // id bytes, big-endian packed: integer order == byte-string order
};

__host__ __device__ inline bool id_less(const PodId& a, const PodId& b) {
  for (int i = 0; i < 4; ++i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
  return false;
}

struct DownAct {
  int32_t kind, pod, quota, _pad;
};

// A function whose commit is known from phase A up to a validation ("straight-line"): a
// scale-up whose speculative vertical walk closes the gap (kFastUp) or leaves `gap` for the
// horizontal branch (kFastTail: the walk is straight-line, the rest runs sequentially), or
// a scale-down of vertical steps only (kFastDown).  Steps are the walked pods / staged
// actions in order: pod, GPU, tick-start partition position and uid, its sm / batch, quota
// before and after, and (scale-up) the tick-start quota allocated on the partition the walk
// assumed.
constexpr int kFastSteps = 2;
struct FastStep {
  int32_t p, g, pos, s, b, qold, qnew, alloc0;  // alloc0 < 0: nothing to validate
  uint32_t uid;
};
enum : int { kFastNone = 0, kFastUp = 1, kFastTail = 2, kFastDown = 3 };
struct FastRec {
  double gap;    // kFastTail: the gap the walk leaves
  int32_t kind;  // kFast*
  int32_t n;     // steps
  FastStep st[kFastSteps];
};

// partition entry: sm (8 bits) | alloc (8 bits) | npods (16 bits) | uid (32 bits)
__host__ __device__ inline uint64_t part_pack(int sm, int alloc, int npods, uint32_t uid) {
  return uint64_t(uint32_t(sm) & 0xFF) | (uint64_t(uint32_t(alloc) & 0xFF) << 8) |
         (uint64_t(uint32_t(npods) & 0xFFFF) << 16) | (uint64_t(uid) << 32);
}
__host__ __device__ inline int part_sm(uint64_t e) { return int(e & 0xFF); }
__host__ __device__ inline int part_alloc(uint64_t e) { return int((e >> 8) & 0xFF); }
__host__ __device__ inline int part_npods(uint64_t e) { return int((e >> 16) & 0xFFFF); }
__host__ __device__ inline uint32_t part_uid(uint64_t e) { return uint32_t(e >> 32); }

// phase A2 tabulates only the tick-start slot sms when the quota step is at most this
// (100 / delta >= 25 quota steps per row); coarser steps tabulate every row
constexpr int kMaskMaxDelta = 4;

// one locate() result (_grid_cy.pyx:9-33): bracket lo, hi and weight t
struct TickBrk {
  int32_t lo, hi;
  double t;
};
constexpr int kBrkPerFn = 201;  // 100 sm values, 100 quota steps, the reference batch

struct World {
  // config
  double alpha, beta, cooldown, r_min, interval_s, cold_start, kA, kQ, kH, kD, kP0;
  int delta, F, G, pod_cap;
  int policy;                    // 0 hybrid, 1 replica-count baseline
  int sum_plain;                 // 1: CPython < 3.12 float sum (left to right, no compensation)
  const int32_t* fn_shape;       // [F][3] replica policy pod shape (b, s, q)
  int32_t* wanted;               // replica scale-up: ceil(gap / pod_cap), clamped
  // tables
  const TableDesc* tds;
  const double* pool;
  // functions
  const int32_t* fn_table;
  const double* fn_min_rps;
  const int64_t* fn_lat_off;     // most_efficient_config lattice offsets (prefix-max index)
  const int64_t* fn_lat_len;     // lattice points of f = nB_f * nS * nQ
  const int32_t* fn_nb;          // |B_f|
  const int64_t* fn_boff;        // batch list offset
  const double* blist;           // batch lattices (sorted unique, as doubles)
  const int32_t* fn_pairs_off;   // (s,q) pairs in key order, per lattice shape
  const int32_t* fn_npairs;
  const int32_t* pairs;          // packed s_index << 16 | q
  const double* pmax;            // prefix max of rps along the key-sorted lattice
  const double* fn_slo;          // opt-in latency SLO per function (NaN: none), or null
  const int64_t* fn_fb;          // with an SLO: index of the unmasked max-rps fallback
  int32_t* k_init;
  double* k_R;
  double* k_P;
  double* last_down;
  int32_t* fn_npods;
  int32_t* fn_pods;              // [F][kMaxPods]
  // gpus
  int32_t* g_npods;
  int32_t* g_hgo;                // sum of sm*quota over resident pods (any state)
  int32_t* g_nparts;
  int32_t* g_freesm;
  uint32_t* g_nextuid;
  uint64_t* g_parts;             // [G][kPartCap] in list order
  // pods
  int32_t* n_pods;               // device counter (pods ever created, incl. released)
  int32_t* p_fn;
  int32_t* p_b;
  int32_t* p_s;
  int32_t* p_q;
  int32_t* p_gpu;
  uint32_t* p_puid;
  int32_t* p_state;
  double* p_ready;
  PodId* p_id;
  int64_t* p_ctr;                // pod-%06d counter of a pod the commit created whose id is
                                 // not formatted yet (-1: formatted) — formatted off the
                                 // commit's critical path (next prologue / before reads)
  const uint8_t* p_idle;         // per tick input
  int64_t* counter;              // next pod-%06d counter
  // phase A / A2 outputs
  double* obs;
  double* pred;
  int32_t* cls;
  double* gap0;
  int32_t* nsorted;              // non-draining pods of f, sorted by (-sm, id)
  int32_t* sorted;               // [F][kMaxPods]
  int32_t* row_kd;               // [F][kMaxPods] index of q0 inside the row
  double* rows;                  // [F][kMaxPods][kRow] throughput at q0 + k*delta
  int32_t* bref;                 // batch of sorted[0]
  int32_t* bref_ok;              // bref inside the table's batch range (hs/perf.py:88-91)
  // speculative vertical walk against tick-start headroom (phase A), per sorted pod:
  int32_t* spec_avail;           // [F][kMaxPods] avail the walk assumed (-1: not walked)
  int32_t* spec_k;               // [F][kMaxPods] steps taken
  double* spec_gain;             // [F][kMaxPods] gain of those steps
  int32_t* spec_kg;              // [F][kMaxPods] first step whose gain closes the gap the
                                 // walk assumed (any headroom; (100 - q0) / d + 1: none)
  FastRec* fast;                 // [F] straight-line commits (n = 0: none)
  double* tgrid;                 // [F][100][100] throughput(bref, sm, q)
  TickBrk* brk;                  // [F][201] phase A2's brackets: sm 1..100, quota steps, bref
  int32_t mask_none;             // tests: tabulate no row (every used-GPU row from brackets)
  uint32_t* sm_mask;             // [4] sm values (bit sm-1) tabulated in tgrid this tick: the
                                 // tick-start partition sms and unallocated shares
  int32_t* ndown;
  DownAct* down;                 // [F][kMaxPods]
  int32_t* stamp;                // 1: record last_down = now
  // outputs
  rapp_action* actions;
  int32_t* n_actions;
  int32_t* err;                  // first error code (RAPP_E_*)
  int32_t* err_fn;
};

// CPython's sum() over floats, started from int 0 (0 + x0 == x0 for the positive rates
// summed here): from 3.12 on it is Neumaier-compensated, before that plain left to right.
// The caller's interpreter decides (rapp_scaler_config.sum_mode).
template <class Get>
__device__ __forceinline__ double py_float_sum(const World& w, int m, Get get) {
  double s = get(0);
  if (w.sum_plain) {
    for (int j = 1; j < m; ++j) s = __dadd_rn(s, get(j));
    return s;
  }
  double c = 0.0;
  for (int j = 1; j < m; ++j) {
    const double x = get(j);
    const double t = __dadd_rn(s, x);
    if (fabs(s) >= fabs(x))
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x));
    else
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), s));
    s = t;
  }
  if (c != 0.0 && isfinite(c)) s = __dadd_rn(s, c);
  return s;
}

__device__ __forceinline__ double thr_at(const World& w, int f, double b, double s, double q) {
  const TableDesc td = w.tds[w.fn_table[f]];
  const double* seg = w.pool + td.off;
  const double lat = interp3(seg + td.ob, td.nb, seg + td.os, td.ns, seg + td.oq, td.nq,
                             seg + td.ov, b, s, q);
  return throughput(b, lat);  // b / (lat / 1000.0), hs/perf.py:95-98
}

// thr_at along one quota row: the batch and sm brackets of (b, s) are located once, each
// entry locates its quota and evaluates the same interp3 expression (same doubles).
struct ThrRow {
  const double* qa;
  const double* v;
  int nq;
  int64_t r00, r01, r10, r11;
  double tb, ts, b;
};

__device__ __forceinline__ ThrRow thr_row(const World& w, int f, double b, double s) {
  const TableDesc td = w.tds[w.fn_table[f]];
  const double* seg = w.pool + td.off;
  ThrRow r;
  int i0, i1, j0, j1;
  locate(seg + td.ob, td.nb, b, i0, i1, r.tb);
  locate(seg + td.os, td.ns, s, j0, j1, r.ts);
  r.qa = seg + td.oq;
  r.v = seg + td.ov;
  r.nq = td.nq;
  r.r00 = (int64_t(i0) * td.ns + j0) * td.nq;
  r.r01 = (int64_t(i0) * td.ns + j1) * td.nq;
  r.r10 = (int64_t(i1) * td.ns + j0) * td.nq;
  r.r11 = (int64_t(i1) * td.ns + j1) * td.nq;
  r.b = b;
  return r;
}

__device__ __forceinline__ double thr_row_at(const ThrRow& r, double q) {
  int k0, k1;
  double tq;
  locate(r.qa, r.nq, q, k0, k1, tq);
  const double* v = r.v;
  const double c00 = lerp_rn(v[r.r00 + k0], v[r.r00 + k1], tq);
  const double c01 = lerp_rn(v[r.r01 + k0], v[r.r01 + k1], tq);
  const double c10 = lerp_rn(v[r.r10 + k0], v[r.r10 + k1], tq);
  const double c11 = lerp_rn(v[r.r11 + k0], v[r.r11 + k1], tq);
  const double c0 = lerp_rn(c00, c01, r.ts);
  const double c1 = lerp_rn(c10, c11, r.ts);
  return throughput(r.b, lerp_rn(c0, c1, r.tb));  // b / (lat / 1000.0), hs/perf.py:95-98
}

__device__ __forceinline__ bool batch_ok(const World& w, int f, int b) {
  const TableDesc td = w.tds[w.fn_table[f]];
  const double* ba = w.pool + td.off + td.ob;
  const double x = double(b);
  return !(x < ba[0] || x > ba[td.nb - 1]);  // hs/perf.py:88-91
}


#ifdef RAPP_TICK_PROF
// diagnostics build only: cycles of the commit's parts, summed over ticks (lane 0)
__device__ unsigned long long g_tick_prof[32];
__shared__ unsigned long long s_tprof[32];  // per-launch accumulators, flushed at the end
#define TPROF_T0() long long _tp0 = clock64()
#define TPROF_ACC(i)                                                   \
  do {                                                                 \
    const long long _tp1 = clock64();                                  \
    if ((threadIdx.x & 31) == 0) s_tprof[i] += (unsigned long long)(_tp1 - _tp0); \
    _tp0 = _tp1;                                                       \
  } while (0)
#else
#define TPROF_T0() (void)0
#define TPROF_ACC(i) (void)0
#endif

__device__ void set_err(const World& w, int code, int f) {
  if (atomicCAS(w.err, 0, code) == 0) *w.err_fn = f;
}

// ---------------------------------------------------------------------------------------
// prologue: cold starts that ended at or before `now` (ready events precede the scaler
// event at equal timestamps, sim.py:40-44), output reset
// ---------------------------------------------------------------------------------------
// "pod-%06d" (sim.py:337-340), big-endian packed so integer order is byte-string order
__device__ __forceinline__ PodId format_pod_id(long long c) {
  char buf[32] = {'p', 'o', 'd', '-'};
  int nd = 1;
  for (unsigned long long v = (unsigned long long)c / 10ull; v; v /= 10ull) ++nd;
  const int width = nd > 6 ? nd : 6;
  unsigned long long v = (unsigned long long)c;
  for (int i = width - 1; i >= 0; --i) {
    buf[4 + i] = char('0' + v % 10ull);
    v /= 10ull;
  }
  PodId id;
  for (int i = 0; i < 4; ++i) {
    uint64_t x = 0;
    for (int k = 0; k < 8; ++k) x = (x << 8) | uint8_t(buf[i * 8 + k]);
    id.w[i] = x;
  }
  return id;
}

__device__ __forceinline__ void format_pending(const World& w, int p) {
  const long long c = w.p_ctr[p];
  if (c >= 0) {
    w.p_id[p] = format_pod_id(c);
    w.p_ctr[p] = -1;
  }
}

__global__ void k_tick_format_ids(World w) {
  const int n = *w.n_pods;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    format_pending(w, p);
}

__global__ void k_tick_prologue(World w, double now) {
  pdl_trigger();
  const int n = *w.n_pods;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    format_pending(w, p);
    if (w.p_state[p] == kCold && w.p_ready[p] <= now) w.p_state[p] = kRunning;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *w.n_actions = 0;
    *w.err = 0;
    *w.err_fn = -1;
  }
  // the sm values a used-GPU slot can have while no partition is released: a tick-start
  // partition's sm (join) or a GPU's unallocated share (new partition) — phase A2 tabulates
  // those rows; a slot on any other share (freed by a release earlier in the tick) is
  // evaluated on demand by the commit.  The commit clears the mask after use.  With coarse
  // quota steps the whole grid is cheap and every row is tabulated.
  if (w.delta > kMaskMaxDelta) {
    if (blockIdx.x == 0 && threadIdx.x < 4) w.sm_mask[threadIdx.x] = threadIdx.x < 3 ? ~0u : 0xFu;
    return;
  }
  if (w.mask_none) return;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < w.G; g += gridDim.x * blockDim.x) {
    const int n = w.g_nparts[g];
    for (int i = 0; i < n; ++i) {
      const int sm = part_sm(w.g_parts[int64_t(g) * kPartCap + i]);
      if (sm >= 1 && sm <= 100) atomicOr(&w.sm_mask[(sm - 1) >> 5], 1u << ((sm - 1) & 31));
    }
    const int fs = w.g_freesm[g];
    if (fs >= 1 && fs <= 100) atomicOr(&w.sm_mask[(fs - 1) >> 5], 1u << ((fs - 1) & 31));
  }
}

// CPython float floor division (Objects/floatobject.c _float_div_mod): fmod-based, with
// the quotient snapped to the nearest integer — not floor(x / y).
__device__ __forceinline__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = __ddiv_rn(__dsub_rn(vx, mod), wx);
  if (mod != 0.0) {
    if ((wx < 0.0) != (mod < 0.0)) {
      mod = __dadd_rn(mod, wx);
      div = __dsub_rn(div, 1.0);
    }
  }
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
  } else {
    fl = copysign(0.0, __ddiv_rn(vx, wx));
  }
  return fl;
}

// Replica-count baselines (hs/policies.py:69-105): fixed-shape pods, capability summed in
// pods-dict order (= pod index order), wanted = ceil(gap / pod_cap) new pods, scale-down
// removes floor(excess / pod_cap) RUNNING pods newest id first, never the last one.
__device__ void replica_phase_a(const World& w, int f, int lane, double R, double now,
                                int* lst) {
  int m = 0;
  if (lane == 0) {
    const int n = w.fn_npods[f];
    for (int i = 0; i < n; ++i) {
      const int p = w.fn_pods[f * kMaxPods + i];
      if (w.p_state[p] == kDraining) continue;
      int j = m++;
      while (j > 0 && lst[j - 1] > p) {
        lst[j] = lst[j - 1];
        --j;
      }
      lst[j] = p;
    }
  }
  __syncwarp();
  m = __shfl_sync(0xffffffffu, m, 0);
  if (m == 0) {
    if (lane == 0) w.cls[f] = kNone;
    return;
  }
  double* vals = w.rows + int64_t(f) * kMaxPods * kRow;  // scratch: one value per pod
  for (int j = lane; j < m; j += 32) {
    const int p = lst[j];
    if (!batch_ok(w, f, w.p_b[p])) set_err(w, RAPP_E_VALUE, f);
    vals[j] = thr_at(w, f, double(w.p_b[p]), double(w.p_s[p]), double(w.p_q[p]));
  }
  __syncwarp();
  if (lane != 0) return;
  const int* shape = w.fn_shape + 3 * f;
  if (!batch_ok(w, f, shape[0])) set_err(w, RAPP_E_VALUE, f);
  const double pod_cap = thr_at(w, f, double(shape[0]), double(shape[1]), double(shape[2]));
  const double cap = py_float_sum(w, m, [&](int j) { return vals[j]; });  // dict order
  const double up_thr = __dmul_rn(cap, w.alpha);
  if (R > up_thr) {
    const double want = ceil(__ddiv_rn(__dsub_rn(R, up_thr), pod_cap));
    w.wanted[f] = want > double(1 << 30) ? (1 << 30) : int(want);
    w.cls[f] = kUp;
    return;
  }
  const double mr = w.fn_min_rps[f];
  const double r_min = mr != mr ? w.r_min : mr;
  if (!(R < __dmul_rn(cap, w.beta) && R > r_min &&
        __dsub_rn(now, w.last_down[f]) >= w.cooldown)) {
    w.cls[f] = kNone;
    return;
  }
  // RUNNING pods newest first: pod id descending
  int run[kMaxPods];
  int nr = 0;
  for (int j = 0; j < m; ++j) {
    const int p = lst[j];
    if (w.p_state[p] != kRunning) continue;
    int i = nr++;
    while (i > 0 && id_less(w.p_id[run[i - 1]], w.p_id[p])) {
      run[i] = run[i - 1];
      --i;
    }
    run[i] = p;
  }
  const int removable = nr - 1 > 0 ? nr - 1 : 0;
  int count = 0;
  if (pod_cap > 0.0) {
    const double k = py_floordiv(__dsub_rn(cap, R), pod_cap);
    count = k < double(removable) ? int(k) : removable;  // min(removable, int(k))
    if (count < 0) count = 0;
  }
  DownAct* out = w.down + f * kMaxPods;
  for (int i = 0; i < count; ++i) out[i] = DownAct{kHDown, run[i], 0, 0};
  w.ndown[f] = count;
  w.stamp[f] = count > 0;
  w.cls[f] = kDown;
}

// ---------------------------------------------------------------------------------------
// phase A: one warp per function
// ---------------------------------------------------------------------------------------
__global__ void k_tick_phase_a(World w, double now, const int64_t* __restrict__ arrivals,
                               const double* __restrict__ pred_in) {
  pdl_trigger();
  pdl_wait();  // the prologue's pod-state promotions
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (f >= w.F) return;
  __shared__ int s_sorted[8][kMaxPods];
  __shared__ int s_run[8][kMaxPods];
  int* srt = s_sorted[(threadIdx.x >> 5) & 7];
  int* run = s_run[(threadIdx.x >> 5) & 7];

  // Kalman (kalman.py:45-62; first tick initialises R = observed, P = P0, sim.py:476-479)
  double R = 0.0;
  if (lane == 0) {
    const double obs = __ddiv_rn(double(arrivals[f]), w.interval_s);
    if (pred_in != nullptr) {
      R = pred_in[f];
    } else {
      double kR = w.k_init[f] ? w.k_R[f] : obs;
      double kP = w.k_init[f] ? w.k_P[f] : w.kP0;
      const double r_pred = __dmul_rn(w.kA, kR);
      const double p_pred = __dadd_rn(__dmul_rn(__dmul_rn(w.kA, kP), w.kA), w.kQ);
      const double denom = __dadd_rn(__dmul_rn(__dmul_rn(w.kH, p_pred), w.kH), w.kD);
      if (denom == 0.0) set_err(w, RAPP_E_DEGENERATE, f);
      const double gain = __ddiv_rn(__dmul_rn(p_pred, w.kH), denom);
      const double r_new =
          __dadd_rn(r_pred, __dmul_rn(gain, __dsub_rn(obs, __dmul_rn(w.kH, r_pred))));
      const double p_new = __dmul_rn(__dsub_rn(1.0, __dmul_rn(gain, w.kH)), p_pred);
      w.k_R[f] = r_new;
      w.k_P[f] = p_new;
      w.k_init[f] = 1;
      R = r_new > 0.0 ? r_new : 0.0;  // max(0.0, r_new)
    }
    w.obs[f] = obs;
    w.pred[f] = R;
  }
  R = __shfl_sync(0xffffffffu, R, 0);
  if (w.policy == 1) {
    replica_phase_a(w, f, lane, R, now, srt);
    return;
  }

  // non-draining pods sorted by (-sm, pod_id) (autoscaler.py:81-85)
  int m = 0;
  if (lane == 0) {
    const int n = w.fn_npods[f];
    for (int i = 0; i < n; ++i) {
      const int p = w.fn_pods[f * kMaxPods + i];
      if (w.p_state[p] == kDraining) continue;
      int j = m++;
      while (j > 0) {
        const int o = srt[j - 1];
        const bool before = w.p_s[p] > w.p_s[o] || (w.p_s[p] == w.p_s[o] && id_less(w.p_id[p], w.p_id[o]));
        if (!before) break;
        srt[j] = o;
        --j;
      }
      srt[j] = p;
    }
    w.nsorted[f] = m;
    for (int j = 0; j < m; ++j) w.sorted[f * kMaxPods + j] = srt[j];
  }
  __syncwarp();
  m = __shfl_sync(0xffffffffu, m, 0);
  if (m == 0) {
    if (lane == 0) w.cls[f] = kNone;
    return;
  }

  // throughput at the current quota of every pod (row entry k = 0)
  const int d = w.delta;
  double* rows = w.rows + int64_t(f) * kMaxPods * kRow;
  for (int j = lane; j < m; j += 32) {
    const int p = srt[j];
    const int q0 = w.p_q[p];
    const int kd = (q0 - 1) / d;
    w.row_kd[f * kMaxPods + j] = kd;
    if (!batch_ok(w, f, w.p_b[p])) set_err(w, RAPP_E_VALUE, f);
    rows[j * kRow + kd] = thr_at(w, f, double(w.p_b[p]), double(w.p_s[p]), double(q0));
  }
  __syncwarp();

  int cls = kNone;
  double cap = 0.0;
  if (lane == 0) {
    // capability = sum(...) in sorted order (hs/autoscaler.py:86-87)
    cap = py_float_sum(w, m, [&](int j) { return rows[j * kRow + w.row_kd[f * kMaxPods + j]]; });
    const double up_thr = __dmul_rn(cap, w.alpha);
    if (R > up_thr) {
      cls = kUp;
      w.gap0[f] = __dsub_rn(R, up_thr);
      w.bref[f] = w.p_b[srt[0]];
      w.bref_ok[f] = batch_ok(w, f, w.p_b[srt[0]]) ? 1 : 0;
    } else {
      const double mr = w.fn_min_rps[f];
      const double r_min = mr != mr ? w.r_min : mr;
      if (R < __dmul_rn(cap, w.beta) && R > r_min &&
          __dsub_rn(now, w.last_down[f]) >= w.cooldown)
        cls = kDown;
    }
  }
  cls = __shfl_sync(0xffffffffu, cls, 0);

  if (cls == kUp) {
    // rows k = 1..ku of RUNNING pods (the vertical walk skips the others)
    for (int j = 0; j < m; ++j) {
      const int p = srt[j];
      if (w.p_state[p] != kRunning) continue;
      const int q0 = w.p_q[p];
      const int kd = (q0 - 1) / d, ku = (100 - q0) / d;
      const ThrRow tr = thr_row(w, f, double(w.p_b[p]), double(w.p_s[p]));
      for (int k = 1 + lane; k <= ku; k += 32)
        rows[j * kRow + kd + k] = thr_row_at(tr, double(q0 + k * d));
    }
    __syncwarp();
    {
      // Speculate the vertical walk (autoscaler.py:115-133) with the tick-start headroom
      // of each pod's partition.  The walk of pod j depends only on that headroom and on
      // the gap left by pods 0..j-1 of this function, so phase B reuses it verbatim while
      // every headroom it observes equals the one assumed here.  Warp-wide: every lane
      // holds the same gap; the partition lookup and the walk's stopping step are found
      // lane-parallel.
      double gap = w.gap0[f];
      FastRec fr;
      fr.n = 0;
      bool simple = true;
      for (int j = 0; j < m; ++j) {
        if (lane == 0) w.spec_avail[f * kMaxPods + j] = -1;
        if (!(gap > 0.0)) continue;
        const int p = srt[j];
        if (w.p_state[p] != kRunning) continue;
        const int g = w.p_gpu[p];
        const uint32_t uid = w.p_puid[p];
        const uint64_t* P = w.g_parts + int64_t(g) * kPartCap;
        const int np = w.g_nparts[g];
        unsigned upos = 1u << 30;
        for (int i = lane; i < np; i += 32)
          if (part_uid(P[i]) == uid) upos = min(upos, unsigned(i));
        upos = __reduce_min_sync(0xffffffffu, upos);
        const int pos = upos < unsigned(np) ? int(upos) : -1;
        const int alloc = pos >= 0 ? part_alloc(P[pos]) : 100;
        const int q0 = w.p_q[p];
        const int avail = q0 + (100 - alloc);
        const double* row = rows + j * kRow + (q0 - 1) / d;
        // k = first step with q0 + (k+1)d > avail or !(gap - gain_k > 0), gain_0 = 0
        // (k <= (100 - q0) / d < 128: lanes hold k = lane + 32u)
        const double cur = row[0];
        int k = -1, kg = -1;
        double gain = 0.0;
        const int ku = (100 - q0) / d;
        // k* = min(kq, kg): kq = (avail - q0) / d, the first step the quota bound stops, and
        // kg, the first step whose gain closes the gap — kg depends on the gap alone, so the
        // commit recomputes k* from it in O(1) when only the headroom changed
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = u * 32 + lane;
          const bool row_in = kk > 0 && kk <= ku;
          const double gk = row_in ? __dsub_rn(row[kk], cur) : 0.0;
          const bool closes = row_in && !(__dsub_rn(gap, gk) > 0.0);
          const bool stop = q0 + (kk + 1) * d > avail || closes;
          const unsigned mask = __ballot_sync(0xffffffffu, stop);
          if (mask && k < 0) {
            const int l = __ffs(mask) - 1;
            k = u * 32 + l;
            gain = __shfl_sync(0xffffffffu, gk, l);
          }
          const unsigned cm = __ballot_sync(0xffffffffu, closes);
          if (cm && kg < 0) kg = u * 32 + __ffs(cm) - 1;
        }
        if (lane == 0) {
          w.spec_avail[f * kMaxPods + j] = avail;
          w.spec_k[f * kMaxPods + j] = k;
          w.spec_gain[f * kMaxPods + j] = gain;
          w.spec_kg[f * kMaxPods + j] = kg < 0 ? ku + 1 : kg;
        }
        if (k > 0) gap = __dsub_rn(gap, gain);
        // a second walked pod on the same partition would see the first one's change
        for (int t = 0; t < fr.n && t < kFastSteps; ++t)
          if (fr.st[t].g == g && fr.st[t].uid == w.p_puid[p]) simple = false;
        if (fr.n < kFastSteps && pos >= 0)
          fr.st[fr.n] = FastStep{p, g, pos, w.p_s[p], w.p_b[p], q0, q0 + k * d, alloc,
                                 w.p_puid[p]};
        else
          simple = false;
        ++fr.n;
      }
      if (lane == 0) {
        w.fast[f].kind = !simple ? kFastNone : gap > 0.0 ? kFastTail : kFastUp;
        w.fast[f].n = fr.n;
        w.fast[f].gap = gap;
        for (int t = 0; t < fr.n && t < kFastSteps; ++t) w.fast[f].st[t] = fr.st[t];
        w.cls[f] = kUp;
      }
    }
    return;
  }
  if (cls != kDown) {
    if (lane == 0) w.cls[f] = kNone;
    return;
  }

  // ---- scale-down (autoscaler.py:188-234): RUNNING pods by (sm, pod_id) ascending ----
  int nr = 0;
  if (lane == 0) {
    for (int j = 0; j < m; ++j) {
      const int p = srt[j];
      if (w.p_state[p] != kRunning) continue;
      int i = nr++;
      while (i > 0) {
        const int o = run[i - 1];
        const bool before = w.p_s[p] < w.p_s[o] || (w.p_s[p] == w.p_s[o] && id_less(w.p_id[p], w.p_id[o]));
        if (!before) break;
        run[i] = o;
        --i;
      }
      run[i] = p;
    }
  }
  __syncwarp();
  nr = __shfl_sync(0xffffffffu, nr, 0);
  // rows k = -kd..-1 for those pods; reuse the sorted-order row slots by pod lookup
  for (int i = 0; i < nr; ++i) {
    const int p = run[i];
    int j = 0;
    while (srt[j] != p) ++j;
    const int q0 = w.p_q[p];
    const int kd = (q0 - 1) / d;
    const ThrRow tr = thr_row(w, f, double(w.p_b[p]), double(w.p_s[p]));
    for (int k = 1 + lane; k <= kd; k += 32)
      rows[j * kRow + kd - k] = thr_row_at(tr, double(q0 - k * d));
  }
  __syncwarp();
  cap = __shfl_sync(0xffffffffu, cap, 0);
  {
    // warp-wide: every lane holds the same excess; each pod's stopping step is found
    // lane-parallel, the staged actions are written by lane 0
    double excess = __dsub_rn(cap, R);
    int alive = nr, na = 0;
    DownAct* out = w.down + f * kMaxPods;
    for (int i = 0; i < nr; ++i) {
      if (excess <= 0.0) break;
      const int p = run[i];
      int j = 0;
      while (srt[j] != p) ++j;
      const double* row = rows + j * kRow;
      const int q0 = w.p_q[p];
      const int kd = (q0 - 1) / d;
      const double cur = row[kd];
      // q_k = max(q0 - k d, 0), shed_k = q_k == 0 ? cur : cur - row[kd - k]; the loop stops
      // at the first k >= 1 with q_k == 0 or !(excess - shed_k > 0) (k <= ceil(q0/d) <= 100)
      int q = q0;
      double shed = 0.0;
      if (__dsub_rn(excess, 0.0) > 0.0) {  // (the loop's first test, k = 0)
        int ks = -1;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = u * 32 + lane + 1;
          const int qk = q0 - kk * d > 0 ? q0 - kk * d : 0;
          const double sk = qk == 0 ? cur : __dsub_rn(cur, row[kd - kk]);
          const bool stop = qk == 0 || !(__dsub_rn(excess, sk) > 0.0);
          const unsigned mask = __ballot_sync(0xffffffffu, stop);
          if (mask && ks < 0) {
            const int l = __ffs(mask) - 1;
            ks = u * 32 + l + 1;
            q = __shfl_sync(0xffffffffu, qk, l);
            shed = __shfl_sync(0xffffffffu, sk, l);
          }
        }
      }
      if (q == 0) {
        if (alive <= 1) {
          const int floor_q = q0 - d * ((q0 - 1) / d);
          if (floor_q < q0) {
            shed = __dsub_rn(cur, row[kd - (q0 - floor_q) / d]);
            if (lane == 0) out[na] = DownAct{kVDown, p, floor_q, 0};
            ++na;
            excess = __dsub_rn(excess, shed);
          }
          continue;
        }
        --alive;
        if (lane == 0) out[na] = DownAct{kHDown, p, 0, 0};
        ++na;
        excess = __dsub_rn(excess, cur);
      } else if (q < q0) {
        if (lane == 0) out[na] = DownAct{kVDown, p, q, 0};
        ++na;
        excess = __dsub_rn(excess, shed);
      }
    }
    __syncwarp();
    if (lane != 0) return;
    w.ndown[f] = na;
    w.stamp[f] = na > 0;
    // vertical steps only: no decision reads shared state, the commit just applies them
    bool simple = na > 0 && na <= kFastSteps;
    for (int i = 0; i < na && simple; ++i) {
      const DownAct a = out[i];
      const int p = a.pod, g = w.p_gpu[p];
      const uint64_t* P = w.g_parts + int64_t(g) * kPartCap;
      int pos = -1;
      for (int k = 0; k < w.g_nparts[g]; ++k)
        if (part_uid(P[k]) == w.p_puid[p]) {
          pos = k;
          break;
        }
      if (a.kind != kVDown || pos < 0) {
        simple = false;
        break;
      }
      w.fast[f].st[i] = FastStep{p, g, pos, w.p_s[p], w.p_b[p], w.p_q[p], a.quota, -1,
                                 w.p_puid[p]};
    }
    w.fast[f].kind = simple ? kFastDown : kFastNone;
    w.fast[f].n = na;
    w.cls[f] = kDown;
  }
}

// ---------------------------------------------------------------------------------------
// phase A2: throughput(batch_ref, sm, q) for sm, q in 1..100 of every scale-up function
// ---------------------------------------------------------------------------------------
// Only the quota multiples of delta are tabulated (the covering-quota scan reads those);
// c_max at an off-step q_max is evaluated on demand by the commit warp.  The batch bracket
// is fixed per function and the sm / quota brackets are shared by a whole row / column, so
// they are located once into shared memory (same locate, same doubles) and every entry is
// then 8 independent corner loads and the reference's 7 lerps + 2 divisions.
__global__ void __launch_bounds__(256) k_tick_grid(World w) {
  pdl_trigger();
  pdl_wait();  // phase A's classes and reference batches
  const int f = blockIdx.x;
  if (w.policy != 0 || w.cls[f] != kUp) return;
  const int b = w.bref[f];
  if (!batch_ok(w, f, b)) return;  // phase B raises if the value is ever needed
  __shared__ int2 s_j[100], s_k[100];
  __shared__ double s_ts[100], s_tq[100];
  __shared__ int s_i0, s_i1;
  __shared__ double s_tb;
  const TableDesc td = w.tds[w.fn_table[f]];
  const double* seg = w.pool + td.off;
  const double* ba = seg + td.ob;
  const double* sa = seg + td.os;
  const double* qa = seg + td.oq;
  const double* v = seg + td.ov;
  const int d = w.delta, nq = 100 / d;
  __shared__ int s_cand[100];
  __shared__ int s_ncand;
  if (threadIdx.x < 32) {  // the mask's sm rows, ascending
    int nc = 0;
    for (int base = 0; base < 100; base += 32) {
      const int sm0 = base + int(threadIdx.x);  // row index sm - 1
      const bool on = sm0 < 100 && ((w.sm_mask[sm0 >> 5] >> (sm0 & 31)) & 1u);
      const unsigned m = __ballot_sync(0xffffffffu, on);
      if (on) s_cand[nc + __popc(m & ((1u << threadIdx.x) - 1u))] = sm0;
      nc += __popc(m);
    }
    if (threadIdx.x == 0) s_ncand = nc;
  }
  for (int i = threadIdx.x; i < 100; i += blockDim.x) {
    int lo, hi;
    double t;
    locate(sa, td.ns, double(i + 1), lo, hi, t);
    s_j[i] = make_int2(lo, hi);
    s_ts[i] = t;
    if (i < nq) {
      locate(qa, td.nq, double((i + 1) * d), lo, hi, t);
      s_k[i] = make_int2(lo, hi);
      s_tq[i] = t;
    }
  }
  if (threadIdx.x == 0) {
    int lo, hi;
    double t;
    locate(ba, td.nb, double(b), lo, hi, t);
    s_i0 = lo;
    s_i1 = hi;
    s_tb = t;
  }
  __syncthreads();
  if (d <= kMaskMaxDelta) {  // the brackets, for rows the commit evaluates itself (sm
                             // values outside the mask)
    TickBrk* B = w.brk + int64_t(f) * kBrkPerFn;
    for (int i = threadIdx.x; i < 100; i += blockDim.x) {
      B[i] = TickBrk{s_j[i].x, s_j[i].y, s_ts[i]};
      if (i < nq) B[100 + i] = TickBrk{s_k[i].x, s_k[i].y, s_tq[i]};
    }
    if (threadIdx.x == 0) B[200] = TickBrk{s_i0, s_i1, s_tb};
  }
  const int64_t plane = int64_t(td.ns) * td.nq;
  const double* v0 = v + s_i0 * plane;
  const double* v1 = v + s_i1 * plane;
  const double tb = s_tb, bb = double(b);
  const bool fast = td.fast != 0;  // finite positive values (checked at upload)
  // kGridU entries per thread per round: every table load of the round is issued before
  // the first store (the stores could alias the loads as far as the compiler knows)
  constexpr int kGridU = 4;
  const int total = s_ncand * nq;
  for (int i0 = threadIdx.x; i0 < total; i0 += kGridU * blockDim.x) {
    double lat[kGridU];
    int64_t out[kGridU];
#pragma unroll
    for (int u = 0; u < kGridU; ++u) {
      const int i = i0 + u * int(blockDim.x);
      out[u] = -1;
      lat[u] = 0.0;
      if (i >= total) continue;
      const int ci = i / nq, qi = i - ci * nq;
      const int si = d > kMaskMaxDelta ? ci : s_cand[ci];
      out[u] = (int64_t(f) * 100 + si) * 100 + (qi + 1) * d - 1;
      const int2 j = s_j[si], k = s_k[qi];
      const double ts = s_ts[si], tq = s_tq[qi];
      const int o00 = j.x * td.nq + k.x, o01 = j.x * td.nq + k.y;
      const int o10 = j.y * td.nq + k.x, o11 = j.y * td.nq + k.y;
      // interp3 (_grid_cy.pyx:45-51): c_ij = lerp along quota, then sm, then batch.  The
      // table reads are streaming (evict-first) so this pass does not push the commit's
      // working set (phase A outputs, cluster state) out of L2.  On a node
      // bracket (lo == hi, t == 0) of a finite table lerp(v, v, 0) == v exactly, so those
      // lerps and their second loads are skipped (every quota step of a 1..100% table, and
      // every sm on the table's own grid, is a node).
      if (fast && k.x == k.y) {
        const double a00 = __ldcs(v0 + o00), a10 = __ldcs(v1 + o00);
        if (j.x == j.y) {
          lat[u] = lerp_rn(a00, a10, tb);
        } else {
          const double a01 = __ldcs(v0 + o10), a11 = __ldcs(v1 + o10);
          lat[u] = lerp_rn(lerp_rn(a00, a01, ts), lerp_rn(a10, a11, ts), tb);
        }
      } else {
        const double c00 = lerp_rn(__ldcs(v0 + o00), __ldcs(v0 + o01), tq);
        const double c01 = lerp_rn(__ldcs(v0 + o10), __ldcs(v0 + o11), tq);
        const double c10 = lerp_rn(__ldcs(v1 + o00), __ldcs(v1 + o01), tq);
        const double c11 = lerp_rn(__ldcs(v1 + o10), __ldcs(v1 + o11), tq);
        lat[u] = lerp_rn(lerp_rn(c00, c01, ts), lerp_rn(c10, c11, ts), tb);
      }
    }
    // default-policy stores: the commit's used-GPU branch reads these rows back from L2
#pragma unroll
    for (int u = 0; u < kGridU; ++u)
      if (out[u] >= 0) w.tgrid[out[u]] = throughput(bb, lat[u]);
  }
}

// ---------------------------------------------------------------------------------------
// phase B: sequential commit (one warp)
// ---------------------------------------------------------------------------------------
// mbarrier + bulk-copy helpers for the commit's row staging
__device__ __forceinline__ void tk_bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
      (uint32_t)__cvta_generic_to_shared(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tk_bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
      (uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tk_bulk(void* dst, const void* src, uint32_t bytes,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
      "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void tk_bar_wait(uint64_t* bar, uint32_t parity) {
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

__device__ __forceinline__ void mbar_init32(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(
      (uint32_t)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void mbar_arrive_rel(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
      (uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity)
      : "memory");
  return done != 0;
}

// the first pod's quota row of a function, staged for the commit (102 doubles = 816 B,
// the 101-entry row plus 8 bytes of the next row so the bulk size is a multiple of 16)
constexpr int kRowStage = 102;

// loads through generic pointers known to address shared memory
__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int lds_s32(const int32_t* p) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}

// conflict-mark slot of partition (g, pos) for fast_run (collisions only shorten runs)
constexpr int kFastHash = 512;
__device__ __forceinline__ int fast_hash(int g, int pos) {
  return int((uint32_t(g) * 2654435761u + uint32_t(pos) * 40503u) >> 23) & (kFastHash - 1);
}

// throughput(bref, sm, q) at this lane's quota steps q = (u*32 + lane + 1)*d <= qmax, from
// phase A2's brackets — the used-GPU branch's row when A2 did not tabulate this sm
struct Row4 {
  double v[4];
};
__device__ __forceinline__ Row4 bracket_row(const World& w, int f, int bref, int sm, int qmax,
                                         int d, int lane) {
  const TickBrk* B = w.brk + int64_t(f) * kBrkPerFn;
  const TickBrk bs = B[sm - 1], bb = B[200];
  const TableDesc td = w.tds[w.fn_table[f]];
  const double* v = w.pool + td.off + td.ov;
  const int64_t r00 = (int64_t(bb.lo) * td.ns + bs.lo) * td.nq;
  const int64_t r01 = (int64_t(bb.lo) * td.ns + bs.hi) * td.nq;
  const int64_t r10 = (int64_t(bb.hi) * td.ns + bs.lo) * td.nq;
  const int64_t r11 = (int64_t(bb.hi) * td.ns + bs.hi) * td.nq;
  Row4 r;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = u * 32 + lane;  // quota step index: q = (k + 1) * d
    r.v[u] = 0.0;
    if ((k + 1) * d <= qmax) {
      const TickBrk bq = B[100 + k];
      const double c00 = lerp_rn(v[r00 + bq.lo], v[r00 + bq.hi], bq.t);
      const double c01 = lerp_rn(v[r01 + bq.lo], v[r01 + bq.hi], bq.t);
      const double c10 = lerp_rn(v[r10 + bq.lo], v[r10 + bq.hi], bq.t);
      const double c11 = lerp_rn(v[r11 + bq.lo], v[r11 + bq.hi], bq.t);
      const double lat = lerp_rn(lerp_rn(c00, c01, bs.t), lerp_rn(c10, c11, bs.t), bb.t);
      r.v[u] = throughput(double(bref), lat);
    }
  }
  return r;
}

struct CommitPre {
  double gap0, sg0;
  int m, p0, st0, gpu0, q0, b0, s0, sav0, sk0, bref, brefok, npods, kd0, kg0;
  int nd, dkind, dquota, didle, stamp;
  int pos0;  // hint: position of the first pod's partition at tick start (-1: none)
  uint32_t uid0;
};

// kMasked: phase A2 tabulated only the sm rows of w.sm_mask (fine quota steps); the
// used-GPU branch evaluates any other row from A2's brackets.
template <bool kMasked>
struct CommitT {
  const World& w;
  int lane;
  // partition lists of GPUs with at most `ps` partitions live in shared memory for the
  // whole commit (sp[g*ps ...]); a GPU that has or grows beyond ps uses its global row
  uint64_t* sp;
  uint8_t* ovf;
  int ps;
  int* nact;             // shared-memory action counter (initial / final value)
  int* serr;             // shared: an error was raised (checked between functions)
  int* snpods;           // shared copy of *w.n_pods for the whole commit
  long long* scounter;   // shared copy of *w.counter
  uint32_t* skey;        // shared argmin keys per GPU: npods > 0 ? occupancy << 18 | rank : ~0
                         // (null: scan the summaries)
  const uint32_t* smask;  // shared copy of w.sm_mask (the sm rows phase A2 tabulated)
  // the action / pod / id counters in registers while the warp commits (every lane holds
  // the same value: updates are warp-uniform), loaded from and stored back to the shared
  // copies above by load_counters / store_counters
  mutable int nact_r = 0, npods_r = 0;
  mutable long long counter_r = 0;

  __device__ void load_counters() const {
    nact_r = *nact;
    npods_r = *snpods;
    counter_r = *scounter;
  }
  __device__ void store_counters() const {
    __syncwarp();
    if (lane == 0) {
      *nact = nact_r;
      *snpods = npods_r;
      *scounter = counter_r;
    }
    __syncwarp();
  }

  // lane-0 code: refresh GPU g's argmin key after its pod count / occupancy changed
  __device__ void rekey0(int g) const {
    if (skey != nullptr)
      skey[g] = w.g_npods[g] > 0 ? (uint32_t(w.g_hgo[g]) << 18) | uint32_t(g) : ~0u;
  }

  // x / delta for 0 <= x <= 100 (delta is 1 on the full grid: no integer division there)
  __device__ __forceinline__ int div_d(int x) const {
    return w.delta == 1 ? x : x / w.delta;
  }

  __device__ uint64_t* parts(int g) const {
    return ovf[g] ? w.g_parts + int64_t(g) * kPartCap : sp + int64_t(g) * ps;
  }

  // lane-0 code: record the first error (global, for the host) and stop the commit
  __device__ void fail0(int code, int f) const {
    set_err(w, code, f);
    *serr = 1;
  }

  // before appending entry n to GPU g: move a full shared-memory list to global memory
  __device__ void make_room(int g, int n) const {
    if (!ovf[g] && n >= ps) {
      uint64_t* dst = w.g_parts + int64_t(g) * kPartCap;
      for (int i = 0; i < n; ++i) dst[i] = sp[int64_t(g) * ps + i];
      ovf[g] = 1;
    }
  }

  // position of the partition with this uid in list P of n entries (partition_of,
  // core.py:148-158)
  __device__ int find_part_in(const uint64_t* P, int n, uint32_t uid) const {
    unsigned pos = 1u << 30;
    for (int i = lane; i < n; i += 32)
      if (part_uid(P[i]) == uid) pos = min(pos, unsigned(i));
    return int(__reduce_min_sync(0xffffffffu, pos));
  }

  __device__ int find_part(int g, uint32_t uid) const {
    return find_part_in(parts(g), w.g_nparts[g], uid);
  }

  // find_part with a position hint (checked by one load of the hinted entry); P, n: the
  // GPU's list, fetched once by the caller
  // (the entry is returned too: the hint's load is the entry, no second read)
  __device__ int find_part_hint(const uint64_t* P, int n, uint32_t uid, int hint,
                                uint64_t& e) const {
    if (hint >= 0 && hint < n) {
      e = P[hint];
      if (part_uid(e) == uid) return hint;
    }
    const int pos = find_part_in(P, n, uid);
    e = P[pos];
    return pos;
  }

  __device__ void set_entry(uint64_t* P, int pos, uint64_t e) const {
    __syncwarp();
    if (lane == 0) P[pos] = e;
    __syncwarp();
  }

  // change_quota (allocator.py:111-125) + occupancy bookkeeping, partition position known;
  // P: GPU g's list, e: its entry at pos (as read by the caller)
  __device__ void change_quota_at(uint64_t* P, uint64_t e, int p, int g, int pos, int s,
                                  int old_q, int new_q) const {
    const int delta = new_q - old_q;
    set_entry(P, pos, part_pack(part_sm(e), part_alloc(e) + delta, part_npods(e), part_uid(e)));
    if (lane == 0) {
      const int h1 = w.g_hgo[g] + s * delta;
      w.g_hgo[g] = h1;
      if (skey != nullptr) skey[g] = (uint32_t(h1) << 18) | uint32_t(g);  // the pod is resident
      w.p_q[p] = new_q;
    }
    __syncwarp();
  }

  // place_pod (allocator.py:85-108): join the first same-sm partition with headroom, else
  // append a new partition
  __device__ void place(int p, int g, int s, int q) const {
    uint64_t* P = parts(g);
    const int n = w.g_nparts[g];
    unsigned upos = 1u << 30;
    for (int i = lane; i < n; i += 32)
      if (part_sm(P[i]) == s && 100 - part_alloc(P[i]) >= q) upos = min(upos, unsigned(i));
    const int pos = int(__reduce_min_sync(0xffffffffu, upos));
    if (lane == 0) {
      if (pos == (1 << 30)) {
        if (n >= kPartCap || w.g_freesm[g] < s) {
          fail0(RAPP_E_PLACEMENT, -1);
        } else {
          make_room(g, n);
          P = parts(g);
          const uint32_t uid = w.g_nextuid[g]++;
          P[n] = part_pack(s, q, 1, uid);
          w.g_nparts[g] = n + 1;
          w.g_freesm[g] -= s;
          w.p_puid[p] = uid;
        }
      } else {
        const uint64_t e = P[pos];
        P[pos] = part_pack(part_sm(e), part_alloc(e) + q, part_npods(e) + 1, part_uid(e));
        w.p_puid[p] = part_uid(e);
      }
      w.p_gpu[p] = g;
      w.g_npods[g] += 1;
      w.g_hgo[g] += s * q;
      rekey0(g);
    }
    __syncwarp();
  }

  // place() right after best_slot(g) (nothing changed g's list since): the lanes still hold
  // the entries of a list of <= 32 partitions, so the join search is one ballot
  __device__ void place_known(int p, int g, int s, int q, uint64_t e0, int n,
                              uint64_t* P) const {
    if (n > 32) {
      place(p, g, s, q);
      return;
    }
    const unsigned hit =
        __ballot_sync(0xffffffffu, lane < n && part_sm(e0) == s && 100 - part_alloc(e0) >= q);
    const int pos = hit ? __ffs(hit) - 1 : -1;
    const uint64_t e = __shfl_sync(0xffffffffu, e0, pos < 0 ? 0 : pos);
    __syncwarp();  // every lane's reads of the list and the argmin keys precede the update
    if (lane == 0) {
      if (pos < 0) {
        if (n >= kPartCap || w.g_freesm[g] < s) {
          fail0(RAPP_E_PLACEMENT, -1);
        } else {
          make_room(g, n);
          P = parts(g);
          const uint32_t uid = w.g_nextuid[g]++;
          P[n] = part_pack(s, q, 1, uid);
          w.g_nparts[g] = n + 1;
          w.g_freesm[g] -= s;
          w.p_puid[p] = uid;
        }
      } else {
        P[pos] = part_pack(part_sm(e), part_alloc(e) + q, part_npods(e) + 1, part_uid(e));
        w.p_puid[p] = part_uid(e);
      }
      w.p_gpu[p] = g;
      const int np1 = w.g_npods[g] + 1;
      const int h1 = w.g_hgo[g] + s * q;
      w.g_npods[g] = np1;
      w.g_hgo[g] = h1;
      if (skey != nullptr) skey[g] = (uint32_t(h1) << 18) | uint32_t(g);
    }
    __syncwarp();
  }

  // release_pod (allocator.py:128-139): an emptied partition leaves the list (list.remove)
  __device__ void release(int p, int f, int g, uint32_t uid, int s, int q) const {
    const int pos = find_part(g, uid);
    __syncwarp();
    if (lane == 0) {
      uint64_t* P = parts(g);
      const uint64_t e = P[pos];
      const int np = part_npods(e) - 1;
      if (np == 0) {
        const int n = w.g_nparts[g];
        for (int i = pos; i + 1 < n; ++i) P[i] = P[i + 1];
        w.g_nparts[g] = n - 1;
        w.g_freesm[g] += part_sm(e);
      } else {
        P[pos] = part_pack(part_sm(e), part_alloc(e) - q, np, part_uid(e));
      }
      w.g_npods[g] -= 1;
      w.g_hgo[g] -= s * q;
      rekey0(g);
      w.p_state[p] = kDead;
    }
    // drop from its function's pod list (swap with the last entry)
    if (f >= 0) {
      int* L = w.fn_pods + f * kMaxPods;
      const int n2 = w.fn_npods[f];
      unsigned uat = 1u << 30;
      for (int i = lane; i < n2; i += 32)
        if (L[i] == p) uat = min(uat, unsigned(i));
      const int at = int(__reduce_min_sync(0xffffffffu, uat));
      if (lane == 0) {
        if (at < n2) L[at] = L[n2 - 1];
        w.fn_npods[f] = n2 - 1;
      }
    }
    __syncwarp();
  }

  __device__ void emit(int f, int kind, int b, int s, int q, int pod, int gpu, int rel) const {
    const int i = nact_r++;
    if (lane == 0) w.actions[i] = rapp_action{f, kind, b, s, q, pod, gpu, rel};
  }

  // new COLD_STARTING pod pod-%06d (sim.py:337-340, 505-516); nothing in this tick reads the
  // new pod's id string, so only its counter value is recorded here.
  // npods: the function's pod count (kept by the caller across its new pods).
  __device__ int new_pod(int f, int b, int s, int q, double now, int& npods) const {
    int p = npods_r++;
    const bool full = p >= w.pod_cap || npods >= kMaxPods;
    const long long c = full ? -1 : counter_r++;
    if (full) p = -1;
    if (lane == 0) {
      if (full) {
        fail0(RAPP_E_ARG, f);
      } else {
        w.p_ctr[p] = c;  // the id string is formatted later (format_pending)
        w.p_fn[p] = f;
        w.p_b[p] = b;
        w.p_s[p] = s;
        w.p_q[p] = q;
        w.p_state[p] = kCold;
        w.p_ready[p] = __dadd_rn(now, w.cold_start);
        w.fn_pods[f * kMaxPods + npods] = p;
        w.fn_npods[f] = npods + 1;
      }
    }
    __syncwarp();
    if (p >= 0) ++npods;
    return p;
  }

  // lowest (occupancy, rank) among used GPUs (autoscaler.py:139-141); occupancy compares
  // as the integer sum(sm*quota): /10000.0 is monotone and injective on 0..10000
  __device__ int argmin_used() const {
    // occupancy <= 100*100 per GPU, so (occupancy, rank) packs into 32 bits for up to 2^18
    // GPUs: one scan and one warp min-reduction
    if (skey != nullptr) {  // maintained keys: one shared-memory word per GPU
      // 16 independent loads per lane in flight: one shared-memory round trip for up to
      // 512 GPUs (a plain strided loop waits on each)
      unsigned best = ~0u;
      for (int g0 = 0; g0 < w.G; g0 += 512) {
        unsigned k[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int g = g0 + u * 32 + lane;
          k[u] = g < w.G ? skey[g] : ~0u;
        }
        // pairwise tree (4 levels) rather than a 16-long dependent chain
#pragma unroll
        for (int h = 8; h > 0; h >>= 1)
#pragma unroll
          for (int u = 0; u < h; ++u) k[u] = min(k[u], k[u + h]);
        best = min(best, k[0]);
      }
      best = __reduce_min_sync(0xffffffffu, best);
      return best == ~0u ? -1 : int(best & ((1u << 18) - 1));
    }
    if (w.G <= (1 << 18)) {
      unsigned best = ~0u;
      for (int g = lane; g < w.G; g += 32)
        if (w.g_npods[g] > 0) best = min(best, (unsigned(w.g_hgo[g]) << 18) | unsigned(g));
      best = __reduce_min_sync(0xffffffffu, best);
      return best == ~0u ? -1 : int(best & ((1u << 18) - 1));
    }
    long long best = LLONG_MAX;
    for (int g = lane; g < w.G; g += 32)
      if (w.g_npods[g] > 0) {
        const long long k = (long long)w.g_hgo[g] << 32 | g;
        best = k < best ? k : best;
      }
    for (int o = 16; o > 0; o >>= 1) {
      const long long x = __shfl_xor_sync(0xffffffffu, best, o);
      best = x < best ? x : best;
    }
    return best == LLONG_MAX ? -1 : int(best & 0xFFFFFFFF);
  }

  __device__ int first_free() const {
    unsigned best = 1u << 30;
    for (int g = lane; g < w.G; g += 32)
      if (w.g_npods[g] == 0) {
        best = unsigned(g);
        break;  // g ascends within a lane
      }
    best = __reduce_min_sync(0xffffffffu, best);
    return best == (1u << 30) ? -1 : int(best);
  }

  // max_avail_quota_and_sm (allocator.py:26-52): max of (sm*hr, sm, join=1) over
  // partitions with headroom (first wins ties), then (free*100, free, 0) if strictly greater
  // e0 / n: this lane's entry of the list (lane < n) and the list length, for place_known
  __device__ void best_slot(int g, int& sm, int& q, uint64_t& e0, int& n, uint64_t*& P) const {
    P = parts(g);
    n = w.g_nparts[g];
    const int free_sm = w.g_freesm[g];
    e0 = lane < n ? P[lane] : 0;
    // key: prod (15 bits) | sm (8) | (255 - pos) (8): max key = max (prod, sm), first pos
    // (prod <= 10^4 -> the key fits 31 bits: one redux instead of a shuffle tree)
    unsigned ukey = 0;
    for (int i = lane; i < n; i += 32) {
      const uint64_t e = i == lane ? e0 : P[i];
      const int hr = 100 - part_alloc(e);
      if (hr > 0) {
        const unsigned k = (unsigned(part_sm(e) * hr) << 16) | (unsigned(part_sm(e)) << 8) |
                           unsigned(255 - i);
        ukey = k > ukey ? k : ukey;
      }
    }
    ukey = __reduce_max_sync(0xffffffffu, ukey);
    const long long best = ukey == 0 ? -1 : (long long)ukey;
    sm = 0;
    q = 0;
    long long bprod = -1, bsm = -1, bjoin = -1;
    if (best >= 0) {  // (sm, headroom) of the best partition: a lane still holds it
      const int pos = 255 - int(ukey & 0xFF);
      const uint64_t eb = __shfl_sync(0xffffffffu, e0, pos & 31);
      const uint64_t e = pos < 32 ? eb : P[pos];
      sm = part_sm(e);
      q = 100 - part_alloc(e);
      bprod = (long long)sm * q;
      bsm = sm;
      bjoin = 1;
    }
    if (free_sm > 0) {
      const long long fp = (long long)free_sm * 100;
      const bool greater = best < 0 || fp > bprod || (fp == bprod && (free_sm > bsm ||
                           (free_sm == bsm && 0 > bjoin)));
      if (greater) {
        sm = free_sm;
        q = 100;
      }
    }
  }

  // most_efficient_config(target) via the key-sorted prefix-max index: the first lattice
  // point (in (s*q, s, q, b) order) with prefix max >= min(target, max rps).  Each round
  // probes 1024 evenly spaced entries of the candidate range (32 independent loads per
  // lane, one memory round trip) and keeps the one bucket that holds the answer, so a
  // 291,200-point full-grid lattice takes two rounds.
  __device__ void mec(int f, double target, int& b, int& s, int& q) const {
    const double* pm = w.pmax + w.fn_lat_off[f];
    const int64_t L = w.fn_lat_len[f];
    const double top = pm[L - 1];
    const double t = target <= top ? target : top;  // target > top -> max-rps fallback
    // invariant: the answer lies in [lo, hi] (pm non-decreasing, pm[hi] >= t)
    int64_t lo = 0, hi = L - 1;
    // opt-in SLO: pm is the prefix max over SLO-compliant points only; with no compliant
    // point meeting the target the answer is the reference's fallback over the whole
    // lattice, precomputed (k_index_fb)
    const int64_t fb = (w.fn_fb != nullptr && !(target <= top)) ? w.fn_fb[f] : -1;
    if (fb >= 0) lo = fb;
    while (fb < 0) {
      const int64_t len = hi - lo + 1;
      const int64_t step = (len + 1023) / 1024;  // probes lo + step*j, j < 1024
      bool ge[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int64_t pos = lo + step * (int64_t(lane) * 32 + u);
        ge[u] = pos > hi || pm[pos] >= t;
      }
      // first probe of this lane that is >= t (32: none): lowest set bit of the probe mask,
      // the mask ORed as a tree
      unsigned bits[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) bits[u] = ge[u] ? 1u << u : 0u;
#pragma unroll
      for (int h = 16; h > 0; h >>= 1)
#pragma unroll
        for (int u = 0; u < h; ++u) bits[u] |= bits[u + h];
      const int first = bits[0] ? __ffs(bits[0]) - 1 : 32;
      const unsigned mask = __ballot_sync(0xffffffffu, first < 32);
      const int l0 = __ffs(mask) - 1;  // lane of the first >= probe (pm[hi] >= t: exists)
      const int u0 = __shfl_sync(0xffffffffu, first, l0);
      const int64_t jfirst = int64_t(l0) * 32 + u0;
      if (jfirst == 0) break;  // pm[lo] >= t: the answer is lo
      if (step == 1) {
        lo = lo + jfirst;
        break;
      }
      const int64_t ph = lo + step * jfirst;
      hi = ph < hi ? ph : hi;
      if (jfirst > 0) lo = lo + step * (jfirst - 1) + 1;
    }
    const int64_t idx = lo;
    const int nb = w.fn_nb[f];
    const int pair = w.pairs[w.fn_pairs_off[f] + int(idx / nb)];
    const TableDesc td = w.tds[w.fn_table[f]];
    b = int(w.blist[w.fn_boff[f] + idx % nb]);
    s = int(w.pool[td.off + td.os + (pair >> 16)]);
    q = pair & 0xFFFF;
  }

  // Function header + its first pod (scale-up: sorted[0]; scale-down: the first staged
  // action's pod), prefetched for 32 functions at once by the commit loop: nothing here can
  // change before the function's own turn in the tick.
  using Pre = CommitPre;

  __device__ Pre prefetch(int f) const { return prefetch_of(w, f); }

  __device__ static Pre prefetch_of(const World& w, int f) {
    Pre r{};
    r.p0 = -1;
    if (f >= w.F) return r;
    const int cls = w.cls[f];
    if (cls == kUp && w.policy == 0) {
      r.gap0 = w.gap0[f];
      r.m = w.nsorted[f];
      r.bref = w.bref[f];
      r.brefok = w.bref_ok[f];
      r.npods = w.fn_npods[f];
      r.sav0 = w.spec_avail[f * kMaxPods];
      r.sk0 = w.spec_k[f * kMaxPods];
      r.sg0 = w.spec_gain[f * kMaxPods];
      r.kd0 = w.row_kd[f * kMaxPods];
      r.kg0 = w.spec_kg[f * kMaxPods];
      r.p0 = r.m > 0 ? w.sorted[f * kMaxPods] : -1;
    } else if (cls == kDown) {
      r.nd = w.ndown[f];
      r.stamp = w.stamp[f];
      if (r.nd > 0) {
        const DownAct a = w.down[f * kMaxPods];
        r.dkind = a.kind;
        r.dquota = a.quota;
        r.p0 = a.pod;
      }
    }
    if (r.p0 >= 0) {
      const int p = r.p0;
      r.st0 = w.p_state[p];
      r.gpu0 = w.p_gpu[p];
      r.uid0 = w.p_puid[p];
      r.q0 = w.p_q[p];
      r.b0 = w.p_b[p];
      r.s0 = w.p_s[p];
      if (cls == kDown) r.didle = w.p_idle[p];
      // partitions keep their order except for removals, so the tick-start position is
      // almost always still right; the committer validates it with one load
      const uint64_t* P = w.g_parts + int64_t(r.gpu0) * kPartCap;
      const int n = w.g_nparts[r.gpu0];
      r.pos0 = -1;
      for (int i = 0; i < n; ++i)
        if (part_uid(P[i]) == r.uid0) {
          r.pos0 = i;
          break;
        }
    }
    return r;
  }

  __device__ static Pre bcast(const Pre& x, int src) {
    Pre r;
    r.gap0 = __shfl_sync(0xffffffffu, x.gap0, src);
    r.sg0 = __shfl_sync(0xffffffffu, x.sg0, src);
    r.m = __shfl_sync(0xffffffffu, x.m, src);
    r.p0 = __shfl_sync(0xffffffffu, x.p0, src);
    r.st0 = __shfl_sync(0xffffffffu, x.st0, src);
    r.gpu0 = __shfl_sync(0xffffffffu, x.gpu0, src);
    r.q0 = __shfl_sync(0xffffffffu, x.q0, src);
    r.b0 = __shfl_sync(0xffffffffu, x.b0, src);
    r.s0 = __shfl_sync(0xffffffffu, x.s0, src);
    r.sav0 = __shfl_sync(0xffffffffu, x.sav0, src);
    r.sk0 = __shfl_sync(0xffffffffu, x.sk0, src);
    r.bref = __shfl_sync(0xffffffffu, x.bref, src);
    r.brefok = __shfl_sync(0xffffffffu, x.brefok, src);
    r.npods = __shfl_sync(0xffffffffu, x.npods, src);
    r.kd0 = __shfl_sync(0xffffffffu, x.kd0, src);
    r.kg0 = __shfl_sync(0xffffffffu, x.kg0, src);
    r.nd = __shfl_sync(0xffffffffu, x.nd, src);
    r.dkind = __shfl_sync(0xffffffffu, x.dkind, src);
    r.dquota = __shfl_sync(0xffffffffu, x.dquota, src);
    r.didle = __shfl_sync(0xffffffffu, x.didle, src);
    r.stamp = __shfl_sync(0xffffffffu, x.stamp, src);
    r.uid0 = __shfl_sync(0xffffffffu, x.uid0, src);
    return r;
  }

  // srow0: the function's first-pod quota row staged in shared memory (see k_tick_commit)
  __device__ void scale_up(int f, double now, const Pre& pre, const double* srow0) const {
    TPROF_T0();
    const int d = w.delta;
    double gap = pre.gap0;
    const int m = pre.m;
    int npods = pre.npods;
    const int* srt = w.sorted + f * kMaxPods;
    const double* rows = w.rows + int64_t(f) * kMaxPods * kRow;
    // vertical first, largest sm first (autoscaler.py:115-133)
    bool spec_ok = true;
    for (int j = 0; j < m; ++j) {
      if (!(gap > 0.0)) break;
      const int p = j == 0 ? pre.p0 : srt[j];
      if ((j == 0 ? pre.st0 : w.p_state[p]) != kRunning) continue;
      const int g = j == 0 ? pre.gpu0 : w.p_gpu[p];
      uint64_t* const P = parts(g);
      const int np = w.g_nparts[g];
      int pos;
      uint64_t ent;
      if (j == 0) {
        pos = find_part_hint(P, np, pre.uid0, pre.pos0, ent);
      } else {
        pos = find_part_in(P, np, w.p_puid[p]);
        ent = P[pos];
      }
      const int q0 = j == 0 ? pre.q0 : w.p_q[p];
      const int avail = q0 + (100 - part_alloc(ent));
      TPROF_ACC(5);  // headroom lookup
      int kstar = -1;
      double gain = 0.0;
      const int sav = j == 0 ? pre.sav0 : w.spec_avail[f * kMaxPods + j];
      if (spec_ok && sav == avail) {
        kstar = j == 0 ? pre.sk0 : w.spec_k[f * kMaxPods + j];  // phase A's walk
        gain = j == 0 ? pre.sg0 : w.spec_gain[f * kMaxPods + j];
      } else if (spec_ok) {
        // only the headroom differs from phase A's (the gap is the one it assumed): the
        // walk stops at min(kq, kg) — kq = (avail - q0) / d from the quota bound, kg the
        // first gap-closing step phase A recorded (autoscaler.py:124-131)
        spec_ok = false;  // later pods start from a different gap: walk them here
        const int kd = j == 0 ? pre.kd0 : w.row_kd[f * kMaxPods + j];
        const double* row = j == 0 ? srow0 + kd : rows + j * kRow + kd;
        const int kg = j == 0 ? pre.kg0 : w.spec_kg[f * kMaxPods + j];
        const int kq = div_d(avail - q0);
        kstar = kg < kq ? kg : kq;
        if (kstar > 0) gain = __dsub_rn(row[kstar], row[0]);
      } else {
        const int kd = j == 0 ? pre.kd0 : w.row_kd[f * kMaxPods + j];
        // row[k] = thr at q0 + k*d
        const double* row = j == 0 ? srow0 + kd : rows + j * kRow + kd;
        // k* = first k >= 0 with q0+(k+1)d > avail or !(gap - gain_k > 0), gain_0 = 0.
        // k <= (100 - q0) / d < 128: every row value the walk may read is loaded in one
        // round (lane l holds k = l, l+32, l+64, l+96), then 4 ballots find k*.
        const double cur = row[0];
        double rk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = u * 32 + lane;
          rk[u] = k > 0 && q0 + k * d <= avail ? row[k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = u * 32 + lane;
          bool stop;
          if (q0 + (k + 1) * d > avail) {
            stop = true;
          } else {
            const double gk = k == 0 ? 0.0 : __dsub_rn(rk[u], cur);
            stop = !(__dsub_rn(gap, gk) > 0.0);
          }
          const unsigned mask = __ballot_sync(0xffffffffu, stop);
          if (mask && kstar < 0) {
            const int l = __ffs(mask) - 1;
            kstar = u * 32 + l;
            const double rs = __shfl_sync(0xffffffffu, rk[u], l);
            if (kstar > 0) gain = __dsub_rn(rs, cur);
          }
        }
      }
      TPROF_ACC(1);  // spec check / re-walk
      if (kstar > 0) {
        const int nq = q0 + kstar * d;
        const int s = j == 0 ? pre.s0 : w.p_s[p];
        change_quota_at(P, ent, p, g, pos, s, q0, nq);
        emit(f, kVUp, j == 0 ? pre.b0 : w.p_b[p], s, nq, p, g, 0);
        gap = __dsub_rn(gap, gain);
      }
      TPROF_ACC(7);  // change_quota + emit
    }
    TPROF_ACC(1);
#ifdef RAPP_TICK_PROF
    if (lane == 0) {
      s_tprof[25] += 1;          // generic scale-up commits
      s_tprof[26] += gap > 0.0;  // ... that go on to the horizontal branch
    }
#endif
    scale_up_h(f, now, pre, gap, npods);
  }

  // the horizontal part of _scale_up (autoscaler.py:137-165) for the gap the walk left
  __device__ void scale_up_h(int f, double now, const Pre& pre, double gap, int npods) const {
    TPROF_T0();
    const int d = w.delta;
    const int bref = pre.bref;
    // one pod on the used GPU with the lowest occupancy (autoscaler.py:137-152)
    if (gap > 0.0) {
      const int g = argmin_used();
      TPROF_ACC(8);
      if (g >= 0) {
        // The slot is usually a new partition on g's unallocated share (its sm * 100 beats
        // every join): that throughput row is requested now, while best_slot runs, and
        // used when best_slot agrees.  Every step's value is loaded (steps past qmax are
        // never read).
        double tv[4];
        int tv_sm = 0;
#ifdef RAPP_TICK_TSPEC  // measured: +-2% (tools/ab_tickprof.sh), off
        if (pre.brefok) {
          const int fs = w.g_freesm[g];
          if (fs > 0 && (!kMasked || ((smask[(fs - 1) >> 5] >> ((fs - 1) & 31)) & 1u))) {
            const double* T = w.tgrid + (int64_t(f) * 100 + (fs - 1)) * 100;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int qq = (u * 32 + lane + 1) * d;
              tv[u] = qq <= 100 ? T[qq - 1] : 0.0;
            }
            tv_sm = fs;
          }
        }
#endif
        int sm, qmax, nl;
        uint64_t el;
        uint64_t* Pl;
        best_slot(g, sm, qmax, el, nl, Pl);
        TPROF_ACC(9);
        if (sm > 0 && qmax > 0) {
          if (!pre.brefok) {
            if (lane == 0) fail0(RAPP_E_VALUE, f);
            __syncwarp();
            return;
          }
          // every throughput the branch may read, in one round of independent loads:
          // lanes hold the quota steps (u*32 + lane + 1)*d <= qmax, u < 4 (d >= 1) —
          // from phase A2's grid when it tabulated this sm, else evaluated here
          if (sm == tv_sm) {
            // prefetched above
          } else if (!kMasked || ((smask[(sm - 1) >> 5] >> ((sm - 1) & 31)) & 1u)) {
            const double* T = w.tgrid + (int64_t(f) * 100 + (sm - 1)) * 100;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int qq = (u * 32 + lane + 1) * d;
              tv[u] = qq <= qmax ? T[qq - 1] : 0.0;
            }
          } else {  // interp3 from phase A2's brackets (the same doubles as locate())
#ifdef RAPP_TICK_PROF
            if (lane == 0) s_tprof[28] += 1;  // rows evaluated here (sm outside the mask)
#endif
            const Row4 r = bracket_row(w, f, bref, sm, qmax, d, lane);
#pragma unroll
            for (int u = 0; u < 4; ++u) tv[u] = r.v[u];
          }
          double cmax;
          const int qd = div_d(qmax);
          if (qd * d == qmax) {
            const int kq = qd - 1;  // the step index of qmax
            // every lane picks the register that holds step kq, then one shuffle
            const int u = kq >> 5;
            const double src = u == 0 ? tv[0] : u == 1 ? tv[1] : u == 2 ? tv[2] : tv[3];
            cmax = __shfl_sync(0xffffffffu, src, kq & 31);
          } else {  // max_quota_capability at an off-step quota (autoscaler.py:144)
            cmax = lane == 0 ? thr_at(w, f, double(bref), double(sm), double(qmax)) : 0.0;
            cmax = __shfl_sync(0xffffffffu, cmax, 0);
          }
#ifdef RAPP_TICK_PROF
          // diagnostics: the row read's own latency (cmax depends on it), how often the slot
          // is a new partition on the GPU's unallocated share, and the step count
          if (lane == 0) {
            s_tprof[22] += (unsigned long long)((long long)clock64() - _tp0) *
                           (unsigned long long)(cmax == cmax);
            s_tprof[23] += sm == w.g_freesm[g] && qmax == 100;
            s_tprof[24] += 1;
          }
#endif
          if (cmax > gap) {
            // _covering_quota (autoscaler.py:168-175): first multiple of d <= qmax with
            // throughput >= gap, else qmax
            int quota = qmax;
            double tq = cmax;
            // the four steps' ballots are independent: all issued, then the first hit
            unsigned mk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int qq = (u * 32 + lane + 1) * d;
              mk[u] = __ballot_sync(0xffffffffu, qq <= qmax && tv[u] >= gap);
            }
            const int uh = mk[0] ? 0 : mk[1] ? 1 : mk[2] ? 2 : mk[3] ? 3 : -1;
            if (uh >= 0) {
              const unsigned mask = mk[uh];
              const int l = __ffs(mask) - 1;
              quota = (uh * 32 + l + 1) * d;
              const double src = uh == 0 ? tv[0] : uh == 1 ? tv[1] : uh == 2 ? tv[2] : tv[3];
              tq = __shfl_sync(0xffffffffu, src, l);
            }
            TPROF_ACC(10);  // T loads + covering quota
            const int p = new_pod(f, bref, sm, quota, now, npods);
            TPROF_ACC(11);  // new_pod
            if (p < 0) return;
            place_known(p, g, sm, quota, el, nl, Pl);
            TPROF_ACC(12);  // place
            emit(f, kHUp, bref, sm, quota, p, g, 0);
            TPROF_ACC(13);  // emit
            gap = __dsub_rn(gap, tq);  // == T[quota] on a step, cmax at the off-step qmax
          }
        }
      }
    }
    TPROF_ACC(2);  // used-GPU branch
    // one pod on a fresh GPU at the most cost-efficient configuration (autoscaler.py:155-165)
    if (gap > 0.0) {
      const int g = first_free();
      if (g >= 0) {
        int b, s, q;
        mec(f, gap, b, s, q);
        const int p = new_pod(f, b, s, q, now, npods);
        if (p < 0) return;
        place(p, g, s, q);
        emit(f, kHUp, b, s, q, p, g, 0);
      }
    }
    TPROF_ACC(3);  // fresh-GPU branch
  }

  // check_placement (allocator.py:63-82) == nullptr: a joinable same-sm partition with
  // headroom >= q, or an unallocated share >= sm
  __device__ bool legal(int g, int s, int q) const {
    if (s < 1 || s > 100 || q < 1 || q > 100) return false;
    if (w.g_freesm[g] >= s) return true;
    const uint64_t* P = parts(g);
    const int n = w.g_nparts[g];
    for (int i = 0; i < n; ++i)
      if (part_sm(P[i]) == s && 100 - part_alloc(P[i]) >= q) return true;
    return false;
  }

  // _pick_gpu (policies.py:128-141): the lowest (occupancy, id) used GPU that can take the
  // shape, else the first free GPU that can, else none
  __device__ int pick_gpu(int s, int q) const {
    long long best = LLONG_MAX;
    int first_free = 1 << 30;
    for (int g = lane; g < w.G; g += 32) {
      if (!legal(g, s, q)) continue;
      if (w.g_npods[g] > 0) {
        const long long k = (long long)w.g_hgo[g] << 32 | g;
        best = k < best ? k : best;
      } else {
        first_free = min(first_free, g);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const long long x = __shfl_xor_sync(0xffffffffu, best, o);
      best = x < best ? x : best;
      first_free = min(first_free, __shfl_xor_sync(0xffffffffu, first_free, o));
    }
    if (best != LLONG_MAX) return int(best & 0xFFFFFFFF);
    return first_free == (1 << 30) ? -1 : first_free;
  }

  // _add_replicas (policies.py:107-126)
  __device__ void replica_up(int f, double now) const {
    const int* shape = w.fn_shape + 3 * f;
    const int want = w.wanted[f];
    int npods = w.fn_npods[f];
    for (int i = 0; i < want; ++i) {
      const int g = pick_gpu(shape[1], shape[2]);
      if (g < 0) break;  // cluster saturated for this shape
      const int p = new_pod(f, shape[0], shape[1], shape[2], now, npods);
      if (p < 0) return;
      place(p, g, shape[1], shape[2]);
      emit(f, kHUp, shape[0], shape[1], shape[2], p, g, 0);
    }
  }

  // Commits a run of straight-line functions (FastRec) at once, one per lane.  `cand`: the
  // active lanes from the next function up to (excluding) the first active function that is
  // not straight-line, in sorted order.  Lane l joins the run when every partition it
  // validates still has its tick-start allocation and is not written by a lower lane of the
  // run — exactly the conditions under which the sequential commit would take phase A's
  // walk verbatim — and every lane below it joined too.  Returns the lanes committed (their
  // changes applied, actions emitted in function order); 0 leaves the first one to the
  // sequential path.  htab: conflict marks (epoch << 5 | 31 - lane) by partition hash.
  // dead: the lanes whose own validation failed (their partitions changed since phase A;
  // the sequential path redoes them).
  __device__ unsigned fast_run(int base, unsigned cand, const FastRec& r, int stamp,
                               double now, uint32_t* htab, uint32_t epoch,
                               unsigned& dead) const {
    const bool in = (cand >> lane) & 1;
    // every field up front (independent shared loads, one latency)
    const int n = r.n, kind = r.kind;
    FastStep st[kFastSteps];
#pragma unroll
    for (int k = 0; k < kFastSteps; ++k) st[k] = r.st[k];
    bool ok = in;
    uint32_t pa[kFastSteps];  // shared address of the entry's low word
    bool wr[kFastSteps];
#pragma unroll
    for (int k = 0; k < kFastSteps; ++k) {
      const bool have = in && k < n;
      const int g = have ? st[k].g : 0;
      const int pos = have && st[k].pos < ps ? st[k].pos : 0;
      pa[k] = (uint32_t)__cvta_generic_to_shared(sp + int64_t(g) * ps + pos);
      const uint64_t e = lds_u64(pa[k]);
      const int np = lds_s32(w.g_nparts + g);
      const int o = ovf[g];
      // shared-memory lists only; the position and uid still those of phase A
      const bool good = o == 0 && st[k].pos < np && st[k].pos < ps &&
                        part_uid(e) == st[k].uid &&
                        (st[k].alloc0 < 0 || part_alloc(e) == st[k].alloc0);
      if (have && !good) ok = false;
      wr[k] = have && st[k].qnew != st[k].qold;
    }
    dead = cand & ~__ballot_sync(0xffffffffu, ok);
    if (cand & (cand - 1)) {  // more than one lane: conflicts with lower lanes' writes
      const uint32_t mark = (epoch << 5) | uint32_t(31 - lane);
#pragma unroll
      for (int k = 0; k < kFastSteps; ++k)
        if (ok && wr[k]) atomicMax(htab + fast_hash(st[k].g, st[k].pos), mark);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kFastSteps; ++k)
        if (ok && k < n && st[k].alloc0 >= 0) {
          const uint32_t v = htab[fast_hash(st[k].g, st[k].pos)];
          if ((v >> 5) == epoch && int(31 - (v & 31)) < lane) ok = false;
        }
    }
    const unsigned bad = cand & ~__ballot_sync(0xffffffffu, ok);
    const unsigned run = bad ? cand & ((1u << (__ffs(bad) - 1)) - 1) : cand;
#ifdef RAPP_TICK_PROF
    if (lane == 0) s_tprof[14] += __popc(run);
#endif
    if (run == 0) return 0;
    const bool mine = (run >> lane) & 1;
    int cnt = 0;
    if (mine) {
#pragma unroll
      for (int k = 0; k < kFastSteps; ++k)
        if (wr[k]) {
          const int delta = st[k].qnew - st[k].qold;
          // shared-memory reductions: the alloc field (bits 8..15 of the entry's low word,
          // 0..100 before and after, so nothing carries) and the GPU's occupancy
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(pa[k]), "r"(uint32_t(delta * 256))
                       : "memory");
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(
              (uint32_t)__cvta_generic_to_shared(w.g_hgo + st[k].g)), "r"(st[k].s * delta)
                       : "memory");
          w.p_q[st[k].p] = st[k].qnew;
          ++cnt;
        }
    }
    const unsigned b1 = __ballot_sync(0xffffffffu, mine && cnt >= 1);
    const unsigned b2 = __ballot_sync(0xffffffffu, mine && cnt >= 2);
    const int at0 = nact_r;
    __syncwarp();  // every lane's reductions are done
    if (mine) {
      int at = at0 + __popc(b1 & ((1u << lane) - 1)) + __popc(b2 & ((1u << lane) - 1));
      const int f = base + lane;
#pragma unroll
      for (int k = 0; k < kFastSteps; ++k)
        if (wr[k]) {
          const int g = st[k].g;
          if (skey != nullptr)
            skey[g] = lds_s32(w.g_npods + g) > 0
                          ? (uint32_t(lds_s32(w.g_hgo + g)) << 18) | uint32_t(g) : ~0u;
          w.actions[at++] = rapp_action{f, kind == kFastDown ? kVDown : kVUp, st[k].b, st[k].s,
                                        st[k].qnew, st[k].p, g, 0};
        }
      if (stamp && kind == kFastDown) w.last_down[f] = now;
    }
    nact_r = at0 + __popc(b1) + __popc(b2);
    __syncwarp();
    return run;
  }

  __device__ void scale_down(int f, double now, const Pre& pre) const {
    TPROF_T0();
    const int na = pre.nd;
    const DownAct* acts = w.down + f * kMaxPods;
    for (int i = 0; i < na; ++i) {
      int kind, p, quota, g, b, s, q, idle;
      uint32_t uid;
      if (i == 0) {
        kind = pre.dkind;
        p = pre.p0;
        quota = pre.dquota;
        g = pre.gpu0;
        uid = pre.uid0;
        b = pre.b0;
        s = pre.s0;
        q = pre.q0;
        idle = pre.didle;
      } else {
        const DownAct a = acts[i];
        kind = a.kind;
        p = a.pod;
        quota = a.quota;
        g = w.p_gpu[p];
        uid = w.p_puid[p];
        b = w.p_b[p];
        s = w.p_s[p];
        q = w.p_q[p];
        idle = w.p_idle[p];
      }
      if (kind == kVDown) {
        uint64_t* const P = parts(g);
        const int np = w.g_nparts[g];
        int pos;
        uint64_t ent;
        if (i == 0) {
          pos = find_part_hint(P, np, uid, pre.pos0, ent);
        } else {
          pos = find_part_in(P, np, uid);
          ent = P[pos];
        }
        change_quota_at(P, ent, p, g, pos, s, q, quota);
        emit(f, kVDown, b, s, quota, p, g, 0);
      } else {
        if (lane == 0) w.p_state[p] = kDraining;
        __syncwarp();
        if (idle) release(p, f, g, uid, s, q);
        emit(f, kHDown, b, s, 0, p, g, idle ? 1 : 0);
      }
    }
    if (lane == 0 && pre.stamp) w.last_down[f] = now;
    __syncwarp();
    TPROF_ACC(4);
  }
};

// One warp.  The per-GPU summaries (pod count, occupancy, partition count, free SM share,
// next partition uid) live in shared memory for the whole tick when they fit: the
// used-GPU argmin and the first-free scan then read shared memory only.  Function classes
// are fetched 32 at a time and only active functions are visited, in sorted order.
#ifndef RAPP_TICK_HELPERS
#define RAPP_TICK_HELPERS 2
#endif
#ifndef RAPP_TICK_PREDEPTH
#define RAPP_TICK_PREDEPTH 4
#endif
constexpr int kHelpers = RAPP_TICK_HELPERS;     // helper warps filling the header ring
constexpr int kPreDepth = RAPP_TICK_PREDEPTH;   // batches of function headers in the ring
constexpr int kCommitThreads = 32 * (1 + kHelpers);

template <bool kMasked>
__global__ void __launch_bounds__(kCommitThreads) k_tick_commit(World w, double now, int smem_g,
                                                                int ps) {
  // dynamic shared layout: [row staging 2 x 32 x kRowStage doubles][5*G summaries]
  //                        [partition cache G*ps uint64 (8-aligned)][ovf G bytes]
  extern __shared__ __align__(16) int32_t smem_dyn[];
  double* s_rows = reinterpret_cast<double*>(smem_dyn);
  int32_t* sg = smem_dyn + 2 * 32 * kRowStage * 2;
  __shared__ int s_nact;
  const int lane = threadIdx.x & 31;
  // Warps 1..kHelpers are helpers: they read the headers of the next kPreDepth batches of
  // 32 functions (each function's own phase-A outputs and first pod — nothing an earlier
  // function of the tick can change) into a shared ring while warp 0 commits, helper h
  // taking batches h-1, h-1+kHelpers, ..., so warp 0 never waits on those dependent
  // global loads.
  __shared__ CommitPre s_pre[kPreDepth][32];
  __shared__ int s_pcls[kPreDepth][32];
  __shared__ FastRec s_fast[kPreDepth][32];
  __shared__ uint32_t s_htab[kFastHash];
  for (int i = threadIdx.x; i < kFastHash; i += blockDim.x) s_htab[i] = 0;
  // ring handoff by mbarriers (acquire/release, and visible to compute-sanitizer's
  // racecheck): full[slot] completes when all 32 helper lanes have written a batch into the
  // slot, empty[slot] when all 32 committing lanes are done with it
  __shared__ uint64_t s_full[kPreDepth], s_empty[kPreDepth];
  __shared__ volatile int s_stop;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kPreDepth; ++k) {
      mbar_init32(&s_full[k]);
      mbar_init32(&s_empty[k]);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_stop = 0;
  }
#ifdef RAPP_TICK_PROF
  const long long _pro0 = clock64();
#endif
  // The tick's cluster state into shared memory, by every warp (the helpers start their
  // ring after it).  Layout: [5*G summaries][partition cache G*ps uint64 (8-aligned)]
  // [ovf G bytes][argmin keys] (no summaries region when they live in global memory).
  const int G = w.G;
  uint64_t* sp = reinterpret_cast<uint64_t*>(sg + (smem_g ? ((5 * G + 1) & ~1) : 0));
  uint8_t* ovf = reinterpret_cast<uint8_t*>(sp + int64_t(G) * ps);
  uint32_t* skey = (smem_g && G <= (1 << 18))
                       ? reinterpret_cast<uint32_t*>(ovf + ((G + 3) & ~3)) : nullptr;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const int n = w.g_nparts[g];
    const bool cached = n <= ps && ps > 0;
    ovf[g] = cached ? 0 : 1;
    if (cached)
      for (int i = 0; i < n; ++i) sp[int64_t(g) * ps + i] = w.g_parts[int64_t(g) * kPartCap + i];
    if (smem_g) {
      const int np = w.g_npods[g], hgo = w.g_hgo[g];
      sg[g] = np;
      sg[G + g] = hgo;
      sg[2 * G + g] = n;
      sg[3 * G + g] = w.g_freesm[g];
      sg[4 * G + g] = int32_t(w.g_nextuid[g]);
      if (skey != nullptr) skey[g] = np > 0 ? (uint32_t(hgo) << 18) | uint32_t(g) : ~0u;
    }
  }
  // (the cluster state above is written only by commits and releases, never by the tick's
  // earlier kernels; everything below reads their outputs)
  pdl_wait();
  __syncthreads();
  if (threadIdx.x >= 32) {
    const int h = (threadIdx.x >> 5) - 1;
    bool quit = false;
    for (int b = h, base = 32 * h; base < w.F; b += kHelpers, base += 32 * kHelpers) {
      const int slot = b % kPreDepth, use = b / kPreDepth;
      if (use > 0) {  // the slot is free once the commit released batch b - depth
        while (true) {
          const bool got = mbar_try(&s_empty[slot], (use - 1) & 1);
          if (__all_sync(0xffffffffu, got)) break;
          if (__any_sync(0xffffffffu, s_stop != 0)) {
            quit = true;
            break;
          }
          __nanosleep(32);
        }
      }
      if (quit || __any_sync(0xffffffffu, s_stop != 0)) break;
      const int f = base + lane;
      const int cf = f < w.F ? w.cls[f] : kNone;
      s_pcls[slot][lane] = cf;
      s_pre[slot][lane] = CommitT<kMasked>::prefetch_of(w, f);
      {
        FastRec& fr = s_fast[slot][lane];
        fr.kind = kFastNone;
        if (w.policy == 0 && cf != kNone) {
          const int kind = w.fast[f].kind;
          if (kind != kFastNone) {
            const int n = w.fast[f].n;
            for (int k = 0; k < n; ++k) fr.st[k] = w.fast[f].st[k];
            fr.n = n;
            fr.gap = w.fast[f].gap;
          }
          fr.kind = kind;
        }
      }
      mbar_arrive_rel(&s_full[slot]);  // release: this lane's entries are written
    }
  } else {  // warp 0: the commit
  World v = w;
  if (smem_g) {
    v.g_npods = sg;
    v.g_hgo = sg + G;
    v.g_nparts = sg + 2 * G;
    v.g_freesm = sg + 3 * G;
    v.g_nextuid = reinterpret_cast<uint32_t*>(sg + 4 * G);
  }
  if (lane == 0) s_nact = 0;
  __syncwarp();
  __shared__ int s_err, s_npods;
  __shared__ long long s_counter;
  if (lane == 0) {
    s_err = *(volatile int32_t*)w.err != 0;  // phase A errors stop the commit at once
    s_npods = *w.n_pods;
    s_counter = (long long)*w.counter;
  }
  __syncwarp();
  __shared__ uint32_t s_smask[4];
  if (lane < 4) s_smask[lane] = w.sm_mask[lane];
  __syncwarp();
  CommitT<kMasked> c{v, lane, sp, ovf, ps, &s_nact, &s_err, &s_npods, &s_counter, skey, s_smask};
  c.load_counters();
  bool stop = s_err != 0;
#ifdef RAPP_TICK_PROF
  s_tprof[lane] = 0;
  __syncwarp();
  if (lane == 0) s_tprof[20] = clock64() - _pro0;  // prologue: state into shared memory
#endif
  // First-pod quota rows of the scale-up functions of a batch of 32 are bulk-copied into
  // shared memory one batch ahead (double buffer), so a vertical walk that has to be
  // redone (its partition's headroom changed since phase A) reads shared memory.
  __shared__ uint64_t s_rbar[2];
  if (lane == 0) {
    tk_bar_init(&s_rbar[0]);
    tk_bar_init(&s_rbar[1]);
  }
  __syncwarp();
  auto stage = [&](int b0, int cls_lane, int buf) {
    const bool want = w.policy == 0 && cls_lane == kUp;
    const unsigned wm = __ballot_sync(0xffffffffu, want);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // WAR vs earlier reads
    if (lane == 0) tk_bar_expect(&s_rbar[buf], uint32_t(__popc(wm)) * kRowStage * 8u);
    __syncwarp();
    if (want)
      tk_bulk(s_rows + (buf * 32 + lane) * kRowStage, w.rows + int64_t(b0 + lane) * kMaxPods * kRow,
              kRowStage * 8u, &s_rbar[buf]);
  };
  int cls_nxt = 32 + lane < w.F ? w.cls[32 + lane] : kNone;
  if (!stop) stage(0, lane < w.F ? w.cls[lane] : kNone, 0);
  int staged = 1;  // batches whose copies were issued
  int j = 0;
  uint32_t epoch = 0;  // fast_run conflict-mark epochs
  TPROF_T0();
  for (int base = 0; base < w.F && !stop; base += 32, ++j) {
    TPROF_ACC(6);  // (the functions of the previous batch, accounted separately)
    const int slot = j % kPreDepth;
    while (!__all_sync(0xffffffffu, mbar_try(&s_full[slot], (j / kPreDepth) & 1))) {
    }
    const int mine = s_pcls[slot][lane];
    if (base + 32 < w.F) {
      stage(base + 32, cls_nxt, (j + 1) & 1);
      ++staged;
    }
    cls_nxt = base + 64 + lane < w.F ? w.cls[base + 64 + lane] : kNone;
    tk_bar_wait(&s_rbar[j & 1], (j >> 1) & 1);
    TPROF_ACC(0);  // waits for the header ring and the staged rows
    unsigned act = __ballot_sync(0xffffffffu, mine != kNone);
    // (straight-line commits update the shared-memory GPU summaries: smem_g only)
    const int fk = mine != kNone && smem_g ? s_fast[slot][lane].kind : kFastNone;
    unsigned fastm = __ballot_sync(0xffffffffu, fk == kFastUp || fk == kFastDown);
    unsigned tailm = __ballot_sync(0xffffffffu, fk == kFastTail);
#ifdef RAPP_TICK_PROF
    if (lane == 0) s_tprof[15] += __popc(fastm | tailm);
#endif
    while (act) {
      const int i = __ffs(act) - 1;
      if (((fastm | tailm) >> i) & 1) {
        // straight-line functions from i up to the next one that is not, plus that one
        // when only its horizontal branch is not
        const unsigned slow = act & ~fastm;
        const int s0 = slow ? __ffs(slow) - 1 : 32;
        unsigned cand = act & fastm & (s0 < 32 ? (1u << s0) - 1 : ~0u);
        if (s0 < 32 && ((tailm >> s0) & 1)) cand |= 1u << s0;
        unsigned dead;
#ifdef RAPP_TICK_PROF
        const long long _fr0 = clock64();
#endif
        const unsigned done = c.fast_run(base, cand, s_fast[slot][lane], s_pre[slot][lane].stamp,
                                         now, s_htab, ++epoch, dead);
        fastm &= ~dead;  // a changed partition stays changed: no second attempt
        tailm &= ~dead;
#ifdef RAPP_TICK_PROF
        if (lane == 0) {
          s_tprof[16] += clock64() - _fr0;
          s_tprof[17] += 1;
          s_tprof[19] += done != 0;
        }
#endif
        if (done) {
          act &= ~done;
          const unsigned tl = done & tailm;  // the run's last lane, walk applied
          if (tl) {
            const int k = __ffs(tl) - 1;
#ifdef RAPP_TICK_PROF
            if (lane == 0) s_tprof[27] += 1;  // straight-line walks ending in the horizontal branch
#endif
            c.scale_up_h(base + k, now, s_pre[slot][k], s_fast[slot][k].gap, s_pre[slot][k].npods);
            __syncwarp();
            if (s_err) {
              stop = true;
              break;
            }
          }
          continue;
        }
      }
      act &= act - 1;
      const int cls = __shfl_sync(0xffffffffu, mine, i);
      const CommitPre& pre = s_pre[slot][i];
      if (cls == kUp) {
        if (w.policy == 0)
          c.scale_up(base + i, now, pre, s_rows + ((j & 1) * 32 + i) * kRowStage);
        else
          c.replica_up(base + i, now);
      } else {
        c.scale_down(base + i, now, pre);
      }
      __syncwarp();
      if (s_err) {
        stop = true;
        break;
      }
    }
    __syncwarp();
    mbar_arrive_rel(&s_empty[slot]);  // the slot's entries are no longer read
  }
  if (lane == 0) s_stop = 1;  // release the helper if the commit stopped early
  // no bulk copy may still be in flight into shared memory when the CTA exits
  for (int k = j; k < staged; ++k) tk_bar_wait(&s_rbar[k & 1], (k >> 1) & 1);
  c.store_counters();
  if (lane == 0) {
    *w.n_pods = s_npods;
    *w.counter = s_counter;
  }
  __syncwarp();
  if (lane == 0) *w.n_actions = s_nact;
  if (lane < 4) w.sm_mask[lane] = 0u;  // rebuilt by the next tick's prologue
#ifdef RAPP_TICK_PROF
  __syncwarp();
  g_tick_prof[lane] += s_tprof[lane];
#endif
  }  // warp 0
  // every warp: the shared-memory cluster state back to global memory
  __syncthreads();
  const int32_t* nparts = smem_g ? sg + 2 * G : w.g_nparts;
  for (int g = threadIdx.x; g < G; g += blockDim.x)
    if (!ovf[g]) {
      const int n = nparts[g];
      for (int i = 0; i < n; ++i) w.g_parts[int64_t(g) * kPartCap + i] = sp[int64_t(g) * ps + i];
    }
  if (smem_g) {
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
      w.g_npods[g] = sg[g];
      w.g_hgo[g] = sg[G + g];
      w.g_nparts[g] = sg[2 * G + g];
      w.g_freesm[g] = sg[3 * G + g];
      w.g_nextuid[g] = uint32_t(sg[4 * G + g]);
    }
  }
}

// Releases reported by the host between ticks (a DRAINING pod whose last request finished:
// hs/sim.py:424-438 -> _release_pod -> allocator.release_pod, hs/allocator.py:128-139), in
// the order given.  One warp; partition lists are read from global memory.
// `rel_ovf` is a G-byte global array of ones: every partition list lives in global memory
// (no shared-memory staging, so any cluster size launches).
__global__ void __launch_bounds__(32) k_tick_release(World w, const int32_t* __restrict__ list,
                                                     int n, uint8_t* rel_ovf) {
  __shared__ int s_nact, s_err, s_npods;
  __shared__ long long s_counter;
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    s_err = 0;
    s_nact = s_npods = 0;  // releases create no actions or pods
    s_counter = 0;
  }
  __syncwarp();
  CommitT<false> c{w, lane, nullptr, rel_ovf, 0, &s_nact, &s_err, &s_npods, &s_counter, nullptr,
           nullptr};
  c.load_counters();
  for (int i = 0; i < n; ++i) {
    const int p = list[i];
    if (w.p_state[p] == kDead) continue;
    c.release(p, w.p_fn[p], w.p_gpu[p], w.p_puid[p], w.p_s[p], w.p_q[p]);
  }
}

// ---------------------------------------------------------------------------------------
// prefix-max index for the fresh-GPU search (built once; tables are immutable)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void index_point(const World& w, int f, int64_t i, double& lat,
                                            double& rps) {
  const int nb = w.fn_nb[f];
  const TableDesc td = w.tds[w.fn_table[f]];
  const int pair = w.pairs[w.fn_pairs_off[f] + int(i / nb)];
  const double b = w.blist[w.fn_boff[f] + i % nb];
  const double s = w.pool[td.off + td.os + (pair >> 16)];
  const double q = double(pair & 0xFFFF);
  const double* seg = w.pool + td.off;
  lat = interp3(seg + td.ob, td.nb, seg + td.os, td.ns, seg + td.oq, td.nq, seg + td.ov, b, s,
                q);
  rps = throughput(b, lat);  // b / (lat / 1000.0), hs/perf.py:95-98
}

// rps of every lattice point in key order; with the opt-in SLO, points whose latency
// exceeds it are -inf (never feasible, never raise the prefix max)
__global__ void k_index_rps(World w, int f0) {
  const int f = f0 + blockIdx.y;
  if (f >= w.F) return;
  const int64_t L = w.fn_lat_len[f];
  const double slo = w.fn_slo != nullptr ? w.fn_slo[f] : __longlong_as_double(-1ll);  // NaN
  double* out = const_cast<double*>(w.pmax) + w.fn_lat_off[f];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
       i += int64_t(gridDim.x) * blockDim.x) {
    double lat, rps;
    index_point(w, f, i, lat, rps);
    out[i] = lat > slo ? -INFINITY : rps;
  }
}

// order-preserving uint64 image of a double (max of images == image of the max)
__device__ __forceinline__ unsigned long long ord_bits(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// SLO functions: the reference's fallback over the WHOLE lattice — max rps (pass 0), then
// the first key-order point with that rps (pass 1) — argmin (-rps, s*q, s, q, b)
__global__ void k_index_fb(World w, int f0, int pass, unsigned long long* best) {
  const int f = f0 + blockIdx.y;
  if (f >= w.F || !(w.fn_slo[f] == w.fn_slo[f])) return;  // NaN: no SLO, no fallback index
  const int64_t L = w.fn_lat_len[f];
  unsigned long long m = pass == 0 ? 0ull : ~0ull;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
       i += int64_t(gridDim.x) * blockDim.x) {
    double lat, rps;
    index_point(w, f, i, lat, rps);
    if (rps != rps) continue;
    if (pass == 0) {
      const unsigned long long o = ord_bits(rps);
      m = o > m ? o : m;
    } else if (ord_bits(rps) == best[f]) {
      m = (unsigned long long)i < m ? (unsigned long long)i : m;
      break;  // later i of this thread are larger
    }
  }
  if (pass == 0) {
    if (m) atomicMax(&best[f], m);
  } else if (m != ~0ull) {
    atomicMin(reinterpret_cast<unsigned long long*>(const_cast<int64_t*>(w.fn_fb)) + f, m);
  }
}

// in-place inclusive prefix max per function (one CTA per function, chunked scan)
__global__ void k_index_scan(World w, int f0) {
  const int f = f0 + blockIdx.x;
  if (f >= w.F) return;
  const int64_t L = w.fn_lat_len[f];
  double* a = const_cast<double*>(w.pmax) + w.fn_lat_off[f];
  __shared__ double s_carry;
  __shared__ double s_warp[32];
  if (threadIdx.x == 0) s_carry = -INFINITY;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t base = 0; base < L; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    double v = i < L ? a[i] : -INFINITY;
    for (int o = 1; o < 32; o <<= 1) {
      const double x = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v = x > v ? x : v;
    }
    if (lane == 31) s_warp[wid] = v;
    __syncthreads();
    if (wid == 0) {
      double x = lane < nw ? s_warp[lane] : -INFINITY;
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = y > x ? y : x;
      }
      if (lane < nw) s_warp[lane] = x;
    }
    __syncthreads();
    const double carry = s_carry;
    if (wid > 0) v = s_warp[wid - 1] > v ? s_warp[wid - 1] : v;
    v = carry > v ? carry : v;
    if (i < L) a[i] = v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = v;
    __syncthreads();
  }
}

}  // namespace rapp

using namespace rapp;

constexpr size_t kOutHead = 16;  // n_actions, err, err_fn, pad (int32 each)

struct rapp_tick {
  rapp_ctx* ctx = nullptr;
  int64_t pend_spec = -1;  // submitted host tick awaiting rapp_tick_collect (-1: none)
  World w{};
  std::vector<std::pair<void*, size_t>> allocs;  // device buffers (returned to the pool)
  size_t h_in_bytes = 0, h_out_bytes = 0;
  cudaStream_t stream = nullptr;
  // staging for the host API
  int64_t* d_arrivals = nullptr;
  uint8_t* d_idle = nullptr;
  double* d_pred_in = nullptr;
  uint8_t* d_in = nullptr;     // input block (d_arrivals, d_pred_in, d_idle point into it)
  uint8_t* d_out = nullptr;    // output block (w.n_actions ... w.actions point into it)
  // pinned staging for the host API: inputs [arrivals F x i64 | predicted F x f64 | idle
  // pod_cap bytes], outputs [actions 1024 | observed F | predicted F], so every copy of a
  // tick is asynchronous and the tick synchronises once
  uint8_t* h_in = nullptr;
  uint8_t* h_out = nullptr;
  int32_t* d_rel = nullptr;   // between-tick release list (grown on demand)
  int32_t* h_rel = nullptr;   // pinned staging for it
  int64_t rel_cap = 0;
  int64_t h_npods = 0;         // pods created so far (host copy of w.n_pods)
  uint8_t* d_ovf_ones = nullptr;  // [G] ones: k_tick_release's "list in global memory" flags
  cudaEvent_t order_ev = nullptr;  // orders rapp_tick_run_dev's stream against t->stream
  double* d_slo = nullptr;         // rapp_tick_set_slo: per-function SLO (NaN: none)
  int64_t* d_fb = nullptr;         //   fallback index per SLO function
  unsigned long long* d_fb_best = nullptr;  //   its max-rps image (k_index_fb pass 0)
};

namespace rapp {

// Allocation cache of tick worlds.  The single-function seams (Autoscaler.scale and the
// replica policies' decide, hs/autoscaler.py:73 / hs/policies.py:25-33) build and drop a
// world on every call, so a world's device buffers, pinned staging, stream and event go
// back to a per-device pool when it is destroyed and the next world of similar shape takes
// them instead of cudaMalloc / cudaMallocHost (which synchronise and cost milliseconds).
// Bounded: beyond the caps buffers are freed; rapp_shutdown empties it.
struct TickPool {
  std::mutex mu;
  std::multimap<size_t, void*> dev, host;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> streams;
  size_t dev_bytes = 0, host_bytes = 0;
};
constexpr size_t kPoolDevCap = size_t(512) << 20, kPoolHostCap = size_t(64) << 20;
static TickPool g_tick_pool[64];

static size_t pool_round(size_t b) {
  b = std::max<size_t>(b, 256);
  if (b <= (size_t(64) << 10)) {
    size_t r = 256;
    while (r < b) r <<= 1;
    return r;
  }
  return (b + 65535) & ~size_t(65535);
}

static TickPool& pool_of(int dev) { return g_tick_pool[dev & 63]; }

static cudaError_t pool_take(int dev, bool host, size_t bytes, void** out) {
  const size_t r = pool_round(bytes);
  TickPool& P = pool_of(dev);
  {
    std::lock_guard<std::mutex> lk(P.mu);
    auto& m = host ? P.host : P.dev;
    auto it = m.find(r);
    if (it != m.end()) {
      *out = it->second;
      m.erase(it);
      (host ? P.host_bytes : P.dev_bytes) -= r;
      return cudaSuccess;
    }
  }
  return host ? cudaMallocHost(out, r) : cudaMalloc(out, r);
}

static void pool_give(int dev, bool host, void* p, size_t bytes) {
  if (p == nullptr) return;
  const size_t r = pool_round(bytes);
  TickPool& P = pool_of(dev);
  {
    std::lock_guard<std::mutex> lk(P.mu);
    size_t& held = host ? P.host_bytes : P.dev_bytes;
    if (held + r <= (host ? kPoolHostCap : kPoolDevCap)) {
      (host ? P.host : P.dev).emplace(r, p);
      held += r;
      return;
    }
  }
  if (host)
    cudaFreeHost(p);
  else
    cudaFree(p);
}

static void pool_drain(int dev) {
  TickPool& P = pool_of(dev);
  std::lock_guard<std::mutex> lk(P.mu);
  for (auto& kv : P.dev) cudaFree(kv.second);
  for (auto& kv : P.host) cudaFreeHost(kv.second);
  for (auto& se : P.streams) {
    cudaEventDestroy(se.second);
    cudaStreamDestroy(se.first);
  }
  P.dev.clear();
  P.host.clear();
  P.streams.clear();
  P.dev_bytes = P.host_bytes = 0;
}

// zeroed device buffer of n T's, ordered on the world's stream
template <typename T>
static int dev_alloc(rapp_tick* t, T** p, size_t n) {
  void* q = nullptr;
  const size_t bytes = std::max<size_t>(1, n) * sizeof(T);
  RAPP_CUDA(pool_take(t->ctx->device, false, bytes, &q));
  t->allocs.emplace_back(q, bytes);
  RAPP_CUDA(cudaMemsetAsync(q, 0, bytes, t->stream));
  *p = static_cast<T*>(q);
  return RAPP_OK;
}

template <typename T>
static int dev_upload(rapp_tick* t, T** p, const std::vector<T>& v) {
  int rc = dev_alloc(t, p, v.size());
  if (rc) return rc;
  if (!v.empty())
    RAPP_CUDA(cudaMemcpyAsync(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice,
                              t->stream));
  return RAPP_OK;
}

static PodId pack_id(const char* s) {
  PodId id;
  for (int i = 0; i < 4; ++i) {
    uint64_t x = 0;
    for (int k = 0; k < 8; ++k) x = (x << 8) | uint8_t(s[i * 8 + k]);
    id.w[i] = x;
  }
  return id;
}

static void unpack_id(const PodId& id, char* s) {
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 8; ++k) s[i * 8 + k] = char((id.w[i] >> (8 * (7 - k))) & 0xFF);
}

static int launch_tick(rapp_tick* t, double now, const int64_t* d_arr, const uint8_t* d_idle,
                       const double* d_pred, cudaStream_t st) {
  World w = t->w;
  w.p_idle = d_idle;
  k_tick_prologue<<<std::max(1, std::min(64, (w.pod_cap + 255) / 256)), 256, 0, st>>>(w, now);
  RAPP_LAUNCHED();
  if (w.F > 0) {
    RAPP_CUDA(launch_pdl(k_tick_phase_a, dim3((w.F + 7) / 8), dim3(256), 0, st, w, now, d_arr,
                         d_pred));
    RAPP_LAUNCHED();
    RAPP_CUDA(launch_pdl(k_tick_grid, dim3(w.F), dim3(256), 0, st, w));
    RAPP_LAUNCHED();
    // shared memory: GPU summaries (5 ints/GPU) + a partition cache of up to 12 entries
    // per GPU + overflow flags, within ~200 KB
    // 227 KB per CTA minus the row staging and the static shared memory
    // fine quota steps: phase A2 tabulated the mask's rows only (see k_tick_prologue)
    const bool masked = w.delta <= kMaskMaxDelta;
    auto commit = masked ? k_tick_commit<true> : k_tick_commit<false>;
    static size_t static_smem = 0;  // the kernels' static shared memory (header ring etc.)
    if (static_smem == 0) {
      cudaFuncAttributes fa{}, fb{};
      RAPP_CUDA(cudaFuncGetAttributes(&fa, k_tick_commit<true>));
      RAPP_CUDA(cudaFuncGetAttributes(&fb, k_tick_commit<false>));
      static_smem = std::max(fa.sharedSizeBytes, fb.sharedSizeBytes) + 1024;
    }
    const size_t budget = 227 * 1024 - size_t(2 * 32 * kRowStage) * 8 - static_smem;
    const size_t gbytes = size_t(5 * w.G + 1) / 2 * 2 * sizeof(int32_t);
    const size_t fixed = gbytes + size_t((w.G + 3) & ~3) + size_t(w.G) * 4 + 16;
    const int smem_g = fixed <= budget ? 1 : 0;
    int ps = 0;
    if (smem_g)
      ps = (int)std::min<size_t>(12, (budget - fixed) / (8 * std::max(1, w.G)));
    const size_t bytes = smem_g ? size_t(2 * 32 * kRowStage) * 8 + gbytes + size_t(w.G) * ps * 8 +
                                      size_t((w.G + 3) & ~3) + size_t(w.G) * 4 + 16  // + keys
                                : size_t(2 * 32 * kRowStage) * 8 + size_t(w.G) + 16;   // ovf only
    RAPP_CUDA(cudaFuncSetAttribute(commit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(bytes, 48 * 1024)));
    RAPP_CUDA(launch_pdl(commit, dim3(1), dim3(kCommitThreads), bytes, st, w, now, smem_g, ps));
    RAPP_LAUNCHED();
  }
  return RAPP_OK;
}

}  // namespace rapp

extern "C" {

int rapp_tick_create(rapp_ctx* ctx, const rapp_scaler_config* cfg, int64_t n_fns,
                     const rapp_fn_desc* fns, const int64_t* batch_lattice, int64_t n_gpus,
                     const int64_t* part_off, const int32_t* part_sm, const int32_t* part_alloc,
                     int64_t n_pods, const rapp_pod_desc* pods, int64_t pod_counter,
                     rapp_tick** out) {
  if (!ctx || !cfg || !out || n_fns < 0 || n_gpus < 0 || n_pods < 0) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  if (cfg->delta_iq < 1 || cfg->delta_iq > 100) {
    set_error("delta_iq %d outside [1, 100]", cfg->delta_iq);
    return RAPP_E_VALUE;
  }
  // world sizes the device layout supports: GPU ranks in 18-bit argmin keys, functions and
  // pods in int32 indices ([F][kMaxPods] tables)
  if (n_gpus > kMaxGpus || n_fns > kMaxFns || n_pods > int64_t(kMaxFns) * kMaxPods) {
    set_error("world of %lld functions / %lld GPUs / %lld pods exceeds the tick's limits "
              "(%d functions, %d GPUs, %d pods per function)", (long long)n_fns,
              (long long)n_gpus, (long long)n_pods, kMaxFns, kMaxGpus, kMaxPods);
    return RAPP_E_ARG;
  }
  std::lock_guard<std::mutex> lk(ctx->mu);
  RAPP_CUDA(cudaSetDevice(ctx->device));
  std::unique_ptr<rapp_tick, int (*)(rapp_tick*)> t(new rapp_tick(), rapp_tick_destroy);
  t->ctx = ctx;
  {
    TickPool& P = pool_of(ctx->device);
    std::lock_guard<std::mutex> plk(P.mu);
    if (!P.streams.empty()) {
      t->stream = P.streams.back().first;
      t->order_ev = P.streams.back().second;
      P.streams.pop_back();
    }
  }
  if (t->stream == nullptr) {
    RAPP_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    RAPP_CUDA(cudaEventCreateWithFlags(&t->order_ev, cudaEventDisableTiming));
  }
  World& w = t->w;
  w.alpha = cfg->alpha;
  w.beta = cfg->beta;
  w.cooldown = cfg->cooldown_ms;
  w.r_min = cfg->r_min;
  w.interval_s = cfg->interval_s;
  w.cold_start = cfg->cold_start_ms;
  w.kA = cfg->kal_A;
  w.kQ = cfg->kal_Q;
  w.kH = cfg->kal_H;
  w.kD = cfg->kal_D;
  w.kP0 = cfg->kal_P0;
  w.delta = cfg->delta_iq;
  w.sum_plain = cfg->sum_mode == 1;
  if (cfg->policy != 0 && cfg->policy != 1) {
    set_error("unknown policy code %d", cfg->policy);
    return RAPP_E_VALUE;
  }
  w.policy = cfg->policy;
  const int F = (int)n_fns, G = (int)n_gpus;
  w.F = F;
  w.G = G;
  // ---- functions, tables, search index ----
  std::vector<int32_t> fn_table(F), fn_nb(F), fn_init(F), fn_npods(F, 0), fn_pairs_off(F),
      fn_npairs(F), fn_shape(3 * (size_t)F);
  std::vector<double> fn_min(F), kR(F), kP(F), last(F), blist;
  std::vector<int64_t> fn_boff(F), fn_lat_off(F), fn_lat_len(F);
  std::vector<int32_t> pairs;
  std::vector<std::pair<std::vector<double>, int32_t>> shape_cache;  // (sms, ..) -> offset
  int64_t lat_total = 0;
  const int d = cfg->delta_iq;
  const int nQ = 100 / d;
  for (int f = 0; f < F; ++f) {
    const rapp_fn_desc& fd = fns[f];
    if (fd.table_id < 0 || fd.table_id >= (int32_t)ctx->tables.size()) {
      set_error("function %d: unknown table id %d", f, fd.table_id);
      return RAPP_E_ARG;
    }
    const TableDesc& td = ctx->tables[fd.table_id];
    if (!td.sm_keyable) {
      set_error("function %d: sm axis must hold integers in [0, 2^24)", f);
      return RAPP_E_ARG;
    }
    fn_table[f] = fd.table_id;
    fn_shape[3 * f] = fd.shape_batch;
    fn_shape[3 * f + 1] = fd.shape_sm;
    fn_shape[3 * f + 2] = fd.shape_quota;
    fn_min[f] = fd.min_rps;
    fn_init[f] = fd.kal_init;
    kR[f] = fd.kal_R;
    kP[f] = fd.kal_P;
    last[f] = fd.last_down_ms;
    fn_nb[f] = (int32_t)fd.lattice_len;
    fn_boff[f] = (int64_t)blist.size();
    if (fd.lattice_len < 1) {
      set_error("function %d: empty batch lattice", f);
      return RAPP_E_ARG;
    }
    for (int64_t i = 0; i < fd.lattice_len; ++i) blist.push_back((double)batch_lattice[fd.lattice_off + i]);
    // (s, q) pairs of the lattice in key order (s*q, s, q); batches vary fastest
    std::vector<double> sms((size_t)td.ns);
    RAPP_CUDA(cudaMemcpy(sms.data(), ctx->d_pool + td.off + td.os, sms.size() * 8,
                         cudaMemcpyDeviceToHost));
    int32_t off = -1;
    for (auto& sc : shape_cache)
      if (sc.first == sms) off = sc.second;
    if (off < 0) {
      std::vector<std::array<int64_t, 4>> keys;
      for (int si = 0; si < td.ns; ++si)
        for (int qi = 1; qi <= nQ; ++qi) {
          const int64_t s = (int64_t)sms[si], q = (int64_t)qi * d;
          keys.push_back({s * q, s, q, (int64_t)si});
        }
      std::sort(keys.begin(), keys.end());
      off = (int32_t)pairs.size();
      for (auto& k : keys) pairs.push_back(int32_t(k[3] << 16 | k[2]));
      shape_cache.push_back({sms, off});
    }
    fn_pairs_off[f] = off;
    fn_npairs[f] = td.ns * nQ;
    fn_lat_off[f] = lat_total;
    fn_lat_len[f] = (int64_t)td.ns * nQ * fd.lattice_len;
    lat_total += fn_lat_len[f];
  }
  int rc;
#define UP(ptr, vec) \
  if ((rc = dev_upload(t.get(), &ptr, vec))) return rc;
  {
    int32_t *a;
    double *b;
    int64_t *c;
    UP(a, fn_table) w.fn_table = a;
    UP(a, fn_shape) w.fn_shape = a;
    UP(b, fn_min) w.fn_min_rps = b;
    UP(c, fn_lat_off) w.fn_lat_off = c;
    UP(c, fn_lat_len) w.fn_lat_len = c;
    UP(a, fn_nb) w.fn_nb = a;
    UP(c, fn_boff) w.fn_boff = c;
    UP(b, blist) w.blist = b;
    UP(a, fn_pairs_off) w.fn_pairs_off = a;
    UP(a, fn_npairs) w.fn_npairs = a;
    UP(a, pairs) w.pairs = a;
    UP(w.k_init, fn_init)
    UP(w.k_R, kR)
    UP(w.k_P, kP)
    UP(w.last_down, last)
    double* pm;
    if ((rc = dev_alloc(t.get(), &pm, (size_t)lat_total))) return rc;
    w.pmax = pm;
  }
  // ---- GPUs and partitions ----
  std::vector<int32_t> g_npods(G, 0), g_hgo(G, 0), g_nparts(G, 0), g_free(G, 100);
  std::vector<uint32_t> g_uid(G, 0);
  std::vector<uint64_t> g_parts((size_t)G * kPartCap, 0);
  for (int g = 0; g < G; ++g) {
    const int64_t n = part_off[g + 1] - part_off[g];
    if (n > kPartCap) {
      set_error("GPU %d holds %lld partitions (> %d)", g, (long long)n, kPartCap);
      return RAPP_E_INVARIANT;
    }
    g_nparts[g] = (int32_t)n;
    g_uid[g] = (uint32_t)n;
    for (int64_t i = 0; i < n; ++i) {
      const int sm = part_sm[part_off[g] + i], al = part_alloc[part_off[g] + i];
      g_parts[(size_t)g * kPartCap + i] = part_pack(sm, al, 0, (uint32_t)i);
      g_free[g] -= sm;
    }
  }
  // ---- pods ----
  const int cap = (int)(n_pods + 2 * (int64_t)F * 64 + 1024);  // room for many ticks of growth
  w.pod_cap = cap;
  std::vector<int32_t> p_fn(cap, -1), p_b(cap, 0), p_s(cap, 0), p_q(cap, 0), p_gpu(cap, 0),
      p_state(cap, kDead), fn_pods((size_t)F * kMaxPods, 0);
  std::vector<uint32_t> p_puid(cap, 0);
  std::vector<double> p_ready(cap, 0.0);
  std::vector<PodId> p_id(cap, PodId{{0, 0, 0, 0}});
  for (int64_t i = 0; i < n_pods; ++i) {
    const rapp_pod_desc& pd = pods[i];
    if (pd.gpu < 0 || pd.gpu >= G) {
      set_error("pod %lld: GPU rank %d out of range", (long long)i, pd.gpu);
      return RAPP_E_INVARIANT;
    }
    const int g = pd.gpu;
    if (pd.part < 0 || pd.part >= g_nparts[g]) {
      set_error("pod %lld: partition %d out of range", (long long)i, pd.part);
      return RAPP_E_INVARIANT;
    }
    uint64_t& e = g_parts[(size_t)g * kPartCap + pd.part];
    e = part_pack(rapp::part_sm(e), rapp::part_alloc(e), part_npods(e) + 1, part_uid(e));
    p_fn[i] = pd.fn;
    p_b[i] = pd.batch;
    p_s[i] = pd.sm;
    p_q[i] = pd.quota;
    p_gpu[i] = g;
    p_puid[i] = part_uid(e);
    p_state[i] = pd.state;
    p_ready[i] = pd.ready_at_ms;
    p_id[i] = pack_id(pd.id);
    g_npods[g] += 1;
    g_hgo[g] += pd.sm * pd.quota;
    if (pd.fn >= 0) {
      if (pd.fn >= F || fn_npods[pd.fn] >= kMaxPods) {
        set_error("function %d: more than %d pods", pd.fn, kMaxPods);
        return RAPP_E_ARG;
      }
      fn_pods[(size_t)pd.fn * kMaxPods + fn_npods[pd.fn]++] = (int32_t)i;
    }
  }
  UP(w.g_npods, g_npods)
  UP(w.g_hgo, g_hgo)
  UP(w.g_nparts, g_nparts)
  UP(w.g_freesm, g_free)
  UP(w.g_nextuid, g_uid)
  UP(w.g_parts, g_parts)
  UP(w.p_fn, p_fn)
  UP(w.p_b, p_b)
  UP(w.p_s, p_s)
  UP(w.p_q, p_q)
  UP(w.p_gpu, p_gpu)
  UP(w.p_puid, p_puid)
  UP(w.p_state, p_state)
  UP(w.p_ready, p_ready)
  UP(w.p_id, p_id)
  if ((rc = dev_alloc(t.get(), &w.p_ctr, (size_t)cap))) return rc;
  RAPP_CUDA(cudaMemsetAsync(w.p_ctr, 0xFF, (size_t)cap * sizeof(int64_t), t->stream));  // -1
  UP(w.fn_npods, fn_npods)
  UP(w.fn_pods, fn_pods)
#undef UP
  {
    std::vector<int32_t> np(1, (int32_t)n_pods);
    if ((rc = dev_upload(t.get(), &w.n_pods, np))) return rc;
    std::vector<int64_t> ctr(1, pod_counter);
    if ((rc = dev_upload(t.get(), &w.counter, ctr))) return rc;
  }
  w.tds = ctx->d_desc;
  w.pool = ctx->d_pool;
  // scratch / outputs
  const size_t FP = (size_t)std::max(F, 1);
  // outputs a host call reads back, in one block so one copy returns them:
  // [n_actions, err, err_fn, pad][observed F][predicted F][actions]
  {
    uint8_t* ob = nullptr;
    const size_t out_bytes = kOutHead + FP * 16 + FP * (kMaxPods + 4) * sizeof(rapp_action);
    if ((rc = dev_alloc(t.get(), &ob, out_bytes))) return rc;
    t->d_out = ob;
    w.n_actions = reinterpret_cast<int32_t*>(ob);
    w.err = reinterpret_cast<int32_t*>(ob + 4);
    w.err_fn = reinterpret_cast<int32_t*>(ob + 8);
    w.obs = reinterpret_cast<double*>(ob + kOutHead);
    w.pred = w.obs + FP;
    w.actions = reinterpret_cast<rapp_action*>(ob + kOutHead + FP * 16);
  }
  if ((rc = dev_alloc(t.get(), &w.cls, FP))) return rc;
  if ((rc = dev_alloc(t.get(), &w.gap0, FP))) return rc;
  if ((rc = dev_alloc(t.get(), &w.wanted, FP))) return rc;
  if ((rc = dev_alloc(t.get(), &w.nsorted, FP))) return rc;
  if ((rc = dev_alloc(t.get(), &w.sorted, FP * kMaxPods))) return rc;
  if ((rc = dev_alloc(t.get(), &w.row_kd, FP * kMaxPods))) return rc;
  if ((rc = dev_alloc(t.get(), &w.rows, FP * kMaxPods * kRow))) return rc;
  if ((rc = dev_alloc(t.get(), &w.bref, FP))) return rc;
  if ((rc = dev_alloc(t.get(), &w.bref_ok, FP))) return rc;
  if ((rc = dev_alloc(t.get(), &w.spec_avail, FP * kMaxPods))) return rc;
  if ((rc = dev_alloc(t.get(), &w.spec_k, FP * kMaxPods))) return rc;
  if ((rc = dev_alloc(t.get(), &w.spec_gain, FP * kMaxPods))) return rc;
  if ((rc = dev_alloc(t.get(), &w.spec_kg, FP * kMaxPods))) return rc;
  if ((rc = dev_alloc(t.get(), &w.fast, FP))) return rc;
  if ((rc = dev_alloc(t.get(), &w.tgrid, FP * 100 * 100))) return rc;
  if ((rc = dev_alloc(t.get(), &w.sm_mask, 4))) return rc;  // zeroed
  {
    const char* mn = getenv("RAPP_TICK_MASK_NONE");  // "1": test switch (see World)
    w.mask_none = mn != nullptr && strcmp(mn, "1") == 0;
  }
  if ((rc = dev_alloc(t.get(), &w.brk, FP * kBrkPerFn))) return rc;
  if ((rc = dev_alloc(t.get(), &w.ndown, FP))) return rc;
  if ((rc = dev_alloc(t.get(), &w.down, FP * kMaxPods))) return rc;
  if ((rc = dev_alloc(t.get(), &w.stamp, FP))) return rc;
  // inputs of a host call, in one block mirrored by the pinned staging (one copy):
  // [arrivals F x i64][predicted F x f64][idle flags pod_cap bytes]
  {
    uint8_t* ib = nullptr;
    if ((rc = dev_alloc(t.get(), &ib, FP * 16 + (size_t)cap))) return rc;
    t->d_in = ib;
    t->d_arrivals = reinterpret_cast<int64_t*>(ib);
    t->d_pred_in = reinterpret_cast<double*>(ib + FP * 8);
    t->d_idle = ib + FP * 16;
  }
  t->h_in_bytes = FP * 16 + (size_t)cap + 64;
  t->h_out_bytes = kOutHead + FP * 16 + 1024 * sizeof(rapp_action);
  RAPP_CUDA(pool_take(ctx->device, true, t->h_in_bytes, reinterpret_cast<void**>(&t->h_in)));
  RAPP_CUDA(pool_take(ctx->device, true, t->h_out_bytes, reinterpret_cast<void**>(&t->h_out)));
  // release staging sized for typical between-tick releases up front: a pinned allocation
  // inside a tick's host call costs milliseconds (rapp_tick_release grows it if needed)
  t->rel_cap = 1024;
  RAPP_CUDA(pool_take(ctx->device, false, (size_t)t->rel_cap * 4,
                      reinterpret_cast<void**>(&t->d_rel)));
  RAPP_CUDA(pool_take(ctx->device, true, (size_t)t->rel_cap * 4,
                      reinterpret_cast<void**>(&t->h_rel)));
  if ((rc = dev_alloc(t.get(), &t->d_ovf_ones, (size_t)std::max(1, w.G)))) return rc;
  RAPP_CUDA(cudaMemsetAsync(t->d_ovf_ones, 1, (size_t)std::max(1, w.G), t->stream));
  t->h_npods = n_pods;
  // build the fresh-GPU search index
  for (int f0 = 0; f0 < F; f0 += 32768) {
    const int nf = std::min(F - f0, 32768);
    k_index_rps<<<dim3(64, nf), 256, 0, t->stream>>>(w, f0);
    RAPP_LAUNCHED();
    k_index_scan<<<nf, 1024, 0, t->stream>>>(w, f0);
    RAPP_LAUNCHED();
  }
  RAPP_CUDA(cudaStreamSynchronize(t->stream));
  *out = t.release();
  return RAPP_OK;
}

int rapp_tick_destroy(rapp_tick* t) {
  if (!t) return RAPP_OK;
  const int dev = t->ctx->device;
  cudaSetDevice(dev);
  if (t->stream) cudaStreamSynchronize(t->stream);  // nothing of this world is in flight
  for (auto& a : t->allocs) pool_give(dev, false, a.first, a.second);
  pool_give(dev, true, t->h_in, t->h_in_bytes);
  pool_give(dev, true, t->h_out, t->h_out_bytes);
  pool_give(dev, false, t->d_rel, (size_t)t->rel_cap * 4);
  pool_give(dev, true, t->h_rel, (size_t)t->rel_cap * 4);
  bool kept = false;
  if (t->stream) {
    TickPool& P = pool_of(dev);
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.streams.size() < 8) {
      P.streams.emplace_back(t->stream, t->order_ev);
      kept = true;
    }
  }
  if (!kept) {
    if (t->order_ev) cudaEventDestroy(t->order_ev);
    if (t->stream) cudaStreamDestroy(t->stream);
  }
  delete t;
  return RAPP_OK;
}

int rapp_tick_pool_drain(int device) {
  rapp::pool_drain(device);
  return RAPP_OK;
}

int rapp_tick_pod_count(rapp_tick* t, int64_t* n) {
  if (!t || !n) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  int32_t v = 0;
  RAPP_CUDA(cudaMemcpy(&v, t->w.n_pods, sizeof v, cudaMemcpyDeviceToHost));
  *n = v;
  return RAPP_OK;
}

static int tick_error(rapp_tick* t) {
  int32_t e[2] = {0, 0};
  RAPP_CUDA(cudaMemcpy(&e[0], t->w.err, 4, cudaMemcpyDeviceToHost));
  RAPP_CUDA(cudaMemcpy(&e[1], t->w.err_fn, 4, cudaMemcpyDeviceToHost));
  if (e[0] == RAPP_OK) return RAPP_OK;
  switch (e[0]) {
    case RAPP_E_VALUE: set_error("function %d: batch outside table range", e[1]); break;
    case RAPP_E_DEGENERATE: set_error("function %d: H*P'*H + D == 0", e[1]); break;
    case RAPP_E_PLACEMENT: set_error("placement rejected (invariant broken)"); break;
    default: set_error("function %d: pod capacity exceeded", e[1]); break;
  }
  return e[0];
}

int rapp_tick_release(rapp_tick* t, const int64_t* pods, int64_t n) {
  RAPP_RANGE("rapp_tick_release");
  if (!t || n < 0 || (n > 0 && !pods)) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  if (n == 0) return RAPP_OK;
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  if (t->pend_spec >= 0) {
    set_error("a submitted tick has not been collected");
    return RAPP_E_ARG;
  }
  RAPP_CUDA(cudaSetDevice(t->ctx->device));
  int64_t known = t->h_npods;
  if (known < 0) {
    int32_t v = 0;
    RAPP_CUDA(cudaMemcpy(&v, t->w.n_pods, sizeof v, cudaMemcpyDeviceToHost));
    known = t->h_npods = v;
  }
  if (n > t->rel_cap) {  // grow the persistent release buffers
    RAPP_CUDA(cudaStreamSynchronize(t->stream));
    pool_give(t->ctx->device, false, t->d_rel, (size_t)t->rel_cap * 4);
    pool_give(t->ctx->device, true, t->h_rel, (size_t)t->rel_cap * 4);
    t->d_rel = nullptr;
    t->h_rel = nullptr;
    t->rel_cap = std::max<int64_t>(n, 1024);
    RAPP_CUDA(pool_take(t->ctx->device, false, (size_t)t->rel_cap * 4,
                        reinterpret_cast<void**>(&t->d_rel)));
    RAPP_CUDA(pool_take(t->ctx->device, true, (size_t)t->rel_cap * 4,
                        reinterpret_cast<void**>(&t->h_rel)));
  }
  for (int64_t i = 0; i < n; ++i) {
    if (pods[i] < 0 || pods[i] >= known) {
      set_error("release: pod index %lld out of range", (long long)pods[i]);
      return RAPP_E_ARG;
    }
  }
  RAPP_CUDA(cudaStreamSynchronize(t->stream));  // the staging buffer is free again
  for (int64_t i = 0; i < n; ++i) t->h_rel[i] = (int32_t)pods[i];
  RAPP_CUDA(cudaMemcpyAsync(t->d_rel, t->h_rel, (size_t)n * 4, cudaMemcpyHostToDevice,
                            t->stream));
  // stream-ordered before the next tick; no host synchronisation needed here
  k_tick_release<<<1, 32, 0, t->stream>>>(t->w, t->d_rel, (int)n, t->d_ovf_ones);
  RAPP_LAUNCHED();
  return RAPP_OK;
}

int rapp_tick_run_dev(rapp_tick* t, double now_ms, const int64_t* d_arrivals,
                      const uint8_t* d_idle, void* stream) {
  RAPP_RANGE("rapp_tick_run_dev");
  if (!t) {
    set_error("null tick");
    return RAPP_E_ARG;
  }
  if (t->pend_spec >= 0) {
    set_error("a submitted tick has not been collected");
    return RAPP_E_ARG;
  }
  RAPP_CUDA(cudaSetDevice(t->ctx->device));
  t->h_npods = -1;  // the host no longer knows the pod count without a read-back
  // the world is shared with the host API's internal stream (releases, host ticks): order
  // this tick after that stream's work and that stream's later work after this tick
  cudaStream_t st = (cudaStream_t)stream;
  RAPP_CUDA(cudaEventRecord(t->order_ev, t->stream));
  RAPP_CUDA(cudaStreamWaitEvent(st, t->order_ev, 0));
  const int rc = launch_tick(t, now_ms, d_arrivals, d_idle, nullptr, st);
  if (rc) return rc;
  RAPP_CUDA(cudaEventRecord(t->order_ev, st));
  RAPP_CUDA(cudaStreamWaitEvent(t->stream, t->order_ev, 0));
  return RAPP_OK;
}

int rapp_tick_outputs_dev(rapp_tick* t, const rapp_action** a, const int32_t** c,
                          const double** o, const double** p) {
  if (!t) {
    set_error("null tick");
    return RAPP_E_ARG;
  }
  if (a) *a = t->w.actions;
  if (c) *c = t->w.n_actions;
  if (o) *o = t->w.obs;
  if (p) *p = t->w.pred;
  return RAPP_OK;
}

int rapp_tick_submit(rapp_tick* t, double now_ms, const int64_t* arrivals, const uint8_t* idle,
                     const double* predicted_in, int64_t max_actions) {
  RAPP_RANGE("rapp_tick_submit");
  if (!t || !arrivals) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  if (t->pend_spec >= 0) {
    set_error("a submitted tick has not been collected");
    return RAPP_E_ARG;
  }
  RAPP_CUDA(cudaSetDevice(t->ctx->device));
  World& w = t->w;
  cudaStream_t st = t->stream;
  const size_t F = (size_t)w.F;
  if (t->h_npods < 0) {  // after device-only ticks
    int32_t v = 0;
    RAPP_CUDA(cudaStreamSynchronize(st));
    RAPP_CUDA(cudaMemcpy(&v, w.n_pods, 4, cudaMemcpyDeviceToHost));
    t->h_npods = v;
  }
  const int64_t np = t->h_npods;  // tracked on the host: no round trip before the launch
  // inputs through pinned staging in the device block's layout: one H2D copy
  const size_t FP = std::max<size_t>(F, 1);
  int64_t* s_arr = reinterpret_cast<int64_t*>(t->h_in);
  double* s_pred = reinterpret_cast<double*>(t->h_in + FP * 8);
  uint8_t* s_idle = t->h_in + FP * 16;
  {
    RAPP_RANGE("tick.h2d");
    if (F) memcpy(s_arr, arrivals, F * 8);
    if (predicted_in && F) memcpy(s_pred, predicted_in, F * 8);
    if (idle && np) memcpy(s_idle, idle, (size_t)np);
    RAPP_CUDA(cudaMemcpyAsync(t->d_in, t->h_in, FP * 16 + (idle ? (size_t)np : 0),
                              cudaMemcpyHostToDevice, st));
    if (!idle && np) RAPP_CUDA(cudaMemsetAsync(t->d_idle, 0, (size_t)np, st));
  }
  int rc;
  {
    RAPP_RANGE("tick.launch (prologue, phase A, A2, commit)");
    rc = launch_tick(t, now_ms, t->d_arrivals, t->d_idle, predicted_in ? t->d_pred_in : nullptr,
                     st);
  }
  if (rc) return rc;
  // one D2H copy for the usual case: count, status, rates and the first actions (the
  // output block's prefix)
  const int64_t spec = std::min<int64_t>(std::max<int64_t>(max_actions, 0), 1024);
  RAPP_CUDA(cudaMemcpyAsync(t->h_out, t->d_out,
                            kOutHead + FP * 16 + (size_t)spec * sizeof(rapp_action),
                            cudaMemcpyDeviceToHost, st));
  t->pend_spec = spec;
  return RAPP_OK;
}

int rapp_tick_collect(rapp_tick* t, rapp_action* actions, int64_t max_actions,
                      int64_t* n_actions, double* observed_out, double* predicted_out) {
  RAPP_RANGE("rapp_tick_collect");
  if (!t || !n_actions) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  if (t->pend_spec < 0) {
    set_error("no submitted tick");
    return RAPP_E_ARG;
  }
  const int64_t spec = actions ? std::min(t->pend_spec, max_actions) : 0;
  t->pend_spec = -1;
  RAPP_CUDA(cudaSetDevice(t->ctx->device));
  World& w = t->w;
  cudaStream_t st = t->stream;
  const size_t F = (size_t)w.F;
  const size_t FP = std::max<size_t>(F, 1);
  int rc;
  RAPP_RANGE("tick.d2h + sync");
  const int32_t* h_count = reinterpret_cast<const int32_t*>(t->h_out);
  const double* s_obs = reinterpret_cast<const double*>(t->h_out + kOutHead);
  const double* s_prd = s_obs + FP;
  const rapp_action* s_act = reinterpret_cast<const rapp_action*>(t->h_out + kOutHead + FP * 16);
  RAPP_CUDA(cudaStreamSynchronize(st));
  if (h_count[1] != RAPP_OK) {
    if ((rc = tick_error(t))) return rc;
  }
  const int64_t n = h_count[0];
  *n_actions = n;
  if (n > max_actions) {
    // the tick is applied on the device already: keep the host's pod count in step so
    // the caller can read the actions from the device (rapp_tick_outputs_dev) and go on
    int32_t v = 0;
    RAPP_CUDA(cudaMemcpy(&v, w.n_pods, 4, cudaMemcpyDeviceToHost));
    t->h_npods = v;
    set_error("action buffer too small (%lld > %lld)", (long long)n, (long long)max_actions);
    return RAPP_E_ARG;
  }
  if (observed_out && F) memcpy(observed_out, s_obs, F * 8);
  if (predicted_out && F) memcpy(predicted_out, s_prd, F * 8);
  if (actions) memcpy(actions, s_act, (size_t)std::min<int64_t>(n, spec) * sizeof(rapp_action));
  if (actions && n > spec) {
    RAPP_CUDA(cudaMemcpyAsync(actions + spec, w.actions + spec,
                              (size_t)(n - spec) * sizeof(rapp_action), cudaMemcpyDeviceToHost,
                              st));
    RAPP_CUDA(cudaStreamSynchronize(st));
  }
  if (actions) {
    for (int64_t i = 0; i < n; ++i) t->h_npods += actions[i].kind == kHUp;
  } else {
    int32_t v = 0;
    RAPP_CUDA(cudaMemcpy(&v, w.n_pods, 4, cudaMemcpyDeviceToHost));
    t->h_npods = v;
  }
  return RAPP_OK;
}

int rapp_tick_run(rapp_tick* t, double now_ms, const int64_t* arrivals, const uint8_t* idle,
                  const double* predicted_in, rapp_action* actions, int64_t max_actions,
                  int64_t* n_actions, double* observed_out, double* predicted_out) {
  RAPP_RANGE("rapp_tick_run");
  if (!t || !arrivals || !n_actions) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  const int rc = rapp_tick_submit(t, now_ms, arrivals, idle, predicted_in,
                                  actions ? max_actions : 0);
  if (rc) return rc;
  return rapp_tick_collect(t, actions, max_actions, n_actions, observed_out, predicted_out);
}

int rapp_tick_read_pods(rapp_tick* t, rapp_pod_desc* out, int64_t cap, int64_t* n) {
  if (!t || !n) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  World& w = t->w;
  int32_t np = 0;
  RAPP_CUDA(cudaMemcpy(&np, w.n_pods, 4, cudaMemcpyDeviceToHost));
  *n = np;
  if (!out) return RAPP_OK;
  if (np > 0) {  // ids of pods created by the last tick are formatted lazily
    k_tick_format_ids<<<std::max(1, std::min(1024, (np + 255) / 256)), 256, 0, t->stream>>>(w);
    RAPP_LAUNCHED();
    RAPP_CUDA(cudaStreamSynchronize(t->stream));
  }
  if (np > cap) {
    set_error("pod buffer too small");
    return RAPP_E_ARG;
  }
  std::vector<int32_t> fn(np), b(np), s(np), q(np), g(np), st(np);
  std::vector<uint32_t> puid(np);
  std::vector<double> rd(np);
  std::vector<PodId> id(np);
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
  };
  if (np) {
    RAPP_CUDA(cp(fn.data(), w.p_fn, np * 4));
    RAPP_CUDA(cp(b.data(), w.p_b, np * 4));
    RAPP_CUDA(cp(s.data(), w.p_s, np * 4));
    RAPP_CUDA(cp(q.data(), w.p_q, np * 4));
    RAPP_CUDA(cp(g.data(), w.p_gpu, np * 4));
    RAPP_CUDA(cp(st.data(), w.p_state, np * 4));
    RAPP_CUDA(cp(puid.data(), w.p_puid, np * 4));
    RAPP_CUDA(cp(rd.data(), w.p_ready, np * 8));
    RAPP_CUDA(cp(id.data(), w.p_id, np * sizeof(PodId)));
  }
  // partition positions from uids
  std::vector<uint64_t> parts((size_t)w.G * kPartCap);
  std::vector<int32_t> nparts(w.G);
  if (w.G) {
    RAPP_CUDA(cp(parts.data(), w.g_parts, parts.size() * 8));
    RAPP_CUDA(cp(nparts.data(), w.g_nparts, w.G * 4));
  }
  for (int i = 0; i < np; ++i) {
    rapp_pod_desc& o = out[i];
    memset(&o, 0, sizeof o);
    o.fn = fn[i];
    o.batch = b[i];
    o.sm = s[i];
    o.quota = q[i];
    o.gpu = g[i];
    o.state = st[i];
    o.ready_at_ms = rd[i];
    o.part = -1;
    if (st[i] != kDead)
      for (int k = 0; k < nparts[g[i]]; ++k)
        if (part_uid(parts[(size_t)g[i] * kPartCap + k]) == puid[i]) {
          o.part = k;
          break;
        }
    unpack_id(id[i], o.id);
  }
  return RAPP_OK;
}

int rapp_tick_set_slo(rapp_tick* t, const double* slo_ms) {
  if (!t) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  World& w = t->w;
  const int F = w.F;
  if (slo_ms != nullptr)
    for (int f = 0; f < F; ++f)
      if (!(slo_ms[f] > 0.0) && !std::isnan(slo_ms[f])) {
        set_error("slo_ms must be positive (NaN: no SLO), got %g for function %d", slo_ms[f], f);
        return RAPP_E_VALUE;
      }
  std::lock_guard<std::mutex> lk(t->ctx->mu);
  RAPP_CUDA(cudaSetDevice(t->ctx->device));
  RAPP_CUDA(cudaStreamSynchronize(t->stream));
  if (slo_ms == nullptr) {
    w.fn_slo = nullptr;
    w.fn_fb = nullptr;
  } else {
    if (t->d_slo == nullptr) {
      int rc;
      if ((rc = dev_alloc(t, &t->d_slo, (size_t)std::max(1, F)))) return rc;
      if ((rc = dev_alloc(t, &t->d_fb, (size_t)std::max(1, F)))) return rc;
      if ((rc = dev_alloc(t, &t->d_fb_best, (size_t)std::max(1, F)))) return rc;
    }
    if (F)
      RAPP_CUDA(cudaMemcpyAsync(t->d_slo, slo_ms, (size_t)F * 8, cudaMemcpyHostToDevice,
                                t->stream));
    RAPP_CUDA(cudaMemsetAsync(t->d_fb, 0xFF, (size_t)std::max(1, F) * 8, t->stream));  // -1
    RAPP_CUDA(cudaMemsetAsync(t->d_fb_best, 0, (size_t)std::max(1, F) * 8, t->stream));
    w.fn_slo = t->d_slo;
    w.fn_fb = t->d_fb;
  }
  // rebuild the fresh-GPU search index (masked by the SLO when set) and the fallbacks
  for (int f0 = 0; f0 < F; f0 += 32768) {
    const int nf = std::min(F - f0, 32768);
    k_index_rps<<<dim3(64, nf), 256, 0, t->stream>>>(w, f0);
    RAPP_LAUNCHED();
    k_index_scan<<<nf, 1024, 0, t->stream>>>(w, f0);
    RAPP_LAUNCHED();
    if (slo_ms != nullptr) {
      k_index_fb<<<dim3(64, nf), 256, 0, t->stream>>>(w, f0, 0, t->d_fb_best);
      RAPP_LAUNCHED();
      k_index_fb<<<dim3(64, nf), 256, 0, t->stream>>>(w, f0, 1, t->d_fb_best);
      RAPP_LAUNCHED();
    }
  }
  RAPP_CUDA(cudaStreamSynchronize(t->stream));
  return RAPP_OK;
}

int rapp_tick_read_fns(rapp_tick* t, rapp_fn_desc* out) {
  if (!t || !out) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  World& w = t->w;
  const int F = w.F;
  std::vector<int32_t> init(F);
  std::vector<double> R(F), P(F), last(F);
  if (F) {
    RAPP_CUDA(cudaMemcpy(init.data(), w.k_init, F * 4, cudaMemcpyDeviceToHost));
    RAPP_CUDA(cudaMemcpy(R.data(), w.k_R, F * 8, cudaMemcpyDeviceToHost));
    RAPP_CUDA(cudaMemcpy(P.data(), w.k_P, F * 8, cudaMemcpyDeviceToHost));
    RAPP_CUDA(cudaMemcpy(last.data(), w.last_down, F * 8, cudaMemcpyDeviceToHost));
  }
  for (int f = 0; f < F; ++f) {
    out[f].kal_init = init[f];
    out[f].kal_R = R[f];
    out[f].kal_P = P[f];
    out[f].last_down_ms = last[f];
  }
  return RAPP_OK;
}

int rapp_tick_read_parts(rapp_tick* t, int64_t* part_off, int32_t* psm, int32_t* palloc,
                         int32_t* pnpods, int64_t cap) {
  if (!t || !part_off) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  World& w = t->w;
  std::vector<uint64_t> parts((size_t)w.G * kPartCap);
  std::vector<int32_t> nparts(w.G);
  if (w.G) {
    RAPP_CUDA(cudaMemcpy(parts.data(), w.g_parts, parts.size() * 8, cudaMemcpyDeviceToHost));
    RAPP_CUDA(cudaMemcpy(nparts.data(), w.g_nparts, w.G * 4, cudaMemcpyDeviceToHost));
  }
  int64_t k = 0;
  part_off[0] = 0;
  for (int g = 0; g < w.G; ++g) {
    for (int i = 0; i < nparts[g]; ++i) {
      if (k < cap) {
        const uint64_t e = parts[(size_t)g * kPartCap + i];
        if (psm) psm[k] = part_sm(e);
        if (palloc) palloc[k] = part_alloc(e);
        if (pnpods) pnpods[k] = part_npods(e);
      }
      ++k;
    }
    part_off[g + 1] = k;
  }
  return RAPP_OK;
}

int rapp_tick_counter(rapp_tick* t, int64_t* c) {
  if (!t || !c) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  RAPP_CUDA(cudaMemcpy(c, t->w.counter, 8, cudaMemcpyDeviceToHost));
  return RAPP_OK;
}

#ifdef RAPP_TICK_PROF
int rapp_tick_prof_read(uint64_t* out8, int reset) {
  RAPP_CUDA(cudaDeviceSynchronize());
  RAPP_CUDA(cudaMemcpyFromSymbol(out8, g_tick_prof, 256));
  if (reset) {
    uint64_t z[32] = {};
    RAPP_CUDA(cudaMemcpyToSymbol(g_tick_prof, z, 256));
  }
  return RAPP_OK;
}
#endif

}  // extern "C"
