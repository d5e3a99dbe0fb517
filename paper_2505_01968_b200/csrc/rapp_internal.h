// Host-side internals shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rapp_b200.h"

// NVTX ranges around the host entry points and the phases of a host tick (header-only
// NVTX3: a push/pop is a couple of branches when no profiler is attached; nsys / ncu
// --nvtx show them).  RAPP_NVTX=0 compiles them out.
#ifndef RAPP_NVTX
#define RAPP_NVTX 1
#endif
#if RAPP_NVTX
#include <nvtx3/nvToolsExt.h>
namespace rapp {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace rapp
#define RAPP_NVTX_CAT2(a, b) a##b
#define RAPP_NVTX_CAT(a, b) RAPP_NVTX_CAT2(a, b)
#define RAPP_RANGE(name) ::rapp::NvtxRange RAPP_NVTX_CAT(rapp_nvtx_, __LINE__)(name)
#else
#define RAPP_RANGE(name) (void)0
#endif

namespace rapp {

#ifndef RAPP_PDL
#define RAPP_PDL 1
#endif
// Launch with programmatic stream serialization (the kernel calls pdl_wait before it reads
// its predecessor's outputs; rapp_device.cuh).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = RAPP_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Thread-local error message behind rapp_last_error().
void set_error(const char* fmt, ...);
extern std::atomic<int64_t> g_launches;

#define RAPP_CUDA(expr)                                                                   \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      ::rapp::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__,     \
                        __LINE__, cudaGetErrorString(_e));                                \
      return RAPP_E_CUDA;                                                                 \
    }                                                                                     \
  } while (0)

#define RAPP_LAUNCHED()                                                                   \
  do {                                                                                    \
    ::rapp::g_launches.fetch_add(1, std::memory_order_relaxed);                           \
    cudaError_t _e = cudaGetLastError();                                                  \
    if (_e != cudaSuccess) {                                                              \
      ::rapp::set_error("kernel launch failed at %s:%d: %s", __FILE__, __LINE__,          \
                        cudaGetErrorString(_e));                                          \
      return RAPP_E_CUDA;                                                                 \
    }                                                                                     \
  } while (0)

// One immutable table inside the context's device pool.  Offsets are in doubles and
// even (16-byte aligned) so a table segment can be moved with one bulk copy:
//   [b_axis | pad][s_axis | pad][q_axis | pad][values | pad]
struct TableDesc {
  int32_t nb, ns, nq;
  int32_t seg_doubles;  // length of the whole segment (even)
  int64_t off;          // segment start in the pool
  int32_t ob, os, oq, ov;  // axis/value offsets relative to the segment start
  int32_t sm_keyable;       // sm axis integral in [0, 2^24): usable in packed search keys
  // fast-path extras (rapp_stream.cu), present when fast != 0 (strictly ascending axes)
  int32_t fast;
  int32_t x_small, x_total;             // doubles: small part (-> smem), whole extras
  int32_t x_iv_b, x_iv_s, x_iv_q;       // interval-table offsets inside the extras
  int32_t modes;                        // FastLayout::modes
  int64_t xoff;                         // extras start in the pool
};

inline int32_t pad2(int64_t n) { return int32_t((n + 1) & ~int64_t(1)); }

// Host pipeline resources for host-pointer entry points.
struct HostPipe {
  static constexpr int kDepth = 3;
  cudaStream_t stream[kDepth] = {};
  cudaEvent_t done[kDepth] = {};
  double* h_in[kDepth] = {};
  double* h_out[kDepth] = {};
  double* d_in[kDepth] = {};
  double* d_out[kDepth] = {};
  int64_t rows = 0;  // capacity per stage (rows of 3 doubles in, 1 double out)
};

}  // namespace rapp

struct rapp_ctx {
  int device = 0;
  int sm_count = 0;
  std::mutex mu;
  std::vector<rapp::TableDesc> tables;  // host mirror of d_desc
  double* d_pool = nullptr;
  int64_t pool_cap = 0, pool_used = 0;  // doubles
  rapp::TableDesc* d_desc = nullptr;
  int64_t desc_cap = 0;
  // scratch table for the stateless reference-shaped entry points
  int32_t scratch_table = -1;
  int32_t scratch_cap = 0;  // reserved doubles of the scratch segment
  bool interp_attr_set = false;
  bool fast_attr_set = false;
  bool force_literal = false;  // RAPP_FORCE_LITERAL=1: always use the literal K2 kernel
  rapp::HostPipe pipe;
  // stateless entry points (rapp_interp3_many & co. take raw axes + values per call): the
  // last few distinct tables stay resident, matched by exact content, so repeated calls on
  // the same table skip the upload and the fast-path build
  struct StatelessTable {
    std::vector<double> key;  // nb, ns, nq, axes, values (exact comparison)
    uint64_t hash = 0;
    int32_t id = -1;
    int64_t cap = 0;         // doubles reserved in the pool for this slot
    uint64_t used = 0;       // LRU stamp
  };
  std::vector<StatelessTable> stateless;
  uint64_t stateless_clock = 0;
  double* d_small = nullptr;  // 64 doubles of scratch for scalar calls
  // small-batch point evaluation (rapp_table_points / rapp_locate): pinned staging
  // [coords 3n | latency n | rps n] mirrored on the device, one stream, grown on demand,
  // so a scalar predict_latency / throughput is one H2D, one launch, one D2H — no
  // allocation per call
  cudaStream_t pts_stream = nullptr;
  double* h_pts = nullptr;
  double* d_pts = nullptr;
  int64_t pts_rows = 0;      // rows the staging holds
};

namespace rapp {
// Appends a table to the pool (or overwrites the scratch slot when scratch == true).
int table_put(rapp_ctx* ctx, int64_t nb, int64_t ns, int64_t nq, const double* b,
              const double* s, const double* q, const double* v, bool scratch,
              int32_t* id, int32_t reuse_slot = -1, int64_t reuse_cap = 0,
              int64_t* total_out = nullptr);
// The per-device default context used by the stateless entry points.
int default_ctx(rapp_ctx** out);
int ensure_pipe(rapp_ctx* ctx, int64_t rows);
// chunked, stream-overlapped host->device->host pipeline over (n,3) coords -> (n) out
int pipe_run(rapp_ctx* ctx, const double* coords, int64_t n, double* out,
             const std::function<int(const double*, int64_t, double*, cudaStream_t)>& launch);
// fast-path extras layout (doubles, see rapp_stream.cu):
//   [params 3 x 8][lut_b|lut_s|lut_q int32 x kLut each][iv_b|iv_s|iv_q (2n each)][pad][cells]
struct FastLayout {
  int32_t o_par, o_lut, o_iv_b, o_iv_s, o_iv_q, o_cells, small_doubles, total_doubles;
  int32_t modes;  // bit a: axis a (0=b, 1=s, 2=q) is an exact power-of-two-step grid
};
int build_fast_extras(int64_t nb, int64_t ns, int64_t nq, const double* b, const double* s,
                      const double* q, const double* v, std::vector<double>& ext,
                      FastLayout& L);
int launch_interp_fast(rapp_ctx* ctx, const TableDesc& td, const double* d_coords, int64_t n,
                       double* d_out, double* d_rps, cudaStream_t st);
// Launches the stream-interpolation kernel for one table.
int launch_interp(rapp_ctx* ctx, int32_t table_id, const double* d_coords, int64_t n,
                  double* d_out, double* d_rps, cudaStream_t st);
}  // namespace rapp

// the tick worlds' allocation cache (rapp_tick.cu), emptied by rapp_shutdown
extern "C" int rapp_tick_pool_drain(int device);
