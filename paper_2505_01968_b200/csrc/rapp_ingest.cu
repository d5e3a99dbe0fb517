// Perf-table ingest: CSV rows -> validated (batch x sm x quota) grid, hs/perf.py:155-267.
//
// The reference parses rows into a {(b, s, q): latency} dict (first occurrence wins, later
// ones are "duplicate" issues, perf.py:175-206), takes the sorted distinct values of each
// coordinate as the axes, scatters the samples into the grid reporting every empty cell as
// "missing" (perf.py:209-227), and — only when no cell is missing — flags every cell that
// is non-positive or breaks monotonicity along batch (non-decreasing), sm and quota
// (non-increasing) (perf.py:239-267), in C order, per cell in that kind order.
//
// Here the per-sample and per-cell work runs on the device:
//   k_ing_insert   distinct values of each coordinate column (open-addressing hash sets)
//   k_ing_rank     rank of each distinct value = number of smaller distinct values (the
//                  axes are short; O(k^2) compares in parallel, no sort needed)
//   k_ing_scatter  cell index of every sample; atomicMin keeps the first row of each cell
//   k_ing_fill     grid value from the first row; every later row of a cell is a duplicate
//   k_ing_check    per-cell flags: missing, then (when nothing is missing) the stencil
// The host reads back the axes, the grid, one flag byte per cell and one per row, and
// formats messages only for flagged entries.
//
// rapp_csv_parse is the native row reader for the strict common form of the file
// (`fid,int,int,int,float` lines, one function id, no quoting or padding); anything else
// is reported as irregular and the caller reads the file with the csv module instead,
// which reproduces the reference's own format-error messages.
#include <cerrno>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "rapp_internal.h"

namespace rapp {

constexpr unsigned long long kEmptyKey = 0x8000000000000000ull;  // INT64_MIN: never a key

__device__ __forceinline__ uint32_t hash64(uint64_t x, uint32_t mask) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return uint32_t(x) & mask;
}

struct IngestDev {
  int64_t n;
  const int64_t* col[3];           // batch, sm, quota per row
  const double* lat;
  unsigned long long* keys[3];     // hash sets (cap entries each)
  int32_t* slot_rank[3];           // rank of the key in each slot
  uint32_t mask;
  int64_t* distinct[3];            // compacted distinct values (<= n each)
  int32_t* ndist;                  // [3]
  int64_t* axis[3];                // sorted distinct values
  int64_t* cell;                   // per row: cell index
  unsigned long long* first;       // per cell: first row index (ULLONG_MAX: none)
  double* grid;
  uint8_t* cflags;                 // per cell
  uint8_t* rdup;                   // per row: 1 = duplicate of an earlier row
  int32_t* counts;                 // [0] missing cells, [1] flagged cells, [2] duplicates
  int64_t nb, ns, nq;
};

__device__ int32_t* slot_of(const IngestDev& d, int a, int64_t key) {
  uint32_t h = hash64(uint64_t(key), d.mask);
  while (true) {
    const unsigned long long k = d.keys[a][h];
    if (k == (unsigned long long)key) return d.slot_rank[a] + h;
    h = (h + 1) & d.mask;  // the key is present: the probe ends
  }
}

__global__ void k_ing_init(IngestDev d, uint32_t cap) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x)
    for (int a = 0; a < 3; ++a) d.keys[a][i] = kEmptyKey;
  if (blockIdx.x == 0 && threadIdx.x < 4) {
    d.ndist[threadIdx.x] = 0;
    d.counts[threadIdx.x] = 0;
  }
}

__global__ void k_ing_insert(IngestDev d) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < d.n;
       i += int64_t(gridDim.x) * blockDim.x) {
    for (int a = 0; a < 3; ++a) {
      const unsigned long long key = (unsigned long long)d.col[a][i];
      uint32_t h = hash64(key, d.mask);
      while (true) {
        const unsigned long long prev = atomicCAS(d.keys[a] + h, kEmptyKey, key);
        if (prev == kEmptyKey) {  // first insertion of this value
          const int32_t j = atomicAdd(d.ndist + a, 1);
          d.distinct[a][j] = int64_t(key);
          break;
        }
        if (prev == key) break;
        h = (h + 1) & d.mask;
      }
    }
  }
}

// one thread per distinct value of one axis (grid.y = axis)
__global__ void k_ing_rank(IngestDev d) {
  const int a = blockIdx.y;
  const int32_t k = d.ndist[a];
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    const int64_t v = d.distinct[a][j];
    int32_t r = 0;
    for (int32_t i = 0; i < k; ++i) r += d.distinct[a][i] < v;
    *slot_of(d, a, v) = r;
    d.axis[a][r] = v;
  }
}

__global__ void k_ing_scatter(IngestDev d) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < d.n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t rb = *slot_of(d, 0, d.col[0][i]);
    const int64_t rs = *slot_of(d, 1, d.col[1][i]);
    const int64_t rq = *slot_of(d, 2, d.col[2][i]);
    const int64_t c = (rb * d.ns + rs) * d.nq + rq;
    d.cell[i] = c;
    atomicMin(d.first + c, (unsigned long long)i);
  }
}

__global__ void k_ing_fill(IngestDev d) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < d.n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = d.cell[i];
    const bool dup = d.first[c] != (unsigned long long)i;
    d.rdup[i] = dup ? 1 : 0;
    if (dup)
      atomicAdd(d.counts + 2, 1);
    else
      d.grid[c] = d.lat[i];
  }
}

// flag bits: 1 missing, 2 non_positive, 4 batch decreases, 8 sm increases, 16 quota increases
__global__ void k_ing_missing(IngestDev d) {
  const int64_t cells = d.nb * d.ns * d.nq;
  int32_t miss = 0;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cells;
       c += int64_t(gridDim.x) * blockDim.x) {
    const bool m = d.first[c] == ~0ull;
    d.cflags[c] = m ? 1 : 0;
    if (m) d.grid[c] = 0.0;  // np.zeros in the reference
    miss += m;
  }
  for (int o = 16; o > 0; o >>= 1) miss += __shfl_xor_sync(0xffffffffu, miss, o);
  if ((threadIdx.x & 31) == 0 && miss) atomicAdd(d.counts, miss);
}

__global__ void k_ing_check(IngestDev d) {
  if (d.counts[0] != 0) return;  // skip_shape (perf.py:225-226, 242-243)
  const int64_t cells = d.nb * d.ns * d.nq;
  const int64_t sq = d.ns * d.nq;
  int32_t flagged = 0;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cells;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t bi = c / sq, si = (c / d.nq) % d.ns, qi = c % d.nq;
    const double v = d.grid[c];
    uint8_t f = 0;
    if (v <= 0.0) f |= 2;                                  // NaN passes, as in Python
    if (bi > 0 && d.grid[c - sq] > v) f |= 4;
    if (si > 0 && d.grid[c - d.nq] < v) f |= 8;
    if (qi > 0 && d.grid[c - 1] < v) f |= 16;
    d.cflags[c] = f;
    flagged += f != 0;
  }
  for (int o = 16; o > 0; o >>= 1) flagged += __shfl_xor_sync(0xffffffffu, flagged, o);
  if ((threadIdx.x & 31) == 0 && flagged) atomicAdd(d.counts + 1, flagged);
}

// ---- strict native CSV row reader -----------------------------------------------------

static bool parse_int(const char* p, const char* e, int64_t* out) {
  if (p == e) return false;
  bool neg = false;
  if (*p == '+' || *p == '-') {
    neg = *p == '-';
    if (++p == e) return false;
  }
  if (e - p > 18) return false;  // stay far inside int64 (longer: irregular)
  int64_t v = 0;
  for (; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    v = v * 10 + (*p - '0');
  }
  *out = neg ? -v : v;
  return true;
}

// decimal literal [+-]digits[.digits][(e|E)[+-]digits] -> strtod (correctly rounded, the
// same double Python's float() returns for such a literal)
static bool parse_float(const char* p, const char* e, double* out) {
  const char* s = p;
  if (s < e && (*s == '+' || *s == '-')) ++s;
  int digits = 0;
  while (s < e && *s >= '0' && *s <= '9') ++s, ++digits;
  if (s < e && *s == '.') {
    ++s;
    while (s < e && *s >= '0' && *s <= '9') ++s, ++digits;
  }
  if (digits == 0) return false;
  if (s < e && (*s == 'e' || *s == 'E')) {
    ++s;
    if (s < e && (*s == '+' || *s == '-')) ++s;
    int ed = 0;
    while (s < e && *s >= '0' && *s <= '9') ++s, ++ed;
    if (ed == 0) return false;
  }
  if (s != e || e - p > 400) return false;
  char buf[408];
  std::memcpy(buf, p, size_t(e - p));
  buf[e - p] = 0;
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(buf, &end);
  if (end != buf + (e - p)) return false;
  *out = v;  // overflow gives inf like float('1e999'); underflow gives 0/denormal likewise
  return true;
}

}  // namespace rapp

using namespace rapp;

struct rapp_ingest {
  rapp_ctx* ctx = nullptr;
  int64_t n = 0, nb = 0, ns = 0, nq = 0;
  int32_t counts[3] = {0, 0, 0};
  std::vector<void*> allocs;
  IngestDev d{};
};

extern "C" {

int rapp_csv_parse(const char* buf, int64_t len, int64_t cap, int64_t* batch, int64_t* sm,
                   int64_t* quota, double* lat, int64_t* n_rows, char* fid, int64_t fid_cap,
                   int32_t* regular) {
  if (!buf || len < 0 || !n_rows || !regular || !fid || fid_cap < 1) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  *regular = 0;
  *n_rows = 0;
  fid[0] = 0;
  static const char kHeader[] = "function_id,batch,sm_percent,quota_percent,latency_ms";
  const char* p = buf;
  const char* end = buf + len;
  auto line_end = [&](const char* s) {
    const char* e = static_cast<const char*>(std::memchr(s, '\n', size_t(end - s)));
    return e ? e : end;
  };
  const char* e = line_end(p);
  const char* he = (e > p && e[-1] == '\r') ? e - 1 : e;
  if (size_t(he - p) != sizeof(kHeader) - 1 || std::memcmp(p, kHeader, sizeof(kHeader) - 1))
    return RAPP_OK;  // irregular (the csv path reports the header issue)
  p = e < end ? e + 1 : end;
  const char* id0 = nullptr;
  size_t idlen = 0;
  int64_t n = 0;
  while (p < end) {
    e = line_end(p);
    const char* le = (e > p && e[-1] == '\r') ? e - 1 : e;
    if (le == p) return RAPP_OK;  // blank line: irregular
    const char* f[6];
    int nf = 0;
    f[nf++] = p;
    for (const char* s = p; s < le; ++s) {
      if (*s == ',') {
        if (nf == 5) return RAPP_OK;  // extra fields: irregular
        f[nf++] = s + 1;
      } else if (*s == '"' || *s == ' ' || (unsigned char)*s < 0x20 ||
                 (unsigned char)*s >= 0x80) {
        return RAPP_OK;  // quoting, padding, control or non-ASCII bytes: irregular
      }
    }
    if (nf != 5) return RAPP_OK;
    f[5] = le + 1;
    const size_t L0 = size_t(f[1] - 1 - f[0]);
    if (L0 == 0) return RAPP_OK;
    if (!id0) {
      id0 = f[0];
      idlen = L0;
      if ((int64_t)idlen + 1 > fid_cap) return RAPP_OK;
    } else if (L0 != idlen || std::memcmp(f[0], id0, idlen)) {
      return RAPP_OK;  // mixed ids: irregular
    }
    if (n >= cap) {
      set_error("row capacity %lld exceeded", (long long)cap);
      return RAPP_E_ARG;
    }
    int64_t b, s, q;
    double v;
    if (!parse_int(f[1], f[2] - 1, &b) || !parse_int(f[2], f[3] - 1, &s) ||
        !parse_int(f[3], f[4] - 1, &q) || !parse_float(f[4], f[5] - 1, &v))
      return RAPP_OK;
    batch[n] = b;
    sm[n] = s;
    quota[n] = q;
    lat[n] = v;
    ++n;
    p = e < end ? e + 1 : end;
  }
  if (n == 0) return RAPP_OK;  // empty table: irregular (the csv path reports it)
  std::memcpy(fid, id0, idlen);
  fid[idlen] = 0;
  *n_rows = n;
  *regular = 1;
  return RAPP_OK;
}

int rapp_ingest_create(rapp_ctx* ctx, int64_t n, const int64_t* batch, const int64_t* sm,
                       const int64_t* quota, const double* lat, rapp_ingest** out) {
  RAPP_RANGE("rapp_ingest_create");
  if (!ctx || !out || n < 1 || !batch || !sm || !quota || !lat) {
    set_error("null argument or empty sample set");
    return RAPP_E_ARG;
  }
  const int64_t* cols[3] = {batch, sm, quota};
  for (int a = 0; a < 3; ++a)
    for (int64_t i = 0; i < n; ++i)
      if ((unsigned long long)cols[a][i] == kEmptyKey) {
        set_error("coordinate %lld out of range", (long long)cols[a][i]);
        return RAPP_E_TABLE;
      }
  std::unique_ptr<rapp_ingest> ing(new rapp_ingest());
  ing->ctx = ctx;
  ing->n = n;
  RAPP_CUDA(cudaSetDevice(ctx->device));
  IngestDev& d = ing->d;
  d.n = n;
  uint32_t cap = 1;
  while (cap < 2 * uint64_t(n)) cap <<= 1;
  d.mask = cap - 1;
  // one device allocation for every per-row and per-slot array (cells come later)
  const size_t per_axis = size_t(n) * 8 * 3 + size_t(cap) * 12;  // col, distinct, axis; keys, rank
  const size_t bytes = 3 * per_axis + size_t(n) * 8 * 3 + size_t(n) + 1024;  // + rounding
  char* base = nullptr;
  RAPP_CUDA(cudaMalloc(&base, bytes));
  ing->allocs.push_back(base);
  char* cur = base;
  auto take = [&](size_t b) {
    char* r = cur;
    cur += (b + 15) & ~size_t(15);
    return r;
  };
  for (int a = 0; a < 3; ++a) d.col[a] = reinterpret_cast<const int64_t*>(take(size_t(n) * 8));
  d.lat = reinterpret_cast<const double*>(take(size_t(n) * 8));
  {  // columns + latencies staged in the device layout: one H2D copy
    const size_t stride = ((size_t(n) * 8 + 15) & ~size_t(15)) / 8;  // take() rounding
    std::vector<int64_t> staged(stride * 4);
    for (int a = 0; a < 3; ++a) std::memcpy(staged.data() + stride * a, cols[a], size_t(n) * 8);
    std::memcpy(staged.data() + stride * 3, lat, size_t(n) * 8);
    RAPP_CUDA(cudaMemcpy((void*)d.col[0], staged.data(), stride * 32, cudaMemcpyHostToDevice));
  }
  for (int a = 0; a < 3; ++a) {
    d.keys[a] = reinterpret_cast<unsigned long long*>(take(size_t(cap) * 8));
    d.slot_rank[a] = reinterpret_cast<int32_t*>(take(size_t(cap) * 4));
    d.distinct[a] = reinterpret_cast<int64_t*>(take(size_t(n) * 8));
    d.axis[a] = reinterpret_cast<int64_t*>(take(size_t(n) * 8));
  }
  d.ndist = reinterpret_cast<int32_t*>(take(16));
  d.counts = reinterpret_cast<int32_t*>(take(16));
  d.cell = reinterpret_cast<int64_t*>(take(size_t(n) * 8));
  d.rdup = reinterpret_cast<uint8_t*>(take(size_t(n)));
  if (size_t(cur - base) > bytes) {
    set_error("ingest scratch layout overflow");
    return RAPP_E_ARG;
  }
  k_ing_init<<<(unsigned)std::min<int64_t>((cap + 255) / 256, int64_t(ctx->sm_count) * 8), 256>>>(d, cap);
  RAPP_LAUNCHED();
  int rc;
  auto alloc = [&](void** p, size_t b) -> int {
    RAPP_CUDA(cudaMalloc(p, b ? b : 8));
    ing->allocs.push_back(*p);
    return RAPP_OK;
  };
  const int threads = 256;
  const unsigned rows_blocks =
      (unsigned)std::min<int64_t>((n + threads - 1) / threads, int64_t(ctx->sm_count) * 8);
  k_ing_insert<<<rows_blocks, threads>>>(d);
  RAPP_LAUNCHED();
  int32_t nd[3];
  RAPP_CUDA(cudaMemcpy(nd, d.ndist, 12, cudaMemcpyDeviceToHost));
  d.nb = nd[0];
  d.ns = nd[1];
  d.nq = nd[2];
  const int64_t cells = d.nb * d.ns * d.nq;
  if (cells > (int64_t(1) << 28)) {
    set_error("grid of %lld x %lld x %lld cells is too large", (long long)d.nb,
              (long long)d.ns, (long long)d.nq);
    return RAPP_E_TABLE;
  }
  const int32_t kmax = std::max(nd[0], std::max(nd[1], nd[2]));
  k_ing_rank<<<dim3((unsigned)std::max(1, (kmax + threads - 1) / threads), 3), threads>>>(d);
  RAPP_LAUNCHED();
  {  // per-cell arrays in one allocation
    char* cb = nullptr;
    if ((rc = alloc((void**)&cb, size_t(cells) * 17 + 32))) return rc;
    d.first = reinterpret_cast<unsigned long long*>(cb);
    d.grid = reinterpret_cast<double*>(cb + size_t(cells) * 8);
    d.cflags = reinterpret_cast<uint8_t*>(cb + size_t(cells) * 16);
    RAPP_CUDA(cudaMemsetAsync(d.first, 0xFF, size_t(cells) * 8));
  }
  k_ing_scatter<<<rows_blocks, threads>>>(d);
  RAPP_LAUNCHED();
  k_ing_fill<<<rows_blocks, threads>>>(d);
  RAPP_LAUNCHED();
  const unsigned cell_blocks =
      (unsigned)std::min<int64_t>((cells + threads - 1) / threads, int64_t(ctx->sm_count) * 8);
  k_ing_missing<<<std::max(1u, cell_blocks), threads>>>(d);
  RAPP_LAUNCHED();
  k_ing_check<<<std::max(1u, cell_blocks), threads>>>(d);
  RAPP_LAUNCHED();
  RAPP_CUDA(cudaMemcpy(ing->counts, d.counts, 12, cudaMemcpyDeviceToHost));
  ing->nb = d.nb;
  ing->ns = d.ns;
  ing->nq = d.nq;
  *out = ing.release();
  return RAPP_OK;
}

int rapp_ingest_shape(rapp_ingest* ing, int64_t* nb, int64_t* ns, int64_t* nq,
                      int32_t* n_missing, int32_t* n_flagged, int32_t* n_duplicates) {
  if (!ing) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  if (nb) *nb = ing->nb;
  if (ns) *ns = ing->ns;
  if (nq) *nq = ing->nq;
  if (n_missing) *n_missing = ing->counts[0];
  if (n_flagged) *n_flagged = ing->counts[1];
  if (n_duplicates) *n_duplicates = ing->counts[2];
  return RAPP_OK;
}

int rapp_ingest_read(rapp_ingest* ing, int64_t* b_axis, int64_t* s_axis, int64_t* q_axis,
                     double* grid, uint8_t* cell_flags, uint8_t* row_dup) {
  if (!ing) {
    set_error("null argument");
    return RAPP_E_ARG;
  }
  RAPP_CUDA(cudaSetDevice(ing->ctx->device));
  const IngestDev& d = ing->d;
  const int64_t cells = d.nb * d.ns * d.nq;
  if (b_axis) RAPP_CUDA(cudaMemcpy(b_axis, d.axis[0], d.nb * 8, cudaMemcpyDeviceToHost));
  if (s_axis) RAPP_CUDA(cudaMemcpy(s_axis, d.axis[1], d.ns * 8, cudaMemcpyDeviceToHost));
  if (q_axis) RAPP_CUDA(cudaMemcpy(q_axis, d.axis[2], d.nq * 8, cudaMemcpyDeviceToHost));
  if (grid) RAPP_CUDA(cudaMemcpy(grid, d.grid, cells * 8, cudaMemcpyDeviceToHost));
  if (cell_flags) RAPP_CUDA(cudaMemcpy(cell_flags, d.cflags, cells, cudaMemcpyDeviceToHost));
  if (row_dup) RAPP_CUDA(cudaMemcpy(row_dup, d.rdup, d.n, cudaMemcpyDeviceToHost));
  return RAPP_OK;
}

int rapp_ingest_destroy(rapp_ingest* ing) {
  if (!ing) return RAPP_OK;
  cudaSetDevice(ing->ctx->device);
  for (void* p : ing->allocs) cudaFree(p);
  delete ing;
  return RAPP_OK;
}

}  // extern "C"
