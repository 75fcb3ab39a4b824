// Row-slab sharded factorized solve across GPUs (BASELINE config 4 on 8 GPUs,
// SURVEY.md §8(e)): rank g owns rows [row0_g, row0_g+rows_g) of W, t, Z, B, x.
//
// Per application t_out = t_in − θ·W·t_in each rank needs t_in at the columns
// its rows reference outside its slab — for a banded operator (the 5-point
// Laplacian: one grid row, 4096 values, on each side) those are the last
// h_lo rows of rank g−1 and the first h_hi rows of rank g+1.  Vectors are
// kept "extended" ([h_lo halo | own rows | h_hi halo]) and the local CSR
// columns are remapped into that layout once, so the single-GPU kernel runs
// unchanged.  Each application:
//   1. halo exchange: NCCL send/recv with both neighbours on a side stream;
//   2. interior rows (no halo reference) on the compute stream meanwhile;
//   3. boundary rows once the halo has landed.
// Arithmetic is the bit-exact reference-ordered kernel of sparse.cu, and a
// row's sum never depends on the partition, so the sharded x is
// BIT-IDENTICAL to the single-GPU x and to the reference's for any world.
//
// Emulation: `world` virtual ranks in one process on one GPU, halos moved by
// device copies — validates partition, remap, halo sizes and the
// interior/boundary split on a single device.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "../../include/nnb.h"
#include "comm.cuh"
#include "engine.cuh"
#include "sparse.cuh"

namespace nnb {
namespace sparse_detail {

thread_local double g_last_solve_ms = 0.0;  // nnb_sparse_last_solve_ms

// CUDA-event bracket of a solve's schedule on stream s
struct SolveTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit SolveTimer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  void stop() {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    g_last_solve_ms = ms;
  }
  ~SolveTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

#define NNB_NCCL2(x)                                                                             \
  do {                                                                                           \
    ncclResult_t _r = (x);                                                                       \
    if (_r != ncclSuccess) return fail(NNB_ERR_NCCL, std::string("NCCL error: ") + nccl_error(_r)); \
  } while (0)

// Per-slab statistics: min/max column, last row referencing below the slab,
// first row referencing above it.  Each thread folds its rows, then a warp reduction and
// one atomic per warp and statistic (per-row atomics on the same four words serialised:
// 23 ms of a 4096² slab's setup).
__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ long long warp_max_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__global__ void slab_stats_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t rows,
                                  int64_t row0, int64_t* __restrict__ stats /* [min_col, max_col, lo_end, hi_start] */) {
  long long mn_all = LLONG_MAX, mx_all = -1, lo_end = 0, hi_start = LLONG_MAX;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t start = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t r = start; r - threadIdx.x % 32 < rows; r += stride) {  // warp-uniform trip count
    if (r < rows) {
      long long mn = LLONG_MAX, mx = -1;
      for (int64_t e = rp[r] - rp[0]; e < rp[r + 1] - rp[0]; ++e) {
        const long long c = col[e];
        mn = c < mn ? c : mn;
        mx = c > mx ? c : mx;
      }
      if (mx >= 0) {  // empty rows contribute nothing
        mn_all = min(mn_all, mn);
        mx_all = max(mx_all, mx);
        if (mn < row0) lo_end = max(lo_end, (long long)(r + 1));
        if (mx >= row0 + rows) hi_start = min(hi_start, (long long)r);
      }
    }
  }
  mn_all = warp_min_ll(mn_all);
  mx_all = warp_max_ll(mx_all);
  lo_end = warp_max_ll(lo_end);
  hi_start = warp_min_ll(hi_start);
  if ((threadIdx.x & 31) == 0) {
    if (mx_all >= 0) {
      atomicMin(reinterpret_cast<unsigned long long*>(stats + 0), static_cast<unsigned long long>(mn_all));
      atomicMax(reinterpret_cast<unsigned long long*>(stats + 1), static_cast<unsigned long long>(mx_all));
    }
    if (lo_end > 0) atomicMax(reinterpret_cast<unsigned long long*>(stats + 2), static_cast<unsigned long long>(lo_end));
    if (hi_start != LLONG_MAX)
      atomicMin(reinterpret_cast<unsigned long long*>(stats + 3), static_cast<unsigned long long>(hi_start));
  }
}

__global__ void remap_cols_kernel(const int32_t* __restrict__ col, int64_t nnz, int64_t shift, int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = static_cast<int32_t>(col[e] + shift);
}

struct Slab {
  int64_t row0 = 0, rows = 0, nnz = 0;
  int64_t h_lo = 0, h_hi = 0;           // halo rows received from g−1 / g+1
  int64_t lo_end = 0, hi_start = 0;     // interior = [lo_end, hi_start)
  int64_t send_prev = 0, send_next = 0; // rows g−1 / g+1 need from us
  DevBuf mem;
  int32_t* rp = nullptr;                // local int32 offsets
  int32_t* col = nullptr;               // remapped into the extended layout (wide operators)
  int16_t* col16 = nullptr;             // column − global row (banded operators), else null
  const double* val = nullptr;
  double* ext[5] = {};                  // T0, T1, Z0, Z1, B (extended)
  int* flags = nullptr;                 // [64]
  // pair / row dictionaries of the slab (one right-hand side), as sparse.cu's single-GPU solve
  DevBuf dict_mem, code_mem, rowdict_mem;
  const uint8_t* code = nullptr;
  const int32_t* dict_delta = nullptr;
  const double* dict_val = nullptr;
  int dict_size = 0, ell_width = 0, band_lo = 0, band_hi = 0;
  int64_t ell_rows = 0;
  const uint8_t* rcode = nullptr;
  const double2* rpat = nullptr;
  const uint8_t* rlen = nullptr;
  int npat = 0;
  int64_t ext_len() const { return h_lo + rows + h_hi; }
  // temporal blocking across slabs (5-point stencils, slabs whole grid rows): the slab's
  // grid rows plus tb_rows() halo rows on each inner side, codes in the global pattern table
  bool tb = false;
  int tbW = 0;
  int64_t tb_lo = 0, tb_hi = 0;  // halo cells above / below (0 at the grid's edges)
  DevBuf tb_mem;
  uint8_t* tb_code = nullptr;
  double* tb_ext[6] = {};        // T0, T1, Z0, Z1, B, X over the extended rows
  int64_t tb_len() const { return tb_lo + rows + tb_hi; }
};

// what every rank contributes to the temporal-blocking decision (gathered, then decided
// identically everywhere): its W (0: not a stencil slab), whether its own edge rows are
// clean, and its row-pattern table
struct TbRecord {
  double w = 0, edges_ok = 0, npat = 0, pad = 0;
  StencilPattern tab[kRowDictMax];
};
// halo grid rows = the most applications a slab pass runs
constexpr int tb_rows() { return kStencilDepthSlab; }

// the slab's own-pattern record (W, edge check over its own rows, table)
int tb_record(const Slab& sl, int64_t n, TbRecord* rec, cudaStream_t s) {
  *rec = TbRecord{};
  if (!sl.rcode || sl.rows == 0) return 0;
  int64_t w = 0;
  std::vector<StencilPattern> tab;
  NNB_TRY(stencil_patterns(sl.rpat, sl.rlen, sl.npat, sl.ell_width, &w, tab, s));
  if (!w || sl.row0 % w || sl.rows % w || n % w || sl.rows / w > INT32_MAX) return 0;
  DevBuf t;
  NNB_TRY(t.alloc(sizeof(StencilPattern) * tab.size(), s));
  NNB_CUDA(cudaMemcpyAsync(t.p, tab.data(), sizeof(StencilPattern) * tab.size(), cudaMemcpyHostToDevice, s));
  bool ok = false;
  NNB_TRY(stencil_edges_ok(sl.rcode, t.as<StencilPattern>(), (int)w, (int)(sl.rows / w), sl.row0 == 0,
                           sl.row0 + sl.rows == n, &ok, s));
  rec->w = (double)w;
  rec->edges_ok = ok ? 1.0 : 0.0;
  rec->npat = (double)tab.size();
  std::copy(tab.begin(), tab.end(), rec->tab);
  return 0;
}

// Decides temporal blocking from every rank's record (identical on every rank): one W, the
// grid rows whole per slab, every slab at least tb_rows() rows (each neighbour's halo comes
// from one slab), clean edges, and at most kRowDictMax patterns in the union of the tables
// (in rank order).  map[g][c]: rank g's code c in the union.
bool tb_decide(const std::vector<TbRecord>& recs, const std::vector<int64_t>& rows, std::vector<StencilPattern>& table,
               std::vector<std::vector<uint8_t>>& map) {
  const int G = (int)recs.size();
  const double w = recs[0].w;
  if (w <= 0) return false;
  for (int g = 0; g < G; ++g)
    if (recs[g].w != w || recs[g].edges_ok != 1.0 || rows[g] < tb_rows() * (int64_t)w) return false;
  table.clear();
  map.assign(G, std::vector<uint8_t>(kRowDictMax, 0));
  for (int g = 0; g < G; ++g)
    for (int c = 0; c < (int)recs[g].npat; ++c) {
      int found = -1;
      for (size_t i = 0; i < table.size() && found < 0; ++i)
        if (std::memcmp(&table[i], &recs[g].tab[c], sizeof(StencilPattern)) == 0) found = (int)i;
      if (found < 0) {
        if (table.size() >= (size_t)kRowDictMax) return false;
        found = (int)table.size();
        table.push_back(recs[g].tab[c]);
      }
      map[g][c] = (uint8_t)found;
    }
  return true;
}

__global__ void remap_codes_kernel(const uint8_t* __restrict__ in, int64_t count, const uint8_t* __restrict__ lut,
                                   uint8_t* __restrict__ out) {
  __shared__ uint8_t l[kRowDictMax];
  for (int i = threadIdx.x; i < kRowDictMax; i += blockDim.x) l[i] = lut[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = l[in[i]];
}

// The slab's extended-grid buffers and its own codes in the union table.
int tb_setup_slab(Slab& sl, int64_t n, int W, const std::vector<uint8_t>& lut, cudaStream_t s) {
  sl.tb = true;
  sl.tbW = W;
  sl.tb_lo = sl.row0 > 0 ? (int64_t)tb_rows() * W : 0;
  sl.tb_hi = sl.row0 + sl.rows < n ? (int64_t)tb_rows() * W : 0;
  const int64_t len = sl.tb_len();
  NNB_TRY(sl.tb_mem.alloc(sizeof(double) * 6 * len + len + kRowDictMax + 64, s));
  double* d = sl.tb_mem.as<double>();
  for (int i = 0; i < 6; ++i) sl.tb_ext[i] = d + i * len;
  NNB_CUDA(cudaMemsetAsync(d, 0, sizeof(double) * 6 * len, s));
  sl.tb_code = reinterpret_cast<uint8_t*>(d + 6 * len);
  uint8_t* lut_d = sl.tb_code + len;
  NNB_CUDA(cudaMemsetAsync(sl.tb_code, 0, len, s));
  NNB_CUDA(cudaMemcpyAsync(lut_d, lut.data(), kRowDictMax, cudaMemcpyHostToDevice, s));
  remap_codes_kernel<<<std::max<int64_t>(1, std::min<int64_t>(1184, (sl.rows + 255) / 256)), 256, 0, s>>>(
      sl.rcode, sl.rows, lut_d, sl.tb_code + sl.tb_lo);
  count_launch();
  NNB_CUDA(cudaStreamSynchronize(s));  // the LUT is a host vector's copy
  NNB_CUDA(cudaGetLastError());
  return 0;
}

// The temporal-blocked factorized solve over row slabs: per pass (up to tb_rows()
// applications, sparse_stencil.cu) the tb_rows()·W halo cells of its input are exchanged
// once, then each slab runs the pass over its extended grid; the halo rows' values go
// stale from the outside in, one row per application, never reaching the slab's own rows.
// Each own row is computed as in the single-GPU pass (bitwise the same inputs), so x stays
// bit-identical.  With a real exchange (`bs` = the communication stream) the tile rows
// whose region stays clear of the halo rows run on s while the exchange is in flight, and
// the edge tile rows run on bs right behind the exchange — at its higher priority, filling
// the interior launch's last wave — before s joins it (`join()`).  Without one (bs null:
// the emulation's device copies) each slab's pass is one launch.
template <class Exchange, class Join>
int run_slabs_tb(std::vector<Slab*>& slabs, const StencilPattern* table, int npat, int s_factors, double theta,
                 std::vector<double*>& x_own, Exchange exchange, Join join, cudaStream_t s, cudaStream_t bs) {
  const int kmax = kStencilDepthSlab, ty = stencil_tile_rows(kStencilDepthSlab);
  int zcur = 4, zi = 0;  // Z starts as B (tb_ext[4])
  for (int f = 0; f < s_factors; ++f) {
    int64_t left = int64_t(1) << f;
    int tin = zcur, ti = 0;
    while (left > 0) {
      const int steps = (int)std::min<int64_t>(kmax, left);
      left -= steps;
      const int mode = left > 0 ? kInner : (f == s_factors - 1 ? kFinal : kFactorEnd);
      const int out = mode == kInner ? ti : (mode == kFinal ? 5 : 2 + zi);
      NNB_TRY(exchange(tin));
      for (Slab* sl : slabs) {
        // output tiles cover the slab's own rows only (from its first own row); the halo rows
        // are inputs, refreshed by the next exchange
        const int W = sl->tbW, H = (int)(sl->tb_len() / W);
        const int hlo = (int)(sl->tb_lo / W), hhi = (int)(sl->tb_hi / W), R = (int)(sl->rows / W);
        if (!bs) {
          NNB_TRY(stencil_pass(sl->tb_ext[tin], sl->tb_code, sl->tb_ext[zcur], sl->tb_ext[out], table, npat, W, H,
                               steps, mode, theta, sl->flags + f, kmax, s, 0, -1, hlo, R));
          continue;
        }
        // own tile row t reads region rows [hlo + t·ty − kmax, hlo + t·ty + ty + kmax)
        const int tiles = (R + ty - 1) / ty;
        int t0 = 0, t1 = tiles;
        if (hlo > 0) t0 = (kmax + ty - 1) / ty;
        if (hhi > 0) {
          const int num = R - ty - kmax;  // the last interior tile row t has t·ty <= num
          t1 = num < 0 ? 0 : std::min(tiles, num / ty + 1);
        }
        if (t0 > t1) t0 = t1 = 0;
        NNB_TRY(stencil_pass(sl->tb_ext[tin], sl->tb_code, sl->tb_ext[zcur], sl->tb_ext[out], table, npat, W, H,
                             steps, mode, theta, sl->flags + f, kmax, s, t0, t1, hlo, R));
        NNB_TRY(stencil_pass(sl->tb_ext[tin], sl->tb_code, sl->tb_ext[zcur], sl->tb_ext[out], table, npat, W, H,
                             steps, mode, theta, sl->flags + f, kmax, bs, 0, t0, hlo, R));
        NNB_TRY(stencil_pass(sl->tb_ext[tin], sl->tb_code, sl->tb_ext[zcur], sl->tb_ext[out], table, npat, W, H,
                             steps, mode, theta, sl->flags + f, kmax, bs, t1, -1, hlo, R));
      }
      NNB_TRY(join());
      if (mode == kInner) {
        tin = ti;
        ti ^= 1;
      } else if (mode == kFactorEnd) {
        zcur = 2 + zi;
        zi ^= 1;
      }
    }
  }
  for (size_t g = 0; g < slabs.size(); ++g)
    NNB_CUDA(cudaMemcpyAsync(x_own[g], slabs[g]->tb_ext[5] + slabs[g]->tb_lo, sizeof(double) * slabs[g]->rows,
                             cudaMemcpyDeviceToDevice, s));
  return 0;
}

// The slab's rows in 1-byte codes when the operator allows (sparse.cu build_pair_dict /
// build_row_dict): the gathers stay r + diag_off + delta into the extended vector.
int setup_slab_dict(Slab& sl, const int64_t* rp_dev, const int32_t* col_dev, const double* val_dev,
                    cudaStream_t s) {
  static const bool dict_on = !(debug_env("NNB_SPARSE_DICT") && std::strcmp(debug_env("NNB_SPARSE_DICT"), "0") == 0);
  static const bool rowdict_on =
      !(debug_env("NNB_SPARSE_ROWDICT") && std::strcmp(debug_env("NNB_SPARSE_ROWDICT"), "0") == 0);
  if (!dict_on || sl.rows == 0) return 0;
  NNB_TRY(sl.dict_mem.alloc((sizeof(int32_t) + sizeof(double)) * kPairDictMax, s));
  double* dv = sl.dict_mem.as<double>();
  int32_t* dd = reinterpret_cast<int32_t*>(dv + kPairDictMax);
  bool ok = false;
  int size = 0, width = 0, lo = 0, hi = 0;
  int64_t plane = 0;
  if (rowdict_on && sl.rows < INT32_MAX / 4) {  // stencil slabs: row codes straight from the CSR
    NNB_TRY(sl.rowdict_mem.alloc(sizeof(double2) * kRowDictMax * kEllMaxWidth + kRowDictMax + sl.rows, s));
    double2* pat = sl.rowdict_mem.as<double2>();
    uint8_t* plen = reinterpret_cast<uint8_t*>(pat + kRowDictMax * kEllMaxWidth);
    uint8_t* rcode = plen + kRowDictMax;
    int npat = 0;
    NNB_TRY(build_row_dict_direct(rp_dev, col_dev, val_dev, sl.rows, sl.row0, dd, dv, &size, &width, &lo, &hi, rcode,
                                  pat, plen, &npat, &ok, s));
    if (ok) {
      sl.dict_delta = dd;
      sl.dict_val = dv;
      sl.dict_size = size;
      sl.ell_width = width;
      sl.band_lo = lo;
      sl.band_hi = hi;
      sl.rcode = rcode;
      sl.rpat = pat;
      sl.rlen = plen;
      sl.npat = npat;
      return 0;
    }
  }
  NNB_TRY(build_pair_dict(rp_dev, col_dev, val_dev, sl.rows, sl.row0, sl.nnz, sl.code_mem, &width, &plane, &lo, &hi,
                          dd, dv, &size, &ok, s));
  if (!ok) return 0;
  sl.code = sl.code_mem.as<uint8_t>();
  sl.dict_delta = dd;
  sl.dict_val = dv;
  sl.dict_size = size;
  sl.ell_width = width;
  sl.ell_rows = plane;
  sl.band_lo = lo;
  sl.band_hi = hi;
  if (!width || !rowdict_on) return 0;
  if (!sl.rowdict_mem.p)
    NNB_TRY(sl.rowdict_mem.alloc(sizeof(double2) * kRowDictMax * kEllMaxWidth + kRowDictMax + sl.rows, s));
  double2* pat = sl.rowdict_mem.as<double2>();
  uint8_t* plen = reinterpret_cast<uint8_t*>(pat + kRowDictMax * kEllMaxWidth);
  uint8_t* rcode = plen + kRowDictMax;
  bool rok = false;
  int npat = 0;
  NNB_TRY(build_row_dict(sl.code, width, plane, sl.rows, dd, dv, rcode, pat, plen, &npat, &rok, s));
  if (rok) {
    sl.rcode = rcode;
    sl.rpat = pat;
    sl.rlen = plen;
    sl.npat = npat;
  }
  return 0;
}

// Builds the slab's device structures from its CSR rows (global columns).
int setup_slab(Slab& sl, const int64_t* rp_dev, const int32_t* col_dev, const double* val_dev, int64_t k,
               cudaStream_t s) {
  NNB_CUDA(cudaMemcpyAsync(&sl.nnz, rp_dev + sl.rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  int64_t base = 0;
  NNB_CUDA(cudaMemcpyAsync(&base, rp_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  trace_mark(s, "  slab: nnz");
  sl.nnz -= base;
  if (sl.nnz >= INT32_MAX) return fail(NNB_ERR_SHAPE, "sharded sparse: a slab exceeds 2^31 nonzeros");
  DevBuf st;
  NNB_TRY(st.alloc(4 * sizeof(int64_t), s));
  int64_t init[4] = {INT64_MAX, 0, 0, sl.rows};  // min col, max col, lo_end, hi_start
  NNB_CUDA(cudaMemcpyAsync(st.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (sl.rows)
    slab_stats_kernel<<<std::max<int64_t>(1, std::min<int64_t>(4736, (sl.rows + 255) / 256)), 256, 0, s>>>(
        rp_dev, col_dev + base, sl.rows, sl.row0, st.as<int64_t>());
  count_launch();
  int64_t h[4];
  NNB_CUDA(cudaMemcpyAsync(h, st.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  trace_mark(s, "  slab: stats");
  const bool any = h[0] != INT64_MAX;  // at least one nonzero in the slab
  sl.h_lo = (any && h[0] < sl.row0) ? sl.row0 - h[0] : 0;
  sl.h_hi = (any && h[1] >= sl.row0 + sl.rows) ? h[1] - (sl.row0 + sl.rows - 1) : 0;
  sl.lo_end = h[2];
  sl.hi_start = h[3];
  if (sl.lo_end > sl.hi_start) sl.lo_end = sl.hi_start = sl.rows;  // no clean interior: all boundary (after halo)
  const size_t ext = (size_t)sl.ext_len() * k;
  const size_t bytes = sizeof(int32_t) * (sl.rows + 1 + sl.nnz) + sizeof(int16_t) * sl.nnz +
                       sizeof(double) * 5 * ext + sizeof(int) * 64 + 256;
  NNB_TRY(sl.mem.alloc(bytes, s));
  char* p = sl.mem.as<char>();
  double* d = reinterpret_cast<double*>(p);
  for (int i = 0; i < 5; ++i) sl.ext[i] = d + i * ext;
  sl.rp = reinterpret_cast<int32_t*>(d + 5 * ext);
  sl.col = sl.rp + sl.rows + 1;
  int16_t* c16 = reinterpret_cast<int16_t*>(sl.col + sl.nnz + 1);
  sl.flags = reinterpret_cast<int*>(c16 + sl.nnz + 8);
  sl.flags = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(sl.flags) + 15) & ~uintptr_t(15));
  NNB_CUDA(cudaMemsetAsync(sl.flags, 0, sizeof(int) * 64, s));
  NNB_CUDA(cudaMemsetAsync(d, 0, sizeof(double) * 5 * ext, s));
  bool fits = false;
  trace_mark(s, "  slab: buffers");
  sl.val = val_dev + base;
  if (k == 1) NNB_TRY(setup_slab_dict(sl, rp_dev, col_dev, val_dev, s));
  trace_mark(s, "  slab: dictionary");
  // int32 offsets and int16 / remapped columns only for the formats that read them: a slab
  // in row codes (spmv_apply's row-dictionary branch, 32-bit index math) never does
  if (!(sl.rcode && sl.rows + sl.h_lo < INT32_MAX / 2)) {
    NNB_TRY(compact_csr(rp_dev, col_dev, sl.rows, sl.row0, sl.rp, c16, &fits, s));
    if (fits) {
      sl.col16 = c16;
    } else if (sl.nnz) {
      remap_cols_kernel<<<std::max<int64_t>(1, std::min<int64_t>(4736, (sl.nnz + 255) / 256)), 256, 0, s>>>(
          col_dev + base, sl.nnz, sl.h_lo - sl.row0, sl.col);
      count_launch();
    }
    trace_mark(s, "  slab: compact");
  }
  set_sparse_bytes_per_nnz(sl.code || sl.rcode ? 1 : (sl.col16 ? 10 : 12));
  set_sparse_format(sl.rcode ? "row-dictionary"
                    : sl.ell_width ? "pair-dictionary-ell"
                    : sl.code ? "pair-dictionary-csr"
                    : sl.col16 ? "csr-int16-delta" : "csr-int32");
  set_sparse_matrix_bytes(sl.rcode ? sl.rows
                          : sl.ell_width ? (int64_t)sl.ell_width * sl.rows
                                         : sl.nnz * (sl.code ? 1 : (sl.col16 ? 10 : 12)) + (sl.rows + 1) * 4);
  NNB_CUDA(cudaGetLastError());
  return 0;
}

// The shared schedule; `exchange(e, g)` fills rank g's halo of extended buffer e.
template <class Exchange, class WaitHalo>
int run_slabs(std::vector<Slab*>& slabs, int64_t k, int s_factors, double theta, std::vector<double*>& x_own,
              Exchange exchange, WaitHalo wait_halo, cudaStream_t s) {
  int64_t reps = 1;
  int zcur = 4, zi = 0;  // Z starts as B (ext index 4)
  for (int f = 0; f < s_factors; ++f) {
    int tin = zcur, ti = 0;
    for (int64_t r = 0; r < reps; ++r) {
      int mode, out;
      if (r < reps - 1) {
        mode = kInner;
        out = ti;
      } else if (f == s_factors - 1) {
        mode = kFinal;
        out = -1;
      } else {
        mode = kFactorEnd;
        out = 2 + zi;
      }
      NNB_TRY(exchange(tin));
      for (size_t g = 0; g < slabs.size(); ++g) {
        Slab& sl = *slabs[g];
        SpmvOp<int32_t> op{sl.rp, sl.col, sl.col16, sl.h_lo, sl.val, k, sl.ext[tin], sl.ext[tin] + sl.h_lo * k,
                           out < 0 ? x_own[g] : sl.ext[out] + sl.h_lo * k, sl.ext[zcur] + sl.h_lo * k, theta,
                           sl.flags + f, sl.code, sl.dict_delta, sl.dict_val, sl.dict_size, sl.ell_width,
                           sl.ell_rows, sl.band_lo, sl.band_hi, sl.rcode, sl.rpat, sl.rlen, sl.npat};
        spmv_apply(op, mode, sl.lo_end, sl.hi_start, s);  // interior, while the halo is in flight
        NNB_TRY(wait_halo(g));
        spmv_apply(op, mode, 0, sl.lo_end, s);            // boundary rows
        spmv_apply(op, mode, sl.hi_start, sl.rows, s);
      }
      if (mode == kInner) {
        tin = ti;
        ti ^= 1;
      } else if (mode == kFactorEnd) {
        zcur = 2 + zi;
        zi ^= 1;
      }
    }
    reps <<= 1;
  }
  return 0;
}

int collect_flags(std::vector<Slab*>& slabs, int s_factors, int* fail_factor, cudaStream_t s,
                  const std::vector<int>* extra = nullptr) {
  std::vector<int> any(64, 0);
  for (Slab* sl : slabs) {
    int h[64];
    NNB_CUDA(cudaMemcpyAsync(h, sl->flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < 64; ++i) any[i] |= h[i];
  }
  if (extra)
    for (int i = 0; i < 64; ++i) any[i] |= (*extra)[i];
  for (int f = 0; f < s_factors && f < 64; ++f)
    if (any[f]) {
      if (fail_factor) *fail_factor = f;
      return fail(NNB_ERR_DIVERGENCE, "solve_sparse_factorized: non-finite block at factor " + std::to_string(f));
    }
  return 0;
}

int check_order(int64_t gamma, int* s_factors) {
  if (gamma < 1 || ((gamma + 1) & gamma) != 0)
    return fail(NNB_ERR_PLAN, "solve_sparse_factorized: order + 1 must be a power of two");
  if (gamma > (int64_t(1) << 30)) return fail(NNB_ERR_BUDGET, "solve_sparse_factorized: order too large to apply");
  *s_factors = 0;
  for (int64_t g = gamma + 1; g > 1; g >>= 1) ++*s_factors;
  return 0;
}

}  // namespace sparse_detail
}  // namespace nnb

using namespace nnb;
using namespace nnb::sparse_detail;

extern "C" {

// A prepared slab: partition, staged CSR, remapped columns, halo sizes and
// the extended vectors — built once, reused by every solve on the operator.
struct nnb_sparse_plan {
  nnb_comm* comm = nullptr;
  int64_t n = 0, k = 0;
  Slab sl;
  DevBuf csr;
  DevBuf tb_table;  // the union pattern table when the slabs run temporal-blocked passes
  int tb_npat = 0;
  cudaEvent_t ready = nullptr, landed = nullptr;
  ~nnb_sparse_plan() {
    if (ready) cudaEventDestroy(ready);
    if (landed) cudaEventDestroy(landed);
  }
};

int nnb_sparse_plan_create(nnb_comm_t comm, const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                           int64_t k, nnb_sparse_plan_t* plan_out, void* stream) {
  NNB_TRY(require_device());
  if (!comm) return fail(NNB_ERR_DOMAIN, "sharded sparse: comm is NULL");
  if (k < 1) return fail(NNB_ERR_SHAPE, "sharded sparse: k must be >= 1");
  cudaStream_t s = resolve(stream);
  auto plan = std::make_unique<nnb_sparse_plan>();
  plan->comm = comm;
  plan->n = n;
  plan->k = k;
  const int G = comm->world, me = comm->rank;
  Slab& sl = plan->sl;
  nnb_partition_rows(n, G, me, &sl.row0, &sl.rows);
  // stage the slab's CSR (host or device) on this device
  const int64_t* rp_d = row_ptr;
  const int32_t* col_d = col;
  const double* val_d = val;
  if (!is_device_ptr(row_ptr) || !is_device_ptr(col) || !is_device_ptr(val)) {
    const int64_t base = row_ptr[0], nnz = row_ptr[sl.rows] - base;
    NNB_TRY(plan->csr.alloc(sizeof(int64_t) * (sl.rows + 1) + sizeof(double) * nnz + sizeof(int32_t) * nnz + 64, s));
    char* b = plan->csr.as<char>();
    NNB_CUDA(cudaMemcpyAsync(b, row_ptr, sizeof(int64_t) * (sl.rows + 1), cudaMemcpyDefault, s));
    NNB_CUDA(cudaMemcpyAsync(b + sizeof(int64_t) * (sl.rows + 1), val + base, sizeof(double) * nnz, cudaMemcpyDefault, s));
    NNB_CUDA(cudaMemcpyAsync(b + sizeof(int64_t) * (sl.rows + 1) + sizeof(double) * nnz, col + base,
                             sizeof(int32_t) * nnz, cudaMemcpyDefault, s));
    rp_d = reinterpret_cast<const int64_t*>(b);
    val_d = reinterpret_cast<const double*>(b + sizeof(int64_t) * (sl.rows + 1)) - base;
    col_d = reinterpret_cast<const int32_t*>(b + sizeof(int64_t) * (sl.rows + 1) + sizeof(double) * nnz) - base;
  }
  if (trace_on()) {
    trace_reset();
    trace_mark(s, "plan start");
  }
  NNB_TRY(setup_slab(sl, rp_d, col_d, val_d, k, s));
  trace_mark(s, "slab setup");
  // halo sizes of every rank (each rank sends its neighbours what they need)
  DevBuf hx;
  NNB_TRY(hx.alloc(sizeof(int64_t) * 2 * (G + 1), s));
  int64_t mine[2] = {sl.h_lo, sl.h_hi};
  NNB_CUDA(cudaMemcpyAsync(hx.as<int64_t>() + 2 * G, mine, sizeof(mine), cudaMemcpyHostToDevice, s));
  NNB_NCCL2(nccl_allgather(hx.as<int64_t>() + 2 * G, hx.as<int64_t>(), 2 * sizeof(int64_t) / sizeof(double), comm, s));
  std::vector<int64_t> halos(2 * G);
  NNB_CUDA(cudaMemcpyAsync(halos.data(), hx.p, sizeof(int64_t) * 2 * G, cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> r0(G), rs(G);
  for (int g = 0; g < G; ++g) nnb_partition_rows(n, G, g, &r0[g], &rs[g]);
  for (int g = 0; g < G; ++g)
    if ((g > 0 && halos[2 * g] > rs[g - 1]) || (g < G - 1 && halos[2 * g + 1] > rs[g + 1]))
      return fail(NNB_ERR_DOMAIN, "sharded sparse: operator bandwidth exceeds a neighbour slab (halo wider than one rank)");
  sl.send_prev = me > 0 ? halos[2 * (me - 1) + 1] : 0;
  sl.send_next = me < G - 1 ? halos[2 * (me + 1)] : 0;
  NNB_CUDA(cudaEventCreateWithFlags(&plan->ready, cudaEventDisableTiming));
  NNB_CUDA(cudaEventCreateWithFlags(&plan->landed, cudaEventDisableTiming));
  if (k == 1) {  // temporal blocking across the slabs: every rank's record, one decision
    static_assert(sizeof(TbRecord) % sizeof(double) == 0, "record in doubles");
    const size_t rd = sizeof(TbRecord) / sizeof(double);
    DevBuf rb;
    NNB_TRY(rb.alloc(sizeof(TbRecord) * (G + 1), s));
    TbRecord mine_rec;
    trace_mark(s, "halo sizes");
    NNB_TRY(tb_record(sl, n, &mine_rec, s));
    trace_mark(s, "tb record");
    NNB_CUDA(cudaMemcpyAsync(rb.as<TbRecord>() + G, &mine_rec, sizeof(TbRecord), cudaMemcpyHostToDevice, s));
    NNB_NCCL2(nccl_allgather(rb.as<TbRecord>() + G, rb.as<TbRecord>(), rd, comm, s));
    std::vector<TbRecord> recs(G);
    NNB_CUDA(cudaMemcpyAsync(recs.data(), rb.p, sizeof(TbRecord) * G, cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaStreamSynchronize(s));
    std::vector<StencilPattern> table;
    std::vector<std::vector<uint8_t>> map;
    if (tb_decide(recs, rs, table, map)) {
      const int W = (int)recs[0].w;
      NNB_TRY(tb_setup_slab(sl, n, W, map[me], s));
      NNB_TRY(plan->tb_table.alloc(sizeof(StencilPattern) * table.size(), s));
      NNB_CUDA(cudaMemcpyAsync(plan->tb_table.p, table.data(), sizeof(StencilPattern) * table.size(),
                               cudaMemcpyHostToDevice, s));
      plan->tb_npat = (int)table.size();
      // the neighbours' edge codes into the halo rows (tb_rows()·W bytes each way)
      const size_t hw = (size_t)tb_rows() * W / sizeof(double);
      NNB_NCCL2(nccl_group(true));
      if (me > 0) {
        NNB_NCCL2(nccl_send(sl.tb_code + sl.tb_lo, hw, me - 1, comm, s));
        NNB_NCCL2(nccl_recv(sl.tb_code, hw, me - 1, comm, s));
      }
      if (me < G - 1) {
        NNB_NCCL2(nccl_send(sl.tb_code + sl.tb_lo + sl.rows - (int64_t)tb_rows() * W, hw, me + 1, comm, s));
        NNB_NCCL2(nccl_recv(sl.tb_code + sl.tb_lo + sl.rows, hw, me + 1, comm, s));
      }
      NNB_NCCL2(nccl_group(false));
      NNB_CUDA(cudaStreamSynchronize(s));
    }
    trace_mark(s, "tb setup");
  }
  trace_dump();
  *plan_out = plan.release();
  return 0;
}

double nnb_sparse_last_solve_ms(void) { return g_last_solve_ms; }

int nnb_sparse_plan_destroy(nnb_sparse_plan_t plan) {
  delete plan;
  return 0;
}

int nnb_sparse_plan_solve(nnb_sparse_plan_t plan, const double* B_rows, int64_t gamma, double theta, double* X_rows,
                          int64_t* spmv_count_out, int32_t* fail_factor_out, void* stream) {
  NNB_TRY(require_device());
  if (!plan) return fail(NNB_ERR_DOMAIN, "sharded sparse: plan is NULL");
  int s_factors = 0;
  NNB_TRY(check_order(gamma, &s_factors));
  cudaStream_t s = resolve(stream);
  nnb_comm* comm = plan->comm;
  const int G = comm->world, me = comm->rank;
  const int64_t k = plan->k;
  Slab& sl = plan->sl;
  NNB_CUDA(cudaMemsetAsync(sl.flags, 0, sizeof(int) * 64, s));
  // Z = B in the extended layout
  if (sl.tb)
    NNB_CUDA(cudaMemcpyAsync(sl.tb_ext[4] + sl.tb_lo, B_rows, sizeof(double) * sl.rows, cudaMemcpyDefault, s));
  else
    NNB_CUDA(cudaMemcpyAsync(sl.ext[4] + sl.h_lo * k, B_rows, sizeof(double) * sl.rows * k, cudaMemcpyDefault, s));
  Out x;
  NNB_TRY(x.prepare(X_rows, (size_t)(sl.rows * k), s));
  std::vector<Slab*> slabs{&sl};
  std::vector<double*> xo{x.d};
  auto exchange_tb = [&](int e) -> int {  // tb_rows()·W cells each way, once per pass
    if (G == 1) return 0;
    double* ext = sl.tb_ext[e];
    const size_t hw = (size_t)tb_rows() * sl.tbW;
    NNB_CUDA(cudaEventRecord(plan->ready, s));
    NNB_CUDA(cudaStreamWaitEvent(comm->cs, plan->ready, 0));
    NNB_NCCL2(nccl_group(true));
    if (me > 0) {
      NNB_NCCL2(nccl_send(ext + sl.tb_lo, hw, me - 1, comm, comm->cs));
      NNB_NCCL2(nccl_recv(ext, hw, me - 1, comm, comm->cs));
    }
    if (me < G - 1) {
      NNB_NCCL2(nccl_send(ext + sl.tb_lo + sl.rows - hw, hw, me + 1, comm, comm->cs));
      NNB_NCCL2(nccl_recv(ext + sl.tb_lo + sl.rows, hw, me + 1, comm, comm->cs));
    }
    NNB_NCCL2(nccl_group(false));
    return 0;
  };
  auto join_tb = [&]() -> int {  // s waits for the edge tile rows launched behind the exchange
    if (G > 1) {
      NNB_CUDA(cudaEventRecord(plan->landed, comm->cs));
      NNB_CUDA(cudaStreamWaitEvent(s, plan->landed, 0));
    }
    return 0;
  };
  auto exchange = [&](int e) -> int {
    if (G == 1) return 0;
    double* ext = sl.ext[e];
    NNB_CUDA(cudaEventRecord(plan->ready, s));
    NNB_CUDA(cudaStreamWaitEvent(comm->cs, plan->ready, 0));
    NNB_NCCL2(nccl_group(true));
    if (me > 0) {
      if (sl.send_prev) NNB_NCCL2(nccl_send(ext + sl.h_lo * k, sl.send_prev * k, me - 1, comm, comm->cs));
      if (sl.h_lo) NNB_NCCL2(nccl_recv(ext, sl.h_lo * k, me - 1, comm, comm->cs));
    }
    if (me < G - 1) {
      if (sl.send_next)
        NNB_NCCL2(nccl_send(ext + (sl.h_lo + sl.rows - sl.send_next) * k, sl.send_next * k, me + 1, comm, comm->cs));
      if (sl.h_hi) NNB_NCCL2(nccl_recv(ext + (sl.h_lo + sl.rows) * k, sl.h_hi * k, me + 1, comm, comm->cs));
    }
    NNB_NCCL2(nccl_group(false));
    NNB_CUDA(cudaEventRecord(plan->landed, comm->cs));
    return 0;
  };
  auto wait = [&](size_t) -> int {
    if (G > 1) NNB_CUDA(cudaStreamWaitEvent(s, plan->landed, 0));
    return 0;
  };
  SolveTimer timer(s);
  int st = sl.tb ? run_slabs_tb(slabs, plan->tb_table.as<StencilPattern>(), plan->tb_npat, s_factors, theta, xo,
                                exchange_tb, join_tb, s, G > 1 ? comm->cs : nullptr)
                 : run_slabs(slabs, k, s_factors, theta, xo, exchange, wait, s);
  if (st == 0) timer.stop();
  if (sl.tb) {
    set_sparse_format("row-dictionary-stencil-tb");
    set_sparse_bytes_per_nnz(1);
  }
  // divergence flags of every rank (so every rank reports the same factor)
  std::vector<int> all(64, 0);
  if (st == 0 && G > 1) {
    DevBuf fb;
    NNB_TRY(fb.alloc(sizeof(int) * 64 * (G + 1), s));
    NNB_CUDA(cudaMemcpyAsync(fb.as<int>() + 64 * G, sl.flags, sizeof(int) * 64, cudaMemcpyDeviceToDevice, s));
    NNB_NCCL2(nccl_allgather(fb.as<int>() + 64 * G, fb.as<int>(), 64 * sizeof(int) / sizeof(double), comm, s));
    std::vector<int> h(64 * G);
    NNB_CUDA(cudaMemcpyAsync(h.data(), fb.p, sizeof(int) * 64 * G, cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaStreamSynchronize(s));
    for (int g = 0; g < G; ++g)
      for (int i = 0; i < 64; ++i) all[i] |= h[64 * g + i];
  }
  if (st) return st;
  int ff = -1;
  st = collect_flags(slabs, s_factors, &ff, s, &all);
  if (fail_factor_out) *fail_factor_out = ff;
  if (st) return st;
  if (spmv_count_out) *spmv_count_out = gamma * k;
  return x.finish(s);
}

int nnb_sparse_factorized_sharded_d(nnb_comm_t comm, const int64_t* row_ptr, const int32_t* col, const double* val,
                                    int64_t n, const double* B_rows, int64_t k, int64_t gamma, double theta,
                                    double* X_rows, int64_t* spmv_count_out, int32_t* fail_factor_out,
                                    void* stream) {
  int s_factors = 0;
  NNB_TRY(check_order(gamma, &s_factors));
  nnb_sparse_plan_t plan = nullptr;
  NNB_TRY(nnb_sparse_plan_create(comm, row_ptr, col, val, n, k, &plan, stream));
  const int st = nnb_sparse_plan_solve(plan, B_rows, gamma, theta, X_rows, spmv_count_out, fail_factor_out, stream);
  nnb_sparse_plan_destroy(plan);
  return st;
}

int nnb_sparse_factorized_sharded_emulated_d(const int64_t* row_ptr, const int32_t* col, const double* val,
                                             int64_t n, int64_t nnz, const double* B, int64_t k, int64_t gamma,
                                             double theta, int32_t world, double* X_out, int64_t* spmv_count_out,
                                             int32_t* fail_factor_out, void* stream) {
  NNB_TRY(require_device());
  if (world < 1) return fail(NNB_ERR_DOMAIN, "sharded sparse: world must be >= 1");
  int s_factors = 0;
  NNB_TRY(check_order(gamma, &s_factors));
  cudaStream_t s = resolve(stream);
  DevBuf csr;
  const int64_t* rp_d = row_ptr;
  const int32_t* col_d = col;
  const double* val_d = val;
  if (!is_device_ptr(row_ptr) || !is_device_ptr(col) || !is_device_ptr(val)) {
    NNB_TRY(csr.alloc(sizeof(int64_t) * (n + 1) + sizeof(double) * nnz + sizeof(int32_t) * nnz + 64, s));
    char* b = csr.as<char>();
    NNB_CUDA(cudaMemcpyAsync(b, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDefault, s));
    NNB_CUDA(cudaMemcpyAsync(b + sizeof(int64_t) * (n + 1), val, sizeof(double) * nnz, cudaMemcpyDefault, s));
    NNB_CUDA(cudaMemcpyAsync(b + sizeof(int64_t) * (n + 1) + sizeof(double) * nnz, col, sizeof(int32_t) * nnz,
                             cudaMemcpyDefault, s));
    rp_d = reinterpret_cast<const int64_t*>(b);
    val_d = reinterpret_cast<const double*>(b + sizeof(int64_t) * (n + 1));
    col_d = reinterpret_cast<const int32_t*>(b + sizeof(int64_t) * (n + 1) + sizeof(double) * nnz);
  }
  std::vector<Slab> store(world);
  std::vector<Slab*> slabs;
  for (int g = 0; g < world; ++g) {
    Slab& sl = store[g];
    nnb_partition_rows(n, world, g, &sl.row0, &sl.rows);
    NNB_TRY(setup_slab(sl, rp_d + sl.row0, col_d, val_d, k, s));
    slabs.push_back(&sl);
  }
  for (int g = 0; g < world; ++g) {
    Slab& sl = store[g];
    if ((g > 0 && sl.h_lo > store[g - 1].rows) || (g < world - 1 && sl.h_hi > store[g + 1].rows))
      return fail(NNB_ERR_DOMAIN, "sharded sparse: operator bandwidth exceeds a neighbour slab (halo wider than one rank)");
  }
  // temporal blocking across the slabs: the same records and decision as the NCCL plan
  bool tb = false;
  DevBuf tb_table;
  int tb_npat = 0;
  if (k == 1) {
    std::vector<TbRecord> recs(world);
    std::vector<int64_t> rows(world);
    for (int g = 0; g < world; ++g) {
      NNB_TRY(tb_record(store[g], n, &recs[g], s));
      rows[g] = store[g].rows;
    }
    std::vector<StencilPattern> table;
    std::vector<std::vector<uint8_t>> map;
    tb = tb_decide(recs, rows, table, map);
    if (tb) {
      const int W = (int)recs[0].w;
      for (int g = 0; g < world; ++g) NNB_TRY(tb_setup_slab(store[g], n, W, map[g], s));
      NNB_TRY(tb_table.alloc(sizeof(StencilPattern) * table.size(), s));
      NNB_CUDA(cudaMemcpyAsync(tb_table.p, table.data(), sizeof(StencilPattern) * table.size(),
                               cudaMemcpyHostToDevice, s));
      tb_npat = (int)table.size();
      const int64_t hw = (int64_t)tb_rows() * W;
      for (int g = 0; g < world; ++g) {  // the neighbours' edge codes into the halo rows
        Slab& sl = store[g];
        if (g > 0)
          NNB_CUDA(cudaMemcpyAsync(sl.tb_code, store[g - 1].tb_code + store[g - 1].tb_lo + store[g - 1].rows - hw, hw,
                                   cudaMemcpyDeviceToDevice, s));
        if (g < world - 1)
          NNB_CUDA(cudaMemcpyAsync(sl.tb_code + sl.tb_lo + sl.rows, store[g + 1].tb_code + store[g + 1].tb_lo, hw,
                                   cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  for (int g = 0; g < world; ++g) {
    Slab& sl = store[g];
    if (tb)
      NNB_CUDA(cudaMemcpyAsync(sl.tb_ext[4] + sl.tb_lo, B + sl.row0, sizeof(double) * sl.rows, cudaMemcpyDefault, s));
    else
      NNB_CUDA(cudaMemcpyAsync(sl.ext[4] + sl.h_lo * k, B + sl.row0 * k, sizeof(double) * sl.rows * k,
                               cudaMemcpyDefault, s));
  }
  Out x;
  NNB_TRY(x.prepare(X_out, (size_t)(n * k), s));
  std::vector<double*> xo;
  for (int g = 0; g < world; ++g) xo.push_back(x.d + store[g].row0 * k);
  auto exchange = [&](int e) -> int {  // device copies from the neighbours' owned rows
    for (int g = 0; g < world; ++g) {
      Slab& sl = store[g];
      if (g > 0 && sl.h_lo) {
        const Slab& pv = store[g - 1];
        NNB_CUDA(cudaMemcpyAsync(sl.ext[e], pv.ext[e] + (pv.h_lo + pv.rows - sl.h_lo) * k,
                                 sizeof(double) * sl.h_lo * k, cudaMemcpyDeviceToDevice, s));
      }
      if (g < world - 1 && sl.h_hi) {
        const Slab& nx = store[g + 1];
        NNB_CUDA(cudaMemcpyAsync(sl.ext[e] + (sl.h_lo + sl.rows) * k, nx.ext[e] + nx.h_lo * k,
                                 sizeof(double) * sl.h_hi * k, cudaMemcpyDeviceToDevice, s));
      }
    }
    return 0;
  };
  auto wait = [](size_t) -> int { return 0; };
  auto exchange_tb = [&](int e) -> int {  // device copies of the neighbours' edge rows
    for (int g = 0; g < world; ++g) {
      Slab& sl = store[g];
      const int64_t hw = (int64_t)tb_rows() * sl.tbW;
      if (g > 0) {
        const Slab& pv = store[g - 1];
        NNB_CUDA(cudaMemcpyAsync(sl.tb_ext[e], pv.tb_ext[e] + pv.tb_lo + pv.rows - hw, sizeof(double) * hw,
                                 cudaMemcpyDeviceToDevice, s));
      }
      if (g < world - 1) {
        const Slab& nx = store[g + 1];
        NNB_CUDA(cudaMemcpyAsync(sl.tb_ext[e] + sl.tb_lo + sl.rows, nx.tb_ext[e] + nx.tb_lo, sizeof(double) * hw,
                                 cudaMemcpyDeviceToDevice, s));
      }
    }
    return 0;
  };
  auto join_tb = []() -> int { return 0; };
  SolveTimer timer(s);
  int st = tb ? run_slabs_tb(slabs, tb_table.as<StencilPattern>(), tb_npat, s_factors, theta, xo, exchange_tb, join_tb,
                             s, nullptr)
              : run_slabs(slabs, k, s_factors, theta, xo, exchange, wait, s);
  if (st == 0) timer.stop();
  if (tb) {
    set_sparse_format("row-dictionary-stencil-tb");
    set_sparse_bytes_per_nnz(1);
  }
  if (st) return st;
  int ff = -1;
  st = collect_flags(slabs, s_factors, &ff, s);
  if (fail_factor_out) *fail_factor_out = ff;
  if (st) return st;
  if (spmv_count_out) *spmv_count_out = gamma * k;
  return x.finish(s);
}

}  // extern "C"
