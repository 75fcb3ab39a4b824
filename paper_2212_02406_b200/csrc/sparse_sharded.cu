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

#define NNB_NCCL2(x)                                                                             \
  do {                                                                                           \
    ncclResult_t _r = (x);                                                                       \
    if (_r != ncclSuccess) return fail(NNB_ERR_NCCL, std::string("NCCL error: ") + nccl_error(_r)); \
  } while (0)

// Per-slab statistics: min/max column, last row referencing below the slab,
// first row referencing above it.
__global__ void slab_stats_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t rows,
                                  int64_t row0, int64_t* __restrict__ stats /* [min_col, max_col, lo_end, hi_start] */) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t mn = INT64_MAX, mx = -1;
    for (int64_t e = rp[r] - rp[0]; e < rp[r + 1] - rp[0]; ++e) {
      const int64_t c = col[e];
      mn = c < mn ? c : mn;
      mx = c > mx ? c : mx;
    }
    if (mx < 0) continue;  // empty row
    atomicMin(reinterpret_cast<unsigned long long*>(stats + 0), static_cast<unsigned long long>(mn));
    atomicMax(reinterpret_cast<unsigned long long*>(stats + 1), static_cast<unsigned long long>(mx));
    if (mn < row0) atomicMax(reinterpret_cast<unsigned long long*>(stats + 2), static_cast<unsigned long long>(r + 1));
    if (mx >= row0 + rows) atomicMin(reinterpret_cast<unsigned long long*>(stats + 3), static_cast<unsigned long long>(r));
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
};

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
  NNB_TRY(compact_csr(rp_dev, col_dev, sl.rows, sl.row0, sl.rp, c16, &fits, s));
  if (fits) {
    sl.col16 = c16;
  } else if (sl.nnz) {
    remap_cols_kernel<<<std::max<int64_t>(1, std::min<int64_t>(4736, (sl.nnz + 255) / 256)), 256, 0, s>>>(
        col_dev + base, sl.nnz, sl.h_lo - sl.row0, sl.col);
    count_launch();
  }
  sl.val = val_dev + base;
  if (k == 1) NNB_TRY(setup_slab_dict(sl, rp_dev, col_dev, val_dev, s));
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
  NNB_TRY(setup_slab(sl, rp_d, col_d, val_d, k, s));
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
  *plan_out = plan.release();
  return 0;
}

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
  NNB_CUDA(cudaMemcpyAsync(sl.ext[4] + sl.h_lo * k, B_rows, sizeof(double) * sl.rows * k, cudaMemcpyDefault, s));
  Out x;
  NNB_TRY(x.prepare(X_rows, (size_t)(sl.rows * k), s));
  std::vector<Slab*> slabs{&sl};
  std::vector<double*> xo{x.d};
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
  int st = run_slabs(slabs, k, s_factors, theta, xo, exchange, wait, s);
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
  int st = run_slabs(slabs, k, s_factors, theta, xo, exchange, wait, s);
  if (st) return st;
  int ff = -1;
  st = collect_flags(slabs, s_factors, &ff, s);
  if (fail_factor_out) *fail_factor_out = ff;
  if (st) return st;
  if (spmv_count_out) *spmv_count_out = gamma * k;
  return x.finish(s);
}

}  // extern "C"
