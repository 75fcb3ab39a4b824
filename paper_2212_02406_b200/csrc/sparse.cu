// Matrix-free factorized Neumann solve on a CSR operator (BASELINE config 4:
// 5-point Laplacian + I on a 4096² grid, θ = 0.2, γ = 63).
//
// Reference: /root/reference/proj/src/factorized.cpp:101-140 —
//   Z = B;  for f < s:  t = Z;  2^f × { y = W t (spmv_block); t = t − θ y };  Z = Z + t
//   x = θ Z
// which streams t, y and Z through three separate N-vector passes per
// application plus an allocation each.  Here one kernel per application does
//   t_out = t_in − θ·W·t_in                         (inner applications)
//   Z_new = Z + (t_in − θ·W·t_in)                   (last application of a factor)
//   X     = θ·(Z + (t_in − θ·W·t_in))               (last application overall)
// so y never exists and the factor update and the final scale ride along.
//
// Every operation is explicitly rounded (no FMA contraction) and ordered as
// the reference's std::complex<double> arithmetic evaluates it for real W:
// spmv sum += v·x from 0 in ascending nonzero order, t = z − θ·y, Z + t, Z·θ.
// The GPU result is therefore BIT-IDENTICAL to the reference's, for any row
// partition (the multi-GPU path, sparse_sharded.cu, relies on this).
//
// Kernel: one thread per row, persistent grid of exactly the resident blocks.
// A row-group variant with coalesced shared staging (20.1 ms), an 8-way
// unrolled per-row variant (19.2 ms) and sliced ELL (17.0 ms; less
// memory-level parallelism than CSR order) all lost to this loop.
// One pass per solve (compact_csr) narrows the row offsets to int32 and, for
// banded operators, the columns to int16 deltas from the row.
// HBM-bound: 10 (int16) or 12 (int32 columns) B per nonzero + 4 B per row of
// CSR, 8 B in + 8 B out per row.  The register cap (32, for 64 resident warps
// per SM) buys the memory-level parallelism: 13.0 vs 13.7 ms per C5 solve at
// 48 warps; 1024-thread blocks shave another 1.6 % (12.8 ms).
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/nnb.h"
#include "engine.cuh"
#include "sparse.cuh"

namespace nnb {

namespace {
thread_local int g_sparse_bytes_per_nnz = 0;
thread_local int64_t g_sparse_matrix_bytes = 0;
}
void set_sparse_bytes_per_nnz(int b) { g_sparse_bytes_per_nnz = b; }
int sparse_bytes_per_nnz() { return g_sparse_bytes_per_nnz; }
void set_sparse_matrix_bytes(int64_t b) { g_sparse_matrix_bytes = b; }
namespace {
thread_local const char* g_sparse_format = "";
}
void set_sparse_format(const char* f) { g_sparse_format = f; }
const char* sparse_format() { return g_sparse_format; }
int64_t sparse_matrix_bytes() { return g_sparse_matrix_bytes; }

template <int MODE>
__device__ __forceinline__ double finish(double tin, double y, double theta, double zold, bool& bad) {
  const double t = __dsub_rn(tin, __dmul_rn(theta, y));  // fused_axpy_sub, factorized.cpp:21-30
  double o;
  if (MODE == kInner) {
    o = t;
  } else if (MODE == kFactorEnd) {
    o = __dadd_rn(zold, t);                              // add(z, t), factorized.cpp:136
  } else {
    o = __dmul_rn(__dadd_rn(zold, t), theta);            // scale(z, theta), factorized.cpp:139
  }
  bad |= !isfinite(y) || !isfinite(t) || !isfinite(o);
  return o;
}

// Rows [r_begin, r_end) of one application.  Gathers read t_ext through the
// (possibly halo-remapped) column indices; the diagonal term, z and the
// output are indexed by row.
// NNB_SPMV_THREADS per block; NNB_SPMV_MINB resident blocks per SM the register budget must allow.
#ifndef NNB_SPMV_THREADS
#define NNB_SPMV_THREADS 1024
#endif
#ifndef NNB_SPMV_MINB
#define NNB_SPMV_MINB (2048 / NNB_SPMV_THREADS)
#endif
template <typename Idx, typename C, int MODE, bool K1>
__global__ void __launch_bounds__(NNB_SPMV_THREADS, NNB_SPMV_MINB)
    spmv_rows_kernel(const Idx* __restrict__ rp, const C* __restrict__ col, const double* __restrict__ val,
                     int64_t r_begin, int64_t r_end, int64_t diag_off, int64_t k, const double* __restrict__ t_ext,
                     const double* __restrict__ t_own, double* __restrict__ out, const double* __restrict__ zold,
                     double theta, int* __restrict__ flag) {
  bool bad = false;
  if (K1) {  // one right-hand side, 32-bit offsets and indices
    for (int r = (int)r_begin + blockIdx.x * blockDim.x + threadIdx.x; r < (int)r_end; r += gridDim.x * blockDim.x) {
      const int e0 = (int)rp[r], e1 = (int)rp[r + 1];
      const double* tg = t_ext + (sizeof(C) == 2 ? r + (int)diag_off : 0);  // int16: column = row + delta
      double y = 0.0;
      for (int e = e0; e < e1; ++e) y = __dadd_rn(y, __dmul_rn(val[e], tg[col[e]]));
      out[r] = finish<MODE>(t_own[r], y, theta, MODE == kInner ? 0.0 : zold[r], bad);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
    return;
  }
  for (int64_t r = r_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r_end;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = rp[r], e1 = rp[r + 1];
    const int64_t g0 = sizeof(C) == 2 ? r + diag_off : 0;  // int16: column = row + delta
    for (int64_t c = 0; c < k; ++c) {
      double y = 0.0;
      for (int64_t e = e0; e < e1; ++e) y = __dadd_rn(y, __dmul_rn(val[e], t_ext[(g0 + col[e]) * k + c]));
      out[r * k + c] = finish<MODE>(t_own[r * k + c], y, theta, MODE == kInner ? 0.0 : zold[r * k + c], bad);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// The same application with the pair dictionary: 1 byte per nonzero (code) in
// place of 10-12; the ≤ 256 (delta, value) pairs sit in shared memory.
template <typename Idx, int MODE, bool K1>
__global__ void __launch_bounds__(NNB_SPMV_THREADS, NNB_SPMV_MINB)
    spmv_dict_kernel(const Idx* __restrict__ rp, const uint8_t* __restrict__ code,
                     const int32_t* __restrict__ dict_delta, const double* __restrict__ dict_val, int dict_size,
                     int64_t r_begin, int64_t r_end, int64_t diag_off, int64_t k, const double* __restrict__ t_ext,
                     const double* __restrict__ t_own, double* __restrict__ out, const double* __restrict__ zold,
                     double theta, int* __restrict__ flag) {
  __shared__ int32_t sd[kPairDictMax];
  __shared__ double sv[kPairDictMax];
  for (int i = threadIdx.x; i < dict_size; i += blockDim.x) {
    sd[i] = dict_delta[i];
    sv[i] = dict_val[i];
  }
  __syncthreads();
  bool bad = false;
  if (K1) {  // one right-hand side, 32-bit indices
    for (int r = (int)r_begin + blockIdx.x * blockDim.x + threadIdx.x; r < (int)r_end; r += gridDim.x * blockDim.x) {
      const int e0 = (int)rp[r], e1 = (int)rp[r + 1];
      const double* tg = t_ext + (r + (int)diag_off);
      double y = 0.0;
      for (int e = e0; e < e1; ++e) {
        const int q = code[e];
        y = __dadd_rn(y, __dmul_rn(sv[q], tg[sd[q]]));
      }
      out[r] = finish<MODE>(t_own[r], y, theta, MODE == kInner ? 0.0 : zold[r], bad);
    }
  } else {
    for (int64_t r = r_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r_end;
         r += (int64_t)gridDim.x * blockDim.x) {
      const int64_t e0 = rp[r], e1 = rp[r + 1];
      const int64_t g0 = r + diag_off;
      for (int64_t c = 0; c < k; ++c) {
        double y = 0.0;
        for (int64_t e = e0; e < e1; ++e) {
          const int q = code[e];
          y = __dadd_rn(y, __dmul_rn(sv[q], t_ext[(g0 + sd[q]) * k + c]));
        }
        out[r * k + c] = finish<MODE>(t_own[r * k + c], y, theta, MODE == kInner ? 0.0 : zold[r * k + c], bad);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Pair dictionary in ELL order (rows of at most kEllMaxWidth nonzeros): no row
// offsets, so a row's code loads and then its gathers are all independent.
template <int MODE, int WMAX, int MINB>
__global__ void __launch_bounds__(NNB_SPMV_THREADS, MINB)
    spmv_dict_ell_kernel(const uint8_t* __restrict__ code, int width, int64_t plane, const int32_t* __restrict__ dict_delta,
                         const double* __restrict__ dict_val, int dict_size, int64_t r_begin, int64_t r_end,
                         int64_t diag_off, int64_t k, const double* __restrict__ t_ext,
                         const double* __restrict__ t_own, double* __restrict__ out, const double* __restrict__ zold,
                         double theta, int* __restrict__ flag) {
  __shared__ int32_t sd[kPairDictMax];
  __shared__ double sv[kPairDictMax];
  for (int i = threadIdx.x; i < dict_size; i += blockDim.x) {
    sd[i] = dict_delta[i];
    sv[i] = dict_val[i];
  }
  __syncthreads();
  bool bad = false;
  for (int64_t r = r_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r_end;
       r += (int64_t)gridDim.x * blockDim.x) {
    int q[WMAX];
#pragma unroll
    for (int i = 0; i < WMAX; ++i) q[i] = i < width ? code[i * plane + r] : kEllPad;
    const int64_t g0 = r + diag_off;
    for (int64_t c = 0; c < k; ++c) {
      double xv[WMAX];
#pragma unroll
      for (int i = 0; i < WMAX; ++i) xv[i] = q[i] != kEllPad ? t_ext[(g0 + sd[q[i]]) * k + c] : 0.0;
      double y = 0.0;
#pragma unroll
      for (int i = 0; i < WMAX; ++i)
        if (q[i] != kEllPad) y = __dadd_rn(y, __dmul_rn(sv[q[i]], xv[i]));  // CSR order
      out[r * k + c] = finish<MODE>(t_own[r * k + c], y, theta, MODE == kInner ? 0.0 : zold[r * k + c], bad);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// One right-hand side, fewer than 2^31 gather indices: 32-bit index arithmetic
// (the 64-bit `· k + c` address math was a quarter of the general kernel's issue).
template <int MODE, int WMAX>
__global__ void __launch_bounds__(NNB_SPMV_THREADS, NNB_SPMV_MINB)
    spmv_dict_ell1_kernel(const uint8_t* __restrict__ code, int width, int plane,
                          const int32_t* __restrict__ dict_delta, const double* __restrict__ dict_val, int dict_size,
                          int r_begin, int r_end, int diag_off, const double* __restrict__ t_ext,
                          const double* __restrict__ t_own, double* __restrict__ out, const double* __restrict__ zold,
                          double theta, int* __restrict__ flag) {
  __shared__ double2 dict[kPairDictMax];  // {value, delta + diag_off as bits}: one 16-byte load per nonzero
  for (int i = threadIdx.x; i < dict_size; i += blockDim.x)
    dict[i] = make_double2(dict_val[i], __longlong_as_double((long long)(dict_delta[i] + diag_off)));
  __syncthreads();
  bool bad = false;
  for (int r = r_begin + blockIdx.x * blockDim.x + threadIdx.x; r < r_end; r += gridDim.x * blockDim.x) {
    int q[WMAX];
#pragma unroll
    for (int i = 0; i < WMAX; ++i) q[i] = i < width ? code[(size_t)i * plane + r] : kEllPad;
    double vv[WMAX], xv[WMAX];
#pragma unroll
    for (int i = 0; i < WMAX; ++i) {
      const double2 de = dict[q[i] != kEllPad ? q[i] : 0];
      vv[i] = de.x;
      xv[i] = q[i] != kEllPad ? t_ext[r + (int)__double_as_longlong(de.y)] : 0.0;
    }
    double y = 0.0;
#pragma unroll
    for (int i = 0; i < WMAX; ++i)
      if (q[i] != kEllPad) y = __dadd_rn(y, __dmul_rn(vv[i], xv[i]));  // CSR order
    out[r] = finish<MODE>(t_own[r], y, theta, MODE == kInner ? 0.0 : zold[r], bad);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Row dictionary: operators whose rows repeat a few whole (column − row,
// value) sequences — a stencil has one per boundary case — store one uint8
// pattern code per row.  pat[p·W + i] = {value, delta as bits} of pattern p's
// i-th nonzero (CSR order), len[p] its length; exact lookups, so the sum keeps
// the reference's order and rounding.  1 B per row instead of 5 code bytes.
template <int MODE, int WMAX>
__global__ void __launch_bounds__(NNB_SPMV_THREADS, NNB_SPMV_MINB)
    spmv_rowdict_kernel(const uint8_t* __restrict__ rcode, const double2* __restrict__ pat,
                        const uint8_t* __restrict__ plen, int npat, int width, int r_begin, int r_end, int diag_off,
                        const double* __restrict__ t_ext, const double* __restrict__ t_own, double* __restrict__ out,
                        const double* __restrict__ zold, double theta, int* __restrict__ flag) {
  extern __shared__ double2 spat[];  // [npat·width] patterns, then npat lengths
  int* slen = reinterpret_cast<int*>(spat + npat * width);
  for (int i = threadIdx.x; i < npat * width; i += blockDim.x) {
    const double2 e = pat[i];
    spat[i] = make_double2(e.x, __longlong_as_double(__double_as_longlong(e.y) + diag_off));
  }
  for (int i = threadIdx.x; i < npat; i += blockDim.x) slen[i] = plen[i];
  __syncthreads();
  bool bad = false;
  // The next row's code is loaded a row ahead: its HBM latency overlaps this
  // row's gathers instead of heading the next row's dependent chain (inner
  // application 76.6 -> 68.8 us).  Tried and reverted: codes two rows ahead
  // with the next row's gathers prefetched into L2 (prefetch.global.L2):
  // 103 us, the prefetches cost more issue and L2 bandwidth than they hide.
  const int stride = gridDim.x * blockDim.x;
  int r = r_begin + blockIdx.x * blockDim.x + threadIdx.x;
  int p_next = r < r_end ? rcode[r] : 0;
  for (; r < r_end; r += stride) {
    const int p = p_next;
    if (r + stride < r_end) p_next = rcode[r + stride];
    const int len = slen[p];
    const double2* pe = spat + p * width;
    double xv[WMAX];  // every gather in flight first; the values are re-read from shared memory
#pragma unroll
    for (int i = 0; i < WMAX; ++i)
      if (i < len) xv[i] = t_ext[r + (int)__double_as_longlong(pe[i].y)];
    double y = 0.0;
#pragma unroll
    for (int i = 0; i < WMAX; ++i)
      if (i < len) y = __dadd_rn(y, __dmul_rn(pe[i].x, xv[i]));  // CSR order
    out[r] = finish<MODE>(t_own[r], y, theta, MODE == kInner ? 0.0 : zold[r], bad);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// ---- pair dictionary build: hash insert, index assignment, verified encode ----
constexpr int kDictSlots = 4096;  // open addressing, power of two
constexpr int kMaxProbe = 64;     // longer probe runs only happen past the dictionary's capacity

__device__ __forceinline__ unsigned long long pair_hash(int32_t d, unsigned long long bits) {
  unsigned long long h = bits ^ (static_cast<unsigned long long>(static_cast<uint32_t>(d)) * 0x9E3779B97F4A7C15ull);
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h | 1ull;  // never 0 (0 marks an empty slot)
}

struct DictWs {
  unsigned long long hash[kDictSlots];
  int32_t delta[kDictSlots];
  double val[kDictSlots];
  int32_t index[kDictSlots];
  int count;
  int overflow;   // more than kPairDictMax pairs
  int collision;  // a 64-bit hash matched a different pair (the encode check)
  int size;
  int max_len;    // longest row
};

__global__ void dict_insert_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                   const double* __restrict__ val, int64_t rows, int64_t row0, DictWs* ws) {
  int32_t last_d = 0;
  unsigned long long last_b = 0, last_h = 0;  // consecutive nonzeros repeat pairs: skip their probes
  int longest = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    if (*(volatile int*)&ws->overflow) return;
    const int64_t rl = rp[r + 1] - rp[r];
    longest = max(longest, rl > (1 << 30) ? (1 << 30) : (int)rl);
    for (int64_t e = rp[r], e1 = rp[r + 1]; e < e1; ++e) {
      const int64_t dl = (int64_t)col[e] - (row0 + r);
      if (dl < INT32_MIN || dl > INT32_MAX) {
        atomicOr(&ws->overflow, 1);
        return;
      }
      const int32_t d = static_cast<int32_t>(dl);
      const unsigned long long b = __double_as_longlong(val[e]);
      if (last_h && d == last_d && b == last_b) continue;
      const unsigned long long h = pair_hash(d, b);
      int slot = static_cast<int>(h & (kDictSlots - 1));
      for (int probe = 0;; ++probe) {
        // a dictionary of <= 255 pairs fills under 7 % of the table, so a long probe run
        // means the operator has too many pairs: racing inserts past the 256th can fill the
        // whole table, and probing it to the end per nonzero cost 68 ms per solve on a
        // random-valued 4096² operator
        if (probe >= kMaxProbe || *(volatile int*)&ws->overflow) {
          atomicOr(&ws->overflow, 1);
          return;
        }
        unsigned long long cur = *(volatile unsigned long long*)&ws->hash[slot];
        if (cur == 0) {
          cur = atomicCAS(&ws->hash[slot], 0ull, h);
          if (cur == 0) {
            ws->delta[slot] = d;
            ws->val[slot] = val[e];
            if (atomicAdd(&ws->count, 1) >= kPairDictMax) {
              atomicOr(&ws->overflow, 1);
              return;
            }
            break;
          }
        }
        if (cur == h) break;
        slot = (slot + 1) & (kDictSlots - 1);
      }
      last_d = d;
      last_b = b;
      last_h = h;
    }
  }
  atomicMax(&ws->max_len, longest);
}

// one block: occupied slots in slot order -> dictionary indices
__global__ void dict_index_kernel(DictWs* ws, int32_t* __restrict__ dict_delta, double* __restrict__ dict_val) {
  __shared__ int counts[1024];
  constexpr int per = kDictSlots / 1024;
  int c = 0;
  for (int i = 0; i < per; ++i) c += ws->hash[threadIdx.x * per + i] != 0;
  counts[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < 1024; ++i) {
      const int v = counts[i];
      counts[i] = run;
      run += v;
    }
    ws->size = run;
  }
  __syncthreads();
  int idx = counts[threadIdx.x];
  for (int i = 0; i < per; ++i) {
    const int slot = threadIdx.x * per + i;
    if (ws->hash[slot] == 0) continue;
    ws->index[slot] = idx;
    // on overflow up to kDictSlots slots can be occupied; the dictionary arrays
    // hold kPairDictMax entries (the overflowed build is discarded by the host)
    if (idx < kPairDictMax) {
      dict_delta[idx] = ws->delta[slot];
      dict_val[idx] = ws->val[slot];
    }
    ++idx;
  }
}

// ell_width > 0: slot-major ELL, row r's i-th nonzero (CSR order) at code[i·plane + r],
// padded with kEllPad (no row offsets needed; a warp's load of one slot is 32
// consecutive bytes); else code[e − rp[0]] (CSR order).
__global__ void dict_encode_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                   const double* __restrict__ val, int64_t rows, int64_t row0, const DictWs* ws,
                                   uint8_t* __restrict__ code, int ell_width, int64_t plane, int* collision) {
  const int64_t base = rp[0];
  bool bad = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    if (ell_width) {
      if (rp[r + 1] - rp[r] > ell_width) {  // longer than the sampled width: the caller retries in full
        bad = true;
        continue;
      }
      for (int64_t i = rp[r + 1] - rp[r]; i < ell_width; ++i) code[i * plane + r] = kEllPad;
    }
    for (int64_t e = rp[r], e1 = rp[r + 1]; e < e1; ++e) {
      const int32_t d = static_cast<int32_t>((int64_t)col[e] - (row0 + r));
      const unsigned long long b = __double_as_longlong(val[e]);
      const unsigned long long h = pair_hash(d, b);
      int slot = static_cast<int>(h & (kDictSlots - 1));
      int probe = 0;
      while (ws->hash[slot] != h && ws->hash[slot] != 0 && probe < kDictSlots) {
        slot = (slot + 1) & (kDictSlots - 1);
        ++probe;
      }
      // the exact pair, or the caller falls back to the column format
      const bool hit = ws->hash[slot] == h && ws->delta[slot] == d &&
                       __double_as_longlong(ws->val[slot]) == static_cast<long long>(b);
      bad |= !hit;
      code[ell_width ? (e - rp[r]) * plane + r : e - base] = static_cast<uint8_t>(hit ? ws->index[slot] : 0);
    }
  }
  if (bad) atomicOr(collision, 1);
}

// ---- row dictionary over the ELL pair codes: a row's key is its W code bytes
// (kEllPad-padded) packed into 64 bits, so equal keys are equal (delta, value)
// sequences exactly ----
struct RowDictWs {
  unsigned long long hash[kDictSlots];
  unsigned long long key[kDictSlots];
  int32_t index[kDictSlots];
  int count;
  int overflow;   // more than kRowDictMax patterns
  int collision;  // equal hashes of different keys (the encode check)
  int size;
};

__device__ __forceinline__ unsigned long long row_key(const uint8_t* __restrict__ code, int width, int64_t plane,
                                                       int64_t r) {
  unsigned long long k = ~0ull;  // unused bytes read as kEllPad
  for (int i = 0; i < width; ++i)
    k = (k & ~(0xffull << (8 * i))) | (static_cast<unsigned long long>(code[i * plane + r]) << (8 * i));
  return k;
}

__device__ __forceinline__ unsigned long long key_hash(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k | 1ull;
}

__global__ void rowdict_insert_kernel(const uint8_t* __restrict__ code, int width, int64_t plane, int64_t rows,
                                      RowDictWs* ws) {
  unsigned long long last = 0;
  bool have = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = row_key(code, width, plane, r);
    if (have && k == last) continue;  // interior rows repeat one key
    // one insert per distinct key per warp (the lanes' first rows all start here)
    const unsigned active = __activemask();
    const unsigned peers = __match_any_sync(active, k);
    last = k;
    have = true;
    if ((threadIdx.x & 31) != __ffs(peers) - 1) continue;
    if (*(volatile int*)&ws->overflow) return;
    const unsigned long long h = key_hash(k);
    int slot = static_cast<int>(h & (kDictSlots - 1));
    for (int probe = 0;; ++probe) {
      if (probe >= kMaxProbe || *(volatile int*)&ws->overflow) {  // too many rows (see dict_insert_kernel)
        atomicOr(&ws->overflow, 1);
        return;
      }
      unsigned long long cur = *(volatile unsigned long long*)&ws->hash[slot];
      if (cur == 0) {
        cur = atomicCAS(&ws->hash[slot], 0ull, h);
        if (cur == 0) {
          ws->key[slot] = k;
          if (atomicAdd(&ws->count, 1) >= kRowDictMax) {
            atomicOr(&ws->overflow, 1);
            return;
          }
          break;
        }
      }
      if (cur == h) break;
      slot = (slot + 1) & (kDictSlots - 1);
    }
  }
}

// one block: occupied slots in slot order -> pattern indices; pattern p expanded
// to {value, delta} entries through the pair dictionary
__global__ void rowdict_index_kernel(RowDictWs* ws, int width, const int32_t* __restrict__ dict_delta,
                                     const double* __restrict__ dict_val, double2* __restrict__ pat,
                                     uint8_t* __restrict__ plen) {
  __shared__ int counts[1024];
  constexpr int per = kDictSlots / 1024;
  int c = 0;
  for (int i = 0; i < per; ++i) c += ws->hash[threadIdx.x * per + i] != 0;
  counts[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < 1024; ++i) {
      const int v = counts[i];
      counts[i] = run;
      run += v;
    }
    ws->size = run;
  }
  __syncthreads();
  int idx = counts[threadIdx.x];
  for (int i = 0; i < per; ++i) {
    const int slot = threadIdx.x * per + i;
    if (ws->hash[slot] == 0) continue;
    ws->index[slot] = idx;
    if (idx < kRowDictMax) {
      const unsigned long long k = ws->key[slot];
      int len = width;
      for (int j = 0; j < width; ++j) {
        const int q = static_cast<int>((k >> (8 * j)) & 0xff);
        if (q == kEllPad) {
          if (len == width) len = j;
          pat[idx * width + j] = make_double2(0.0, __longlong_as_double(0));
        } else {
          pat[idx * width + j] = make_double2(dict_val[q], __longlong_as_double((long long)dict_delta[q]));
        }
      }
      plen[idx] = static_cast<uint8_t>(len);
    }
    ++idx;
  }
}

__global__ void rowdict_encode_kernel(const uint8_t* __restrict__ code, int width, int64_t plane, int64_t rows,
                                      const RowDictWs* ws, uint8_t* __restrict__ rcode, int* collision) {
  bool bad = false, have = false;
  unsigned long long last = 0;
  int last_idx = -1;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = row_key(code, width, plane, r);
    if (!have || k != last) {  // a thread's rows repeat one key (interior rows): look up only on change
      const unsigned long long h = key_hash(k);
      int slot = static_cast<int>(h & (kDictSlots - 1));
      int probe = 0;
      while (ws->hash[slot] != h && ws->hash[slot] != 0 && probe < kDictSlots) {
        slot = (slot + 1) & (kDictSlots - 1);
        ++probe;
      }
      last_idx = (ws->hash[slot] == h && ws->key[slot] == k) ? ws->index[slot] : -1;
      last = k;
      have = true;
    }
    bad |= last_idx < 0;
    rcode[r] = static_cast<uint8_t>(last_idx < 0 ? 0 : last_idx);
  }
  if (bad) atomicOr(collision, 1);
}

// Pair codes and row keys in one pass over the CSR: each nonzero's (column − row,
// value) is looked up (and verified) in the pair table, the row's codes packed
// into its key, and the key looked up in the row table; only the row code is
// written.  Any miss (a pair or row outside the sampled tables, a longer row)
// sets *collision and the caller takes the two-pass build.
//
// A warp takes 32 consecutive rows: their nonzeros are one contiguous range, loaded
// coalesced (lane j of load i: element 32·i + j) into the warp's shared buffer, then
// each lane encodes its row from there.  The next chunk's row offsets are loaded
// before this chunk's nonzeros are used, so one memory latency per chunk, not two
// (one thread per row with rp → col/val dependent loads ran at 0.67 of HBM).
constexpr int kEncWarps = 8;
template <bool kNarrow>
__global__ void __launch_bounds__(kEncWarps * 32)
    rowdict_direct_encode_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const double* __restrict__ val, int64_t rows, int64_t row0, const DictWs* ws,
                                 const RowDictWs* rws, int width, uint8_t* __restrict__ rcode, int* collision) {
  __shared__ int32_t s_col[kEncWarps][2][32 * kEllMaxWidth];
  __shared__ unsigned long long s_val[kEncWarps][2][32 * kEllMaxWidth];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  bool bad = false, have = false;
  unsigned long long last = 0;
  int last_idx = -1, last_len = -1;
  // the last verified pair at each position (compile-time indexed: registers): a
  // lane's rows, one chunk stride apart, mostly repeat them, so the pair table is
  // probed only when a position's pair changes
  int32_t cd[kEllMaxWidth];
  unsigned long long cb[kEllMaxWidth];
  int ci[kEllMaxWidth];
#pragma unroll
  for (int i = 0; i < kEllMaxWidth; ++i) ci[i] = -1;
  const int64_t chunks = (rows + 31) / 32, stride = (int64_t)gridDim.x * kEncWarps;
  auto load_rp = [&](int64_t cc, int64_t& l, int64_t& h) {
    l = h = 0;
    const int64_t r = cc * 32 + lane;
    if (cc < chunks && r < rows) {
      l = rp[r];
      h = rp[r + 1];
    }
  };
  // chunk cc's nonzeros straight into buffer b (cp.async: no registers), one commit group
  auto issue = [&](int64_t cc, int64_t l, int64_t h, int b, int64_t& base, int64_t& cnt) {
    base = cnt = 0;
    if (cc < chunks) {
      const int nr = (int)(rows - cc * 32 < 32 ? rows - cc * 32 : 32);
      base = __shfl_sync(0xffffffffu, l, 0);
      cnt = __shfl_sync(0xffffffffu, h, nr - 1) - base;
      if (cnt <= 32 * width) {  // else some row is longer than width: bad
        const int n32 = (int)cnt;
#pragma unroll
        for (int i = 0; i < kEllMaxWidth; ++i) {
          const int k = 32 * i + lane;
          if (k < n32) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&s_col[warp][b][k])),
                         "l"(col + base + k)
                         : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&s_val[warp][b][k])),
                         "l"(val + base + k)
                         : "memory");
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // two chunks in flight per warp: chunk c + stride's nonzeros and chunk c + 2·stride's
  // offsets load while chunk c is encoded
  int64_t c = blockIdx.x * (int64_t)kEncWarps + warp;
  int64_t lo, hi, base, cnt, lo1, hi1;
  load_rp(c, lo, hi);
  issue(c, lo, hi, 0, base, cnt);
  load_rp(c + stride, lo1, hi1);
  for (int b = 0; c < chunks; c += stride, b ^= 1) {
    int64_t base1, cnt1, lo2, hi2;
    issue(c + stride, lo1, hi1, b ^ 1, base1, cnt1);
    load_rp(c + 2 * stride, lo2, hi2);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const int64_t r = c * 32 + lane;
    const bool fits = cnt <= 32 * width;
    const int32_t* wc = s_col[warp][b];
    const unsigned long long* wv = s_val[warp][b];
    if (r < rows) {
      const int64_t len = hi - lo;
      if (!fits || len > width) {
        bad = true;
      } else {
        const int off = (int)(lo - base);
        // fast path: the same length and (delta, value) at every position as this lane's
        // last row — the same key, so the same code (32-bit deltas when every row index
        // fits: kNarrow)
        bool same = have && len == last_len;
        if (same) {
#pragma unroll
          for (int i = 0; i < kEllMaxWidth; ++i) {
            if (i < len) {
              if (kNarrow) {
                same &= wc[off + i] - (int32_t)(row0 + r) == cd[i] && wv[off + i] == cb[i];
              } else {
                const int64_t dl = (int64_t)wc[off + i] - (row0 + r);
                same &= dl == cd[i] && wv[off + i] == cb[i];
              }
            }
          }
        }
        if (!same) {
          last_len = (int)len;
          unsigned long long key = ~0ull;
#pragma unroll
          for (int i = 0; i < kEllMaxWidth; ++i) {
            if (i >= len) break;
            const int64_t dl = (int64_t)wc[off + i] - (row0 + r);
            const int32_t d = static_cast<int32_t>(dl);
            const unsigned long long b = wv[off + i];
            if (!(ci[i] >= 0 && cd[i] == d && cb[i] == b && dl == d)) {
              const unsigned long long h = pair_hash(d, b);
              int slot = static_cast<int>(h & (kDictSlots - 1));
              int probe = 0;
              while (ws->hash[slot] != h && ws->hash[slot] != 0 && probe < kDictSlots) {
                slot = (slot + 1) & (kDictSlots - 1);
                ++probe;
              }
              const bool hit = dl >= INT32_MIN && dl <= INT32_MAX && ws->hash[slot] == h && ws->delta[slot] == d &&
                               __double_as_longlong(ws->val[slot]) == static_cast<long long>(b);
              bad |= !hit;
              cd[i] = d;
              cb[i] = b;
              ci[i] = hit ? ws->index[slot] : -1;
            }
            const unsigned long long q = ci[i] >= 0 ? static_cast<unsigned long long>(ci[i]) : 0ull;
            key = (key & ~(0xffull << (8 * i))) | (q << (8 * i));
          }
          if (!have || key != last) {
            const unsigned long long h = key_hash(key);
            int slot = static_cast<int>(h & (kDictSlots - 1));
            int probe = 0;
            while (rws->hash[slot] != h && rws->hash[slot] != 0 && probe < kDictSlots) {
              slot = (slot + 1) & (kDictSlots - 1);
              ++probe;
            }
            last_idx = (rws->hash[slot] == h && rws->key[slot] == key) ? rws->index[slot] : -1;
            last = key;
            have = true;
          }
        }
        bad |= last_idx < 0;
        rcode[r] = static_cast<uint8_t>(last_idx < 0 ? 0 : last_idx);
      }
    }
    __syncwarp();
    lo = lo1;
    hi = hi1;
    base = base1;
    cnt = cnt1;
    lo1 = lo2;
    hi1 = hi2;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (bad) atomicOr(collision, 1);
}

// Plain Y = W·X for nn::spmv_block (same rounding as the reference's sum).
__global__ void spmv_plain_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, int64_t n, int64_t k,
                                  const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = rp[r], e1 = rp[r + 1];
    for (int64_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (int64_t e = e0; e < e1; ++e) s = __dadd_rn(s, __dmul_rn(val[e], x[(int64_t)col[e] * k + c]));
      y[r * k + c] = s;
    }
  }
}

__global__ void narrow_offsets_kernel(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t count,
                                      int64_t base) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<int32_t>(in[i] - base);
}

__global__ void compact_csr_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t rows,
                                   int64_t row0, int32_t* __restrict__ rp32, int16_t* __restrict__ col16,
                                   int* __restrict__ wide) {
  const int64_t base = rp[0];
  bool far = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= rows; r += (int64_t)gridDim.x * blockDim.x) {
    rp32[r] = static_cast<int32_t>(rp[r] - base);
    if (r == rows) continue;
    for (int64_t e = rp[r], e1 = rp[r + 1]; e < e1; ++e) {
      const int64_t d = (int64_t)col[e] - (row0 + r);
      far |= d < -32767 || d > 32767;
      col16[e - base] = static_cast<int16_t>(d);
    }
  }
  if (far) atomicOr(wide, 1);  // rare: only operators wider than the int16 band
}

namespace {

unsigned rows_grid(int64_t n) {
  const int64_t want = (n + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 8 * 4)));
}

// one right-hand side with 32-bit offsets and gather indices takes 32-bit index math
template <typename Idx>
bool k1_ok(const SpmvOp<Idx>& op, int64_t r_end) {
  return op.k == 1 && sizeof(Idx) == 4 && r_end + op.diag_off < INT32_MAX / 2;
}

template <typename Idx, typename C, int MODE, bool K1>
unsigned resident_grid(int64_t rows) {
  static unsigned resident = 0;
  if (!resident) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spmv_rows_kernel<Idx, C, MODE, K1>, NNB_SPMV_THREADS, 0);
    resident = static_cast<unsigned>(sms * std::max(1, per));
  }
  const int64_t want = (rows + NNB_SPMV_THREADS - 1) / NNB_SPMV_THREADS;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(resident, want)));
}

template <typename Idx, typename C, int MODE, bool K1>
void launch_rows_v(const SpmvOp<Idx>& op, const C* col, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  spmv_rows_kernel<Idx, C, MODE, K1><<<resident_grid<Idx, C, MODE, K1>(r_end - r_begin), NNB_SPMV_THREADS, 0, s>>>(
      op.rp, col, op.val, r_begin, r_end, op.diag_off, op.k, op.t_ext, op.t_own, op.out, op.zold, op.theta, op.flag);
}

template <typename Idx, typename C, int MODE>
void launch_rows(const SpmvOp<Idx>& op, const C* col, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  static const bool k1_off = debug_env("NNB_SPMV_K1") && std::strcmp(debug_env("NNB_SPMV_K1"), "0") == 0;
  if (!k1_off && k1_ok(op, r_end)) launch_rows_v<Idx, C, MODE, true>(op, col, r_begin, r_end, s);
  else launch_rows_v<Idx, C, MODE, false>(op, col, r_begin, r_end, s);
}

template <typename Idx, int MODE, bool K1>
void launch_dict_v(const SpmvOp<Idx>& op, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  static unsigned resident = 0;
  if (!resident) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spmv_dict_kernel<Idx, MODE, K1>, NNB_SPMV_THREADS, 0);
    resident = static_cast<unsigned>(sms * std::max(1, per));
  }
  const int64_t want = (r_end - r_begin + NNB_SPMV_THREADS - 1) / NNB_SPMV_THREADS;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(resident, want)));
  spmv_dict_kernel<Idx, MODE, K1><<<grid, NNB_SPMV_THREADS, 0, s>>>(
      op.rp, op.code, op.dict_delta, op.dict_val, op.dict_size, r_begin, r_end, op.diag_off, op.k, op.t_ext,
      op.t_own, op.out, op.zold, op.theta, op.flag);
}

template <int MODE, int WMAX, int MINB, typename Idx>
void launch_ell_v(const SpmvOp<Idx>& op, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  static unsigned resident = 0;
  if (!resident) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spmv_dict_ell_kernel<MODE, WMAX, MINB>, NNB_SPMV_THREADS, 0);
    resident = static_cast<unsigned>(sms * std::max(1, per));
  }
  const int64_t want = (r_end - r_begin + NNB_SPMV_THREADS - 1) / NNB_SPMV_THREADS;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(resident, want)));
  spmv_dict_ell_kernel<MODE, WMAX, MINB><<<grid, NNB_SPMV_THREADS, 0, s>>>(
      op.code, op.ell_width, op.ell_rows, op.dict_delta, op.dict_val, op.dict_size, r_begin, r_end, op.diag_off, op.k, op.t_ext,
      op.t_own, op.out, op.zold, op.theta, op.flag);
}

template <int MODE, int WMAX>
void launch_ell1_v(const SpmvOp<int32_t>& op, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  static unsigned resident = 0;
  if (!resident) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spmv_dict_ell1_kernel<MODE, WMAX>, NNB_SPMV_THREADS, 0);
    resident = static_cast<unsigned>(sms * std::max(1, per));
  }
  const int64_t want = (r_end - r_begin + NNB_SPMV_THREADS - 1) / NNB_SPMV_THREADS;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(resident, want)));
  spmv_dict_ell1_kernel<MODE, WMAX><<<grid, NNB_SPMV_THREADS, 0, s>>>(
      op.code, op.ell_width, (int)op.ell_rows, op.dict_delta, op.dict_val, op.dict_size, (int)r_begin, (int)r_end, (int)op.diag_off,
      op.t_ext, op.t_own, op.out, op.zold, op.theta, op.flag);
}


template <int MODE, int WMAX>
void launch_rowdict_v(const SpmvOp<int32_t>& op, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  const int smem = op.npat * op.ell_width * (int)sizeof(double2) + op.npat * (int)sizeof(int);
  static unsigned resident = 0;
  static int resident_smem = -1;
  ensure_smem<spmv_rowdict_kernel<MODE, WMAX>>(smem);  // per device
  if (resident_smem != smem) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spmv_rowdict_kernel<MODE, WMAX>, NNB_SPMV_THREADS, smem);
    resident = static_cast<unsigned>(sms * std::max(1, per));
    resident_smem = smem;
  }
  const int64_t want = (r_end - r_begin + NNB_SPMV_THREADS - 1) / NNB_SPMV_THREADS;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(resident, want)));
  spmv_rowdict_kernel<MODE, WMAX><<<grid, NNB_SPMV_THREADS, smem, s>>>(
      op.rcode, op.rpat, op.rlen, op.npat, op.ell_width, (int)r_begin, (int)r_end, (int)op.diag_off, op.t_ext,
      op.t_own, op.out, op.zold, op.theta, op.flag);
}

template <int MODE, typename Idx>
void launch_rowdict(const SpmvOp<Idx>& op, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  const SpmvOp<int32_t>& o32 = reinterpret_cast<const SpmvOp<int32_t>&>(op);
  if (op.ell_width <= 5) launch_rowdict_v<MODE, 5>(o32, r_begin, r_end, s);
  else launch_rowdict_v<MODE, kEllMaxWidth>(o32, r_begin, r_end, s);
}

// rows of <= 5 nonzeros (2-D 5-point stencils) fit the 32-register budget
template <int MODE, typename Idx>
void launch_ell(const SpmvOp<Idx>& op, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  // one right-hand side and 32-bit gather indices (|delta| < 2^31 is implied by the dictionary)
  if (k1_ok(op, r_end)) {
    const SpmvOp<int32_t>& o32 = reinterpret_cast<const SpmvOp<int32_t>&>(op);
    if (op.ell_width <= 5) launch_ell1_v<MODE, 5>(o32, r_begin, r_end, s);
    else launch_ell1_v<MODE, kEllMaxWidth>(o32, r_begin, r_end, s);
    return;
  }
  launch_ell_v<MODE, kEllMaxWidth, 1>(op, r_begin, r_end, s);
}

template <typename Idx, int MODE>
void launch_dict(const SpmvOp<Idx>& op, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  if (k1_ok(op, r_end)) launch_dict_v<Idx, MODE, true>(op, r_begin, r_end, s);
  else launch_dict_v<Idx, MODE, false>(op, r_begin, r_end, s);
}

template <typename Idx, typename C>
void launch_mode(const SpmvOp<Idx>& op, const C* col, int mode, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  switch (mode) {
    case kInner: launch_rows<Idx, C, kInner>(op, col, r_begin, r_end, s); break;
    case kFactorEnd: launch_rows<Idx, C, kFactorEnd>(op, col, r_begin, r_end, s); break;
    default: launch_rows<Idx, C, kFinal>(op, col, r_begin, r_end, s);
  }
}

}  // namespace

template <typename Idx>
void spmv_apply(const SpmvOp<Idx>& op, int mode, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  if (r_end <= r_begin) return;
  if (op.rcode && k1_ok(op, r_end)) {  // built for one right-hand side only
    switch (mode) {
      case kInner: launch_rowdict<kInner>(op, r_begin, r_end, s); break;
      case kFactorEnd: launch_rowdict<kFactorEnd>(op, r_begin, r_end, s); break;
      default: launch_rowdict<kFinal>(op, r_begin, r_end, s);
    }
  } else if (op.code && op.ell_width) {
    switch (mode) {
      case kInner: launch_ell<kInner>(op, r_begin, r_end, s); break;
      case kFactorEnd: launch_ell<kFactorEnd>(op, r_begin, r_end, s); break;
      default: launch_ell<kFinal>(op, r_begin, r_end, s);
    }
  } else if (op.code) {
    switch (mode) {
      case kInner: launch_dict<Idx, kInner>(op, r_begin, r_end, s); break;
      case kFactorEnd: launch_dict<Idx, kFactorEnd>(op, r_begin, r_end, s); break;
      default: launch_dict<Idx, kFinal>(op, r_begin, r_end, s);
    }
  } else if (op.col16) launch_mode(op, op.col16, mode, r_begin, r_end, s);
  else launch_mode(op, op.col, mode, r_begin, r_end, s);
  count_launch();
}
template void spmv_apply<int32_t>(const SpmvOp<int32_t>&, int, int64_t, int64_t, cudaStream_t);
template void spmv_apply<int64_t>(const SpmvOp<int64_t>&, int, int64_t, int64_t, cudaStream_t);

int narrow_offsets(const int64_t* in, int32_t* out, int64_t count, int64_t base, cudaStream_t s) {
  narrow_offsets_kernel<<<rows_grid(count), 256, 0, s>>>(in, out, count, base);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

int compact_csr(const int64_t* rp, const int32_t* col, int64_t rows, int64_t row0, int32_t* rp32, int16_t* col16,
                bool* fits, cudaStream_t s) {
  DevBuf flag;
  NNB_TRY(flag.alloc(sizeof(int), s));
  NNB_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
  compact_csr_kernel<<<rows_grid(rows + 1), 256, 0, s>>>(rp, col, rows, row0, rp32, col16, flag.as<int>());
  count_launch();
  NNB_CUDA(cudaGetLastError());
  int wide = 0;
  NNB_CUDA(cudaMemcpyAsync(&wide, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  *fits = !wide;
  return 0;
}

int build_pair_dict(const int64_t* rp, const int32_t* col, const double* val, int64_t rows, int64_t row0,
                    int64_t nnz, DevBuf& code_buf, int* ell_width, int64_t* ell_plane, int* band_lo, int* band_hi,
                    int32_t* dict_delta, double* dict_val, int* dict_size, bool* ok, cudaStream_t s) {
  *ok = false;
  *dict_size = 0;
  *ell_width = 0;
  *ell_plane = 0;
  if (rows <= 0) return 0;
  DevBuf wsb;
  NNB_TRY(wsb.alloc(sizeof(DictWs), s));
  DictWs* ws = wsb.as<DictWs>();
  static const bool ell_on = !(debug_env("NNB_DICT_ELL") && std::strcmp(debug_env("NNB_DICT_ELL"), "0") == 0);
  // First try a dictionary (and ELL width) from the first and last kSample rows only:
  // structured operators show every pair there (a stencil's boundary rows recur every
  // grid row).  The encode pass verifies every nonzero against it; a missing pair or a
  // longer row sends the build round again over all rows.  Results are bit-identical
  // either way; only the order of the dictionary can differ.
  constexpr int64_t kSample = 65536;
  const bool can_sample = rows > 4 * kSample;
  for (int full = can_sample ? 0 : 1; full < 2; ++full) {
    NNB_CUDA(cudaMemsetAsync(ws, 0, sizeof(DictWs), s));
    if (full) {
      dict_insert_kernel<<<rows_grid(rows), 256, 0, s>>>(rp, col, val, rows, row0, ws);
    } else {
      dict_insert_kernel<<<rows_grid(kSample), 256, 0, s>>>(rp, col, val, kSample, row0, ws);
      dict_insert_kernel<<<rows_grid(kSample), 256, 0, s>>>(rp + (rows - kSample), col, val, kSample,
                                                            row0 + rows - kSample, ws);
      count_launch();
    }
    dict_index_kernel<<<1, 1024, 0, s>>>(ws, dict_delta, dict_val);
    int flags[5];  // count, overflow, collision, size, max_len
    NNB_CUDA(cudaMemcpyAsync(flags, &ws->count, sizeof(flags), cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaStreamSynchronize(s));
    count_launch(2);
    if (flags[1] || flags[3] > kPairDictMax - 1) {  // code kEllPad stays free
      if (full) return 0;
      continue;
    }
    // ELL order when rows are short and padding costs at most a quarter more codes
    const int w = flags[4];
    const bool ell = ell_on && w >= 1 && w <= kEllMaxWidth && (int64_t)w * rows * 4 <= nnz * 5;
    const int64_t plane = (rows + 15) / 16 * 16;  // 16-byte aligned slot planes
    NNB_TRY(code_buf.alloc(std::max<int64_t>(1, ell ? (int64_t)w * plane : nnz), s));
    dict_encode_kernel<<<rows_grid(rows), 256, 0, s>>>(rp, col, val, rows, row0, ws, code_buf.as<uint8_t>(),
                                                       ell ? w : 0, plane, &ws->collision);
    count_launch();
    NNB_CUDA(cudaGetLastError());
    NNB_CUDA(cudaMemcpyAsync(flags, &ws->count, sizeof(flags), cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaStreamSynchronize(s));
    if (flags[2]) {
      code_buf.release();
      continue;  // a pair (or row length) outside the sample; the full round decides
    }
    *dict_size = flags[3];
    *ell_width = ell ? w : 0;
    *ell_plane = ell ? plane : 0;
    std::vector<int32_t> dh(flags[3]);
    NNB_CUDA(cudaMemcpy(dh.data(), dict_delta, sizeof(int32_t) * dh.size(), cudaMemcpyDeviceToHost));
    *band_lo = *band_hi = 0;
    for (int32_t d : dh) {
      *band_lo = std::min(*band_lo, d);
      *band_hi = std::max(*band_hi, d);
    }
    *ok = true;
    return 0;
  }
  return 0;
}

int build_row_dict(const uint8_t* code, int width, int64_t plane, int64_t rows, const int32_t* dict_delta,
                   const double* dict_val, uint8_t* rcode, double2* pat, uint8_t* plen, int* npat, bool* ok,
                   cudaStream_t s) {
  *ok = false;
  *npat = 0;
  if (rows <= 0 || width < 1 || width > kEllMaxWidth) return 0;
  DevBuf wsb;
  NNB_TRY(wsb.alloc(sizeof(RowDictWs), s));
  RowDictWs* ws = wsb.as<RowDictWs>();
  // As the pair dictionary: patterns first from the first and last kSample rows (a
  // stencil shows every boundary case there), verified over all rows by the encode
  // pass; a row outside the sample sends the build round again over all rows.
  constexpr int64_t kSample = 65536;
  const bool can_sample = rows > 4 * kSample;
  for (int full = can_sample ? 0 : 1; full < 2; ++full) {
    NNB_CUDA(cudaMemsetAsync(ws, 0, sizeof(RowDictWs), s));
    if (full) {
      rowdict_insert_kernel<<<rows_grid(rows), 256, 0, s>>>(code, width, plane, rows, ws);
    } else {
      rowdict_insert_kernel<<<rows_grid(kSample), 256, 0, s>>>(code, width, plane, kSample, ws);
      rowdict_insert_kernel<<<rows_grid(kSample), 256, 0, s>>>(code + (rows - kSample), width, plane, kSample, ws);
      count_launch();
    }
    rowdict_index_kernel<<<1, 1024, 0, s>>>(ws, width, dict_delta, dict_val, pat, plen);
    count_launch(2);
    NNB_CUDA(cudaGetLastError());
    int flags[4];  // count, overflow, collision, size
    NNB_CUDA(cudaMemcpyAsync(flags, &ws->count, sizeof(flags), cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaStreamSynchronize(s));
    if (flags[1] || flags[3] > kRowDictMax) {
      if (full) return 0;
      continue;
    }
    rowdict_encode_kernel<<<rows_grid(rows), 256, 0, s>>>(code, width, plane, rows, ws, rcode, &ws->collision);
    count_launch();
    NNB_CUDA(cudaGetLastError());
    NNB_CUDA(cudaMemcpyAsync(flags, &ws->count, sizeof(flags), cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaStreamSynchronize(s));
    if (flags[2]) continue;  // a row outside the sample (or a hash collision): the full round decides
    *npat = flags[3];
    *ok = true;
    return 0;
  }
  return 0;
}

int build_row_dict_direct(const int64_t* rp, const int32_t* col, const double* val, int64_t rows, int64_t row0,
                          int32_t* dict_delta, double* dict_val, int* dict_size, int* width, int* band_lo,
                          int* band_hi, uint8_t* rcode, double2* pat, uint8_t* plen, int* npat, bool* ok,
                          cudaStream_t s, std::vector<double2>* pat_host, std::vector<uint8_t>* plen_host) {
  *ok = false;
  constexpr int64_t kSample = 65536;
  if (rows <= 4 * kSample) return 0;  // small operators: the two-pass build
  DevBuf wsb, rwsb, sample;
  NNB_TRY(wsb.alloc(sizeof(DictWs), s));
  NNB_TRY(rwsb.alloc(sizeof(RowDictWs), s));
  DictWs* ws = wsb.as<DictWs>();
  RowDictWs* rws = rwsb.as<RowDictWs>();
  NNB_CUDA(cudaMemsetAsync(ws, 0, sizeof(DictWs), s));
  NNB_CUDA(cudaMemsetAsync(rws, 0, sizeof(RowDictWs), s));
  // pair table from the first and last kSample rows
  dict_insert_kernel<<<rows_grid(kSample), 256, 0, s>>>(rp, col, val, kSample, row0, ws);
  dict_insert_kernel<<<rows_grid(kSample), 256, 0, s>>>(rp + (rows - kSample), col, val, kSample,
                                                        row0 + rows - kSample, ws);
  dict_index_kernel<<<1, 1024, 0, s>>>(ws, dict_delta, dict_val);
  count_launch(3);
  int f[5];  // count, overflow, collision, size, max_len
  NNB_CUDA(cudaMemcpyAsync(f, &ws->count, sizeof(f), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  const int w = f[4];
  if (f[1] || f[3] > kPairDictMax - 1 || w < 1 || w > kEllMaxWidth) return 0;
  // the sampled rows' ELL codes, then the row table from them
  const int64_t plane = 2 * kSample;
  NNB_TRY(sample.alloc((size_t)w * plane, s));
  uint8_t* sc = sample.as<uint8_t>();
  dict_encode_kernel<<<rows_grid(kSample), 256, 0, s>>>(rp, col, val, kSample, row0, ws, sc, w, plane,
                                                        &ws->collision);
  dict_encode_kernel<<<rows_grid(kSample), 256, 0, s>>>(rp + (rows - kSample), col, val, kSample,
                                                        row0 + rows - kSample, ws, sc + kSample, w, plane,
                                                        &ws->collision);
  rowdict_insert_kernel<<<rows_grid(plane), 256, 0, s>>>(sc, w, plane, plane, rws);
  rowdict_index_kernel<<<1, 1024, 0, s>>>(rws, w, dict_delta, dict_val, pat, plen);
  count_launch(4);
  // every row: pair codes verified, row key looked up, one byte written.  No wait for the
  // sample's verdicts first: a sample collision or an overflowed row table only makes
  // this pass miss (it writes nothing but rcode), and all of them are read below.
  {
    const unsigned grid =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(148 * 8, ((rows + 31) / 32 + kEncWarps - 1) / kEncWarps));
    if (row0 + rows < INT32_MAX)
      rowdict_direct_encode_kernel<true><<<grid, kEncWarps * 32, 0, s>>>(rp, col, val, rows, row0, ws, rws, w, rcode,
                                                                         &rws->collision);
    else
      rowdict_direct_encode_kernel<false><<<grid, kEncWarps * 32, 0, s>>>(rp, col, val, rows, row0, ws, rws, w, rcode,
                                                                          &rws->collision);
  }
  count_launch();
  NNB_CUDA(cudaGetLastError());
  // one round trip: the pair table's and row table's counters, the pair deltas (band)
  // and, if asked for, the row patterns
  const bool want_pat = pat_host && plen_host;
  const size_t off_dd = 64, off_pat = off_dd + sizeof(int32_t) * kPairDictMax;
  const size_t off_len = off_pat + sizeof(double2) * kRowDictMax * w;
  const size_t bytes = want_pat ? off_len + kRowDictMax : off_pat;
  uint8_t* h = static_cast<uint8_t*>(pinned_stage(bytes));
  if (!h) return fail(NNB_ERR_OOM, "sparse: pinned staging buffer");
  NNB_CUDA(cudaMemcpyAsync(h, &ws->count, sizeof(int) * 5, cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaMemcpyAsync(h + 32, &rws->count, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaMemcpyAsync(h + off_dd, dict_delta, sizeof(int32_t) * kPairDictMax, cudaMemcpyDeviceToHost, s));
  if (want_pat) {
    NNB_CUDA(cudaMemcpyAsync(h + off_pat, pat, sizeof(double2) * kRowDictMax * w, cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaMemcpyAsync(h + off_len, plen, kRowDictMax, cudaMemcpyDeviceToHost, s));
  }
  NNB_CUDA(cudaStreamSynchronize(s));
  int rf[4];  // count, overflow, collision, size
  std::memcpy(f, h, sizeof(int) * 5);
  std::memcpy(rf, h + 32, sizeof(rf));
  if (f[1] || f[2] || f[3] > kPairDictMax - 1 || rf[1] || rf[2] || rf[3] > kRowDictMax) return 0;
  const int32_t* dh = reinterpret_cast<const int32_t*>(h + off_dd);
  *band_lo = *band_hi = 0;
  for (int i = 0; i < f[3]; ++i) {
    *band_lo = std::min(*band_lo, dh[i]);
    *band_hi = std::max(*band_hi, dh[i]);
  }
  if (want_pat) {
    const double2* hp = reinterpret_cast<const double2*>(h + off_pat);
    pat_host->assign(hp, hp + (size_t)rf[3] * w);
    plen_host->assign(h + off_len, h + off_len + rf[3]);
  }
  *dict_size = f[3];
  *width = w;
  *npat = rf[3];
  *ok = true;
  return 0;
}

int spmv_csr(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n, const double* X, int64_t k,
             double* Y, cudaStream_t s) {
  if (n == 0) return 0;
  spmv_plain_kernel<<<rows_grid(n), 256, 0, s>>>(row_ptr, col, val, n, k, X, Y);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

namespace {

struct PairDict {
  const uint8_t* code = nullptr;
  const int32_t* delta = nullptr;
  const double* val = nullptr;
  int size = 0;
  int ell_width = 0;
  int64_t ell_rows = 0;  // slot-plane stride
  int band_lo = 0, band_hi = 0;
  const uint8_t* rcode = nullptr;  // row dictionary (over the ELL codes)
  const double2* rpat = nullptr;
  const uint8_t* rlen = nullptr;
  int npat = 0;
};

template <typename Idx>
void run_factors(const Idx* rp, const int32_t* col, const int16_t* col16, const double* val, int64_t n,
                 const double* B, int64_t k, int s_factors, double theta, double* X, double* z[2], double* tb[2],
                 int* flags, cudaStream_t s, const PairDict& dict = PairDict{}) {
  const double* zcur = B;  // Z = B (read in place, never written)
  int zi = 0;
  int64_t reps = 1;
  for (int f = 0; f < s_factors; ++f) {
    const double* tin = zcur;  // t = Z
    int ti = 0;
    for (int64_t r = 0; r < reps; ++r) {
      SpmvOp<Idx> op{rp, col, col16, 0, val, k, tin, tin, nullptr, zcur, theta, flags + f,
                     dict.code, dict.delta, dict.val, dict.size, dict.ell_width, dict.ell_rows, dict.band_lo,
                     dict.band_hi, dict.rcode, dict.rpat, dict.rlen, dict.npat};
      int mode;
      if (r < reps - 1) {
        mode = kInner;
        op.out = tb[ti];
      } else if (f == s_factors - 1) {
        mode = kFinal;
        op.out = X;
      } else {
        mode = kFactorEnd;
        op.out = z[zi];
      }
      spmv_apply(op, mode, 0, n, s);
      if (mode == kInner) {
        tin = tb[ti];
        ti ^= 1;
      } else if (mode == kFactorEnd) {
        zcur = z[zi];
        zi ^= 1;
      }
    }
    reps <<= 1;
  }
}

}  // namespace

int sparse_factorized(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n, const double* B,
                      int64_t k, int s_factors, double theta, double* X, int* fail_factor, cudaStream_t s) {
  const size_t vec = (size_t)n * k;
  int64_t nnz = 0;
  NNB_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  const bool narrow = nnz < INT32_MAX;
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(double) * vec * 4 + sizeof(int) * 64 +
                         (narrow ? sizeof(int32_t) * (n + 1) + sizeof(int16_t) * nnz + 32 : 0),
                     s));
  static const bool dict_on = [] {  // NNB_SPARSE_DICT=0: keep the column format (A/B measurement)
    const char* e = debug_env("NNB_SPARSE_DICT");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  double* z[2] = {work.as<double>(), work.as<double>() + vec};
  double* tb[2] = {z[1] + vec, z[1] + 2 * vec};
  int* flags = reinterpret_cast<int*>(tb[1] + vec);
  NNB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 64, s));
  if (narrow) {
    int32_t* rp32 = flags + 64;
    int16_t* col16 = reinterpret_cast<int16_t*>(rp32 + n + 2);
    static const bool force32 = [] {  // NNB_SPARSE_COL=32: int32 columns (A/B measurement)
      const char* e = debug_env("NNB_SPARSE_COL");
      return e && std::strcmp(e, "32") == 0;
    }();
    // operators with <= 255 distinct (column − row, value) pairs: 1 byte per nonzero
    DevBuf dict_buf, code_buf, rowdict_buf;
    PairDict dict;
    std::vector<double2> pat_host;  // the direct build's row patterns (empty otherwise)
    std::vector<uint8_t> plen_host;
    if (dict_on && !force32) {
      NNB_TRY(dict_buf.alloc((sizeof(int32_t) + sizeof(double)) * kPairDictMax, s));
      double* dv = dict_buf.as<double>();
      int32_t* dd = reinterpret_cast<int32_t*>(dv + kPairDictMax);
      bool ok = false;
      int size = 0, width = 0, lo = 0, hi = 0;
      int64_t plane = 0;
      static const bool rowdict_on = [] {  // NNB_SPARSE_ROWDICT=0: keep the ELL pair codes (A/B measurement)
        const char* e = debug_env("NNB_SPARSE_ROWDICT");
        return !(e && std::strcmp(e, "0") == 0);
      }();
      static const bool direct_on = [] {  // NNB_SPARSE_DIRECT=0: the two-pass row-dictionary build (A/B)
        const char* e = debug_env("NNB_SPARSE_DIRECT");
        return !(e && std::strcmp(e, "0") == 0);
      }();
      const bool want_rows = k == 1 && rowdict_on && n < INT32_MAX / 2;
      if (want_rows) NNB_TRY(rowdict_buf.alloc(sizeof(double2) * kRowDictMax * kEllMaxWidth + kRowDictMax + n, s));
      double2* pat = want_rows ? rowdict_buf.as<double2>() : nullptr;
      uint8_t* plen = want_rows ? reinterpret_cast<uint8_t*>(pat + kRowDictMax * kEllMaxWidth) : nullptr;
      uint8_t* rcode = want_rows ? plen + kRowDictMax : nullptr;
      bool rok = false;
      int npat = 0;
      // stencil-like operators: pair and row tables from sampled rows, then one pass
      // over the CSR writing only the row codes (no ELL pair codes are materialised)
      if (want_rows && direct_on)
        NNB_TRY(build_row_dict_direct(row_ptr, col, val, n, 0, dd, dv, &size, &width, &lo, &hi, rcode, pat, plen,
                                      &npat, &rok, s, &pat_host, &plen_host));
      if (rok) {
        dict = PairDict{nullptr, dd, dv, size, width, 0, lo, hi, rcode, pat, plen, npat};
      } else {
        NNB_TRY(build_pair_dict(row_ptr, col, val, n, 0, nnz, code_buf, &width, &plane, &lo, &hi, dd, dv, &size,
                                &ok, s));
        if (ok) dict = PairDict{code_buf.as<uint8_t>(), dd, dv, size, width, plane, lo, hi};
        // ELL codes with few distinct rows (stencils): one pattern code per row
        if (ok && width && want_rows) {
          NNB_TRY(build_row_dict(dict.code, width, plane, n, dd, dv, rcode, pat, plen, &npat, &rok, s));
          if (rok) {
            dict.rcode = rcode;
            dict.rpat = pat;
            dict.rlen = plen;
            dict.npat = npat;
          }
        }
      }
    }
    // int32 offsets, and int16 column deltas when the operator's band allows (the ELL
    // dictionary needs neither)
    bool fits = false;
    if (!(dict.code && dict.ell_width) && !dict.rcode) NNB_TRY(compact_csr(row_ptr, col, n, 0, rp32, col16, &fits, s));
    fits = fits && !force32;
    // 5-point stencils: temporal blocking, up to 8 applications per pass through HBM
    static const bool tb_on = [] {  // NNB_SPARSE_TB=0: one launch per application (A/B measurement)
      const char* e = debug_env("NNB_SPARSE_TB");
      return !(e && std::strcmp(e, "0") == 0);
    }();
    if (dict.rcode && tb_on && k == 1 && s_factors <= 62) {
      DevBuf table;
      int W = 0, H = 0;
      bool sok = false;
      // with the direct build's host patterns: no round trip before the passes, the edge
      // check's verdict (flags[63]) read with the factors' flags after them
      const bool host_pat = (int)plen_host.size() == dict.npat && dict.npat > 0;
      NNB_TRY(stencil_plan(n, dict.rcode, dict.rpat, dict.rlen, dict.npat, dict.ell_width, table, &W, &H, &sok, s,
                           host_pat ? pat_host.data() : nullptr, host_pat ? plen_host.data() : nullptr,
                           host_pat ? flags + 63 : nullptr));
      if (sok) {
        int64_t moved = 0;
        NNB_TRY(stencil_factors(dict.rcode, table, dict.npat, W, H, B, s_factors, theta, X, z, tb, flags, &moved, s));
        NNB_CUDA(cudaGetLastError());
        int hf[64];
        NNB_CUDA(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
        NNB_CUDA(cudaStreamSynchronize(s));
        if (!hf[63]) {
          set_sparse_bytes_per_nnz(1);
          set_sparse_format("row-dictionary-stencil-tb");
          // per application, averaged over the solve (the bench multiplies by the applications)
          const int64_t apps = (int64_t(1) << s_factors) - 1;
          set_sparse_matrix_bytes(moved / std::max<int64_t>(1, apps) - 2 * n * 8);
          for (int f = 0; f < s_factors && f < 64; ++f)
            if (hf[f]) {
              if (fail_factor) *fail_factor = f;
              return fail(3, "solve_sparse_factorized: non-finite block at factor " + std::to_string(f));
            }
          return 0;
        }
        // a pattern reaches across the grid's edges: not a stencil after all; the passes'
        // results are discarded and the solve runs one launch per application from B
        NNB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 64, s));
      }
    }
    set_sparse_bytes_per_nnz(dict.code || dict.rcode ? 1 : (fits ? 10 : 12));
    set_sparse_format(dict.rcode ? "row-dictionary"
                      : dict.ell_width ? "pair-dictionary-ell"
                      : dict.code ? "pair-dictionary-csr"
                      : fits ? "csr-int16-delta" : "csr-int32");
    // operator bytes one application streams: one code per row (row dictionary), codes
    // (ELL: width·n, no offsets) or values + columns, plus int32 row offsets
    set_sparse_matrix_bytes(dict.rcode ? n
                            : dict.ell_width ? (int64_t)dict.ell_width * n
                                             : nnz * (dict.code ? 1 : (fits ? 10 : 12)) + (n + 1) * 4);
    run_factors<int32_t>(rp32, col, fits ? col16 : nullptr, val, n, B, k, s_factors, theta, X, z, tb, flags, s,
                         dict);
  } else {
    set_sparse_bytes_per_nnz(12);
    set_sparse_format("csr-int64-offsets");
    set_sparse_matrix_bytes(nnz * 12 + (n + 1) * 8);
    run_factors<int64_t>(row_ptr, col, nullptr, val, n, B, k, s_factors, theta, X, z, tb, flags, s);
  }
  NNB_CUDA(cudaGetLastError());
  int hflags[64];
  NNB_CUDA(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  for (int f = 0; f < s_factors && f < 64; ++f)
    if (hflags[f]) {
      if (fail_factor) *fail_factor = f;
      return fail(3, "solve_sparse_factorized: non-finite block at factor " + std::to_string(f));
    }
  return 0;
}

}  // namespace nnb
