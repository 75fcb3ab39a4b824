// Shared pieces of the single-GPU and row-sharded sparse factorized solves.
#pragma once

#include <vector>

#include <cstdint>

#include <cuda_runtime.h>

namespace nnb {

enum SpmvMode { kInner = 0, kFactorEnd = 1, kFinal = 2 };

// One application t_out = t_in − θ·W·t_in (+ factor update / final scale by mode).
// Columns come either as int32 indices into t_ext (`col`) or, when every
// |column − row| ≤ 32767 (banded operators such as the C5 Laplacian), as
// int16 deltas from the row's own global index (`col16`; gather index =
// r + diag_off + delta): 10 instead of 12 bytes per nonzero, same CSR order.
template <typename Idx>
struct SpmvOp {
  const Idx* rp;        // row offsets of the rows this call owns (local, from 0)
  const int32_t* col;   // column indices into t_ext (when col16 is null)
  const int16_t* col16; // column − global row (when not null)
  int64_t diag_off;     // gather index of owned row 0 (the halo width when sharded)
  const double* val;
  int64_t k;            // right-hand sides
  const double* t_ext;  // gather base (own rows, plus halo rows around them when sharded)
  const double* t_own;  // t_in indexed by owned row
  double* out;          // indexed by owned row
  const double* zold;   // indexed by owned row (factor end / final)
  double theta;
  int* flag;            // non-finite flag of this factor
  // Pair dictionary (CSR-VI style, when the operator has <= 256 distinct
  // (column − row, value) pairs, e.g. stencils): one uint8 code per nonzero
  // replaces column and value.  Lookups are exact, so sums stay bit-identical.
  const uint8_t* code = nullptr;
  const int32_t* dict_delta = nullptr;
  const double* dict_val = nullptr;
  int dict_size = 0;
  int ell_width = 0;  // > 0: slot-major ELL codes (code[i·ell_rows + r], kEllPad-padded), no row offsets
  int64_t ell_rows = 0;  // slot-plane stride (rows rounded up to 16)
  int band_lo = 0, band_hi = 0;  // min / max (column − row) over the dictionary
  // Row dictionary (over the ELL pair codes, <= kRowDictMax distinct rows): one
  // uint8 pattern code per row; rpat[p·ell_width + i] = {value, delta as bits}
  const uint8_t* rcode = nullptr;
  const double2* rpat = nullptr;
  const uint8_t* rlen = nullptr;
  int npat = 0;
};

constexpr int kPairDictMax = 256;
constexpr int kEllMaxWidth = 8;     // rows this short store their codes in ELL order
constexpr uint8_t kEllPad = 255;    // ELL padding code (the dictionary keeps it free)
constexpr int kRowDictMax = 256;    // row patterns (uint8 row codes)

// Bytes per nonzero of the format the last single-GPU sparse solve on this thread
// consumed (1 = pair dictionary, 10 = int16 column deltas, 12 = int32 columns).
void set_sparse_bytes_per_nnz(int b);
int sparse_bytes_per_nnz();
// Operator bytes (codes or values + columns, plus row offsets) one application of that solve streams.
void set_sparse_matrix_bytes(int64_t b);
// Name of that format: "row-dictionary", "pair-dictionary-ell", "pair-dictionary-csr",
// "csr-int16-delta", "csr-int32", "csr-int64-offsets" ("" before any solve).
void set_sparse_format(const char* f);
const char* sparse_format();
int64_t sparse_matrix_bytes();

// Builds the pair dictionary of rows [0, rows) (global row index row0 + r; nonzeros
// rp[r]..rp[r+1]) and allocates + fills code_buf: ELL order (*ell_width > 0) when
// every row has at most kEllMaxWidth nonzeros and padding adds at most 25 %, else
// CSR order (code[e − rp[0]]).  *ok = false when the operator has more than
// kPairDictMax − 1 distinct pairs; the caller keeps its column format then.
struct DevBuf;
int build_pair_dict(const int64_t* rp, const int32_t* col, const double* val, int64_t rows, int64_t row0,
                    int64_t nnz, DevBuf& code_buf, int* ell_width, int64_t* ell_plane, int* band_lo, int* band_hi,
                    int32_t* dict_delta, double* dict_val, int* dict_size, bool* ok, cudaStream_t s);

// Row dictionary over ELL pair codes (code, width, plane from build_pair_dict):
// fills rcode[rows], pat[npat·width] ({value, delta as bits}) and plen[npat];
// *ok = false when the operator has more than kRowDictMax distinct rows.
int build_row_dict(const uint8_t* code, int width, int64_t plane, int64_t rows, const int32_t* dict_delta,
                   const double* dict_val, uint8_t* rcode, double2* pat, uint8_t* plen, int* npat, bool* ok,
                   cudaStream_t s);

// Both tables from the first and last 65536 rows, then one verified pass over the
// CSR writing only the row codes (operators above 4·65536 rows; *ok = false on any
// miss, the caller then takes build_pair_dict + build_row_dict).  Two host round
// trips: the sample's width, then every verdict (and, when pat_host / plen_host are
// given, host copies of the row patterns) in one pinned copy.
int build_row_dict_direct(const int64_t* rp, const int32_t* col, const double* val, int64_t rows, int64_t row0,
                          int32_t* dict_delta, double* dict_val, int* dict_size, int* width, int* band_lo,
                          int* band_hi, uint8_t* rcode, double2* pat, uint8_t* plen, int* npat, bool* ok,
                          cudaStream_t s, std::vector<double2>* pat_host = nullptr,
                          std::vector<uint8_t>* plen_host = nullptr);

template <typename Idx>
void spmv_apply(const SpmvOp<Idx>& op, int mode, int64_t r_begin, int64_t r_end, cudaStream_t s);

int narrow_offsets(const int64_t* in, int32_t* out, int64_t count, int64_t base, cudaStream_t s);

// Temporal blocking for 5-point-stencil operators (sparse_stencil.cu): from the row
// dictionary, *ok when every pattern is a CSR-ordered subset of {−W, −1, 0, +1, +W}
// for one W with n = W·H and no pattern reaches across the grid's edges; `table`
// then holds the device pattern table.
// With host copies of the patterns (pat_host / plen_host) the table is built on the device
// without a round trip; with edge_bad_dev the edge check only sets that device flag (no
// wait) and *ok covers the patterns alone — the caller discards the passes if it is set.
int stencil_plan(int64_t n, const uint8_t* rcode, const double2* pat, const uint8_t* plen, int npat, int width,
                 DevBuf& table, int* W, int* H, bool* ok, cudaStream_t s, const double2* pat_host = nullptr,
                 const uint8_t* plen_host = nullptr, int* edge_bad_dev = nullptr);
// a row pattern of the stencil table (device layout): values of the N, W, C, E, S entries
struct StencilPattern {
  double v[5];
  int mask;
  int pad;
};
// the pieces of stencil_plan, for row slabs (sparse_sharded.cu): the host pattern table and W
// from a row dictionary (*W = 0 when it is not a 5-point stencil), and the edge check of an
// H-row grid of codes (top / bottom rows checked only where they are the grid's)
int stencil_patterns(const double2* pat, const uint8_t* plen, int npat, int width, int64_t* W,
                     std::vector<StencilPattern>& tab, cudaStream_t s);
int stencil_patterns_host(const double2* pat, const uint8_t* plen, int npat, int width, int64_t* W,
                          std::vector<StencilPattern>& tab);
int stencil_edges_ok(const uint8_t* rcode, const StencilPattern* table_dev, int W, int H, bool top, bool bottom,
                     bool* ok, cudaStream_t s);
// Pass depths (most applications per launch): the whole-grid solve's, and the row slabs'
// (fewer passes, so fewer halo exchanges; a slab's halo is kStencilDepthSlab grid rows)
constexpr int kStencilDepthSolo = 4, kStencilDepthSlab = 8;
// one temporal-blocked pass: `steps` (<= depth) applications over a W×H grid, in the tile
// shape of that depth.  Output tile rows [ty0, ty1) only (ty1 < 0: to the last) of the
// out_rows rows from row y_off (out_rows < 0: all H); the grid's other rows are inputs only
// (a slab's halo rows).
int stencil_pass(const double* tin, const uint8_t* rcode, const double* zold, double* out,
                 const StencilPattern* table_dev, int npat, int W, int H, int steps, int mode, double theta, int* flag,
                 int depth, cudaStream_t s, int ty0 = 0, int ty1 = -1, int y_off = 0, int out_rows = -1);
int stencil_tile_rows(int depth);
double stencil_region_ratio(int depth);
// The whole factorized solve (one RHS) in passes of up to 4 applications per launch;
// bit-identical to run_factors.  *bytes_moved: HBM bytes the passes stream.
int stencil_factors(const uint8_t* rcode, const DevBuf& table, int npat, int W, int H, const double* B,
                    int s_factors, double theta, double* X, double* z[2], double* tb[2], int* flags,
                    int64_t* bytes_moved, cudaStream_t s);

// rp32[r] = rp[r] − rp[0] and col16[e] = col[e] − (row0 + r) for `rows` rows
// (col indexed by rp).  Returns 0 and sets *fits = false when some delta does
// not fit in int16 (col16 is then garbage; use int32 columns).
int compact_csr(const int64_t* rp, const int32_t* col, int64_t rows, int64_t row0, int32_t* rp32, int16_t* col16,
                bool* fits, cudaStream_t s);

}  // namespace nnb
