// Temporal blocking of the factorized sparse solve for 5-point-stencil operators
// (BASELINE config 4: the 4096² Dirichlet Laplacian + I).
//
// solve_sparse_factorized (proj/src/factorized.cpp:101-140) runs, per factor f,
// 2^f applications t ← t − θ·W·t — 63 for γ = 63.  One launch per application
// streams t in and out of HBM each time (68 µs at 4096², sparse.cu K8).  When the
// row dictionary shows a 5-point stencil — every row pattern's deltas are a subset
// of {−W, −1, 0, +1, +W} in that (CSR) order, rows at x = 0 / W−1 have no −1 / +1
// entry, n = W·H — a block instead loads a 2-D tile of t with an S-cell halo into
// shared memory and runs S applications there (the valid region shrinks by one cell
// per step), writing only the tile's interior: HBM traffic falls ≈S-fold.
//
// Exactness: each row is still computed as the reference does — y summed from 0 in
// CSR order with one rounded multiply and one rounded add per entry, then
// fused_axpy_sub / add / scale exactly as sparse.cu's finish<> — from bitwise the
// same inputs, so x is bit-identical to the reference and to the one-launch kernels
// (tests: array_equal, and the 4096² SHA-256 golden).
//
// Layout: a block owns a TX × TY output tile (112 × 40 at S = 4, 112 × 32 at S = 8); its
// region is (TX + 2S) × (TY + 2S) = 120 × 48 / 128 × 48 cells, two double buffers
// (ping-pong between steps) and one code byte per cell: ≤ 104 KB of shared memory with the
// patterns, filled by cp.async (the whole region in flight at once), two blocks per SM.  Thread (cx, seg) sweeps column cx over a
// 12-row segment with the column's y−1 / y / y+1 values in
// registers (a sliding window), so a cell costs three shared loads (own row below,
// left, right) and one store; a row's pattern (mask + 5 values) is reloaded only
// when its code changes along the sweep.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/nnb.h"
#include "common.cuh"
#include "engine.cuh"
#include "sparse.cuh"

namespace nnb {
namespace {

// Two tile shapes, chosen by the pass depth S (applications per launch): the whole-grid
// solve runs 112 × 40 tiles with a 4-cell halo (a 120 × 48 region, 1.29 region cells per
// output cell: 3.06 ms per C5 solve against 3.15 at 112 × 32 / S = 8, 1.71 cells), the row
// slabs 112 × 32 with an 8-cell halo (128 × 48): half the passes, so half the halo
// exchanges and launches per solve, which the slabs' schedule pays for more than the
// region's extra cells.  Both: 4 column segments of 12 rows, 480 / 512 threads; with the
// pattern table sized to the patterns in use a block needs ≤ 104 KB, so two blocks share an
// SM and one's region loads and barriers overlap the other's steps (128 × 64 tiles at one
// 1008-thread block per SM: 3.30 ms).
constexpr int kTX = 112, kSeg = 4, kMinBlocks = 2;
template <int S>
struct Tile {
  static constexpr int TY = S == 4 ? 40 : 32;
  static constexpr int RX = kTX + 2 * S, RY = TY + 2 * S;
  static constexpr int SegRows = (RY + kSeg - 1) / kSeg;
  static constexpr int Threads = RX * kSeg;
  // two region buffers, the region's codes, then the patterns in use (npat)
  static constexpr int SmemBase = 2 * RX * RY * 8 + (RX * RY + 15) / 16 * 16;
  static constexpr int Smem = SmemBase + kRowDictMax * 48;
  static int smem(int npat) { return SmemBase + npat * 48; }
};
static_assert(Tile<kStencilDepthSolo>::RX % 4 == 0 && Tile<kStencilDepthSlab>::RX % 4 == 0 &&
                  kStencilDepthSolo % 4 == 0 && kStencilDepthSlab % 4 == 0,
              "codes load in 4-byte groups: region x0 and width multiples of 4");

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct StPat {
  double v[5];  // values of the N (−W), W (−1), C (0), E (+1), S (+W) entries present
  int mask;     // bit i: direction i present
  int pad;
};

// One thread's column segment of one step.  UNI: the whole tile is one full 5-point
// pattern (no per-cell code lookups); else each cell's pattern from its code.
template <int S, int MODE, bool UNI>
__device__ __forceinline__ bool sweep(const double* __restrict__ src, double* __restrict__ dst,
                                      const uint8_t* __restrict__ code, const StPat* __restrict__ spat, int uc,
                                      int cx, int ya, int yb, int y0, int gx, int W, double theta, bool last,
                                      double* __restrict__ out) {
  constexpr int kRX = Tile<S>::RX;
  bool bad = false;
  const double* col = src + cx;
  int64_t r = (int64_t)(y0 + ya) * W + gx;  // the cell's global index (last step's output)
  double tN = col[(ya - 1) * kRX], tC = col[ya * kRX];
  int pc = UNI ? uc : -1;
  int mask = 31;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0, v4 = 0.0;
  if (UNI) {
    v0 = spat[uc].v[0];
    v1 = spat[uc].v[1];
    v2 = spat[uc].v[2];
    v3 = spat[uc].v[3];
    v4 = spat[uc].v[4];
  }
  for (int y = ya; y < yb; ++y) {
    const double tS = col[(y + 1) * kRX];
    const double tW = col[y * kRX - 1], tE = col[y * kRX + 1];
    double acc;  // CSR order: −W, −1, 0, +1, +W, from 0
    if (UNI) {
      acc = __dadd_rn(0.0, __dmul_rn(v0, tN));
      acc = __dadd_rn(acc, __dmul_rn(v1, tW));
      acc = __dadd_rn(acc, __dmul_rn(v2, tC));
      acc = __dadd_rn(acc, __dmul_rn(v3, tE));
      acc = __dadd_rn(acc, __dmul_rn(v4, tS));
    } else {
      const int c = code[y * kRX + cx];
      if (c != pc) {
        const StPat& P = spat[c];
        v0 = P.v[0];
        v1 = P.v[1];
        v2 = P.v[2];
        v3 = P.v[3];
        v4 = P.v[4];
        mask = P.mask;
        pc = c;
      }
      acc = 0.0;
      if (mask & 1) acc = __dadd_rn(acc, __dmul_rn(v0, tN));
      if (mask & 2) acc = __dadd_rn(acc, __dmul_rn(v1, tW));
      if (mask & 4) acc = __dadd_rn(acc, __dmul_rn(v2, tC));
      if (mask & 8) acc = __dadd_rn(acc, __dmul_rn(v3, tE));
      if (mask & 16) acc = __dadd_rn(acc, __dmul_rn(v4, tS));
    }
    const double t = __dsub_rn(tC, __dmul_rn(theta, acc));  // fused_axpy_sub, factorized.cpp:21-30
    if (last) {
      // a non-finite value persists in its cell (t keeps its own term) and every cell is
      // some block's interior, so the pass's outputs see it: checking them flags the
      // same factor the reference's per-application check would
      double o = t;
      if (MODE == kFactorEnd) o = __dadd_rn(dst[y * kRX + cx], t);                    // factorized.cpp:136
      else if (MODE == kFinal) o = __dmul_rn(__dadd_rn(dst[y * kRX + cx], t), theta);  // factorized.cpp:139
      bad |= !isfinite(acc) || !isfinite(t) || !isfinite(o);
      out[r] = o;
    } else {
      dst[y * kRX + cx] = t;
    }
    tN = tC;
    tC = tS;
    r += W;
  }
  return bad;
}

template <int S, int MODE>
__global__ void __launch_bounds__(Tile<S>::Threads, kMinBlocks)
    stencil_tb_kernel(const double* __restrict__ tin, const uint8_t* __restrict__ rcode,
                      const double* __restrict__ zold, double* __restrict__ out, const StPat* __restrict__ pats,
                      int npat, int W, int H, int steps, double theta, int* __restrict__ flag, int ty0,
                      int y_off) {
  constexpr int kS = S, kTY = Tile<S>::TY, kRX = Tile<S>::RX, kRY = Tile<S>::RY;
  constexpr int kSegRows = Tile<S>::SegRows, kThreads = Tile<S>::Threads;
  static_assert(kRY % kSeg == 0 && kThreads % (kRX / 4) == 0 && kRY % (kThreads / (kRX / 4)) == 0,
                "region rows split evenly over the load passes");
  extern __shared__ __align__(16) uint8_t sm[];
  double* buf0 = reinterpret_cast<double*>(sm);
  double* buf1 = buf0 + kRX * kRY;
  uint8_t* code = reinterpret_cast<uint8_t*>(buf1 + kRX * kRY);
  StPat* spat = reinterpret_cast<StPat*>(code + (kRX * kRY + 15) / 16 * 16);
  const int x0 = blockIdx.x * kTX - kS, y0 = (blockIdx.y + ty0) * kTY + y_off - kS;
  for (int i = threadIdx.x; i < npat; i += kThreads) spat[i] = pats[i];
  const int cx = threadIdx.x % kRX, seg = threadIdx.x / kRX;
  // the region through cp.async (all of it in flight at once; cells off the grid
  // zero-filled): thread (cx, seg) loads column cx of rows seg, seg + kSeg, …, its
  // address stepped by kSeg grid rows
  {
    const int gx = x0 + cx;
    const bool xin = gx >= 0 && gx < W;
    int64_t off = (int64_t)(y0 + seg) * W + gx;
    const int64_t step = (int64_t)kSeg * W;
#pragma unroll
    for (int j = 0; j < kRY / kSeg; ++j) {
      const int gy = y0 + seg + j * kSeg;
      const bool in = xin && gy >= 0 && gy < H;
      cp_async8(buf0 + (seg + j * kSeg) * kRX + cx, in ? tin + off : tin, in);
      off += step;
    }
  }
  {  // codes in 4-byte groups (W % 4 == 0, x0 % 4 == 0): group g of rows r, r + kCodeRowStep, …
    constexpr int kGroups = kRX / 4, kCodeRowStep = kThreads / kGroups;
    const int g = threadIdx.x % kGroups, r = threadIdx.x / kGroups;
    const int gx = x0 + 4 * g;
    const bool xin = gx >= 0 && gx < W;
    int64_t off = (int64_t)(y0 + r) * W + gx;
#pragma unroll
    for (int j = 0; j < kRY / kCodeRowStep; ++j) {
      const int gy = y0 + r + j * kCodeRowStep;
      const bool in = xin && gy >= 0 && gy < H;
      cp_async4(code + (r + j * kCodeRowStep) * kRX + 4 * g, in ? rcode + off : rcode, in);
      off += (int64_t)kCodeRowStep * W;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  // a tile whose whole region is one full 5-point pattern (all but the grid's edge
  // tiles) skips the per-cell code lookups
  const int uc = code[0];
  bool uniform = spat[uc].mask == 31 && x0 >= 0 && y0 >= 0 && x0 + kRX <= W && y0 + kRY <= H;
  const uint32_t uc4 = 0x01010101u * (uint32_t)uc;
  for (int i = threadIdx.x; i < kRX * kRY / 4 && uniform; i += kThreads)
    uniform = reinterpret_cast<const uint32_t*>(code)[i] == uc4;
  uniform = __syncthreads_and(uniform);
  const int gx = x0 + cx;
  const bool col_in = gx >= 0 && gx < W;
  bool bad = false;
  for (int s = 1; s <= steps; ++s) {
    const double* src = (s & 1) ? buf0 : buf1;
    double* dst = (s & 1) ? buf1 : buf0;
    const int m = steps - s;  // cells still needed beyond the interior after this step
    const int xlo = kS - m, xhi = kS + kTX + m, ylo = kS - m, yhi = kS + kTY + m;
    const bool last = s == steps;
    if (last && MODE != kInner) {  // Z of the interior into the free buffer, one wait per pass
      static_assert(kTY % kSeg == 0, "interior rows split evenly over the segments");
      if (cx >= kS && cx < kS + kTX) {  // column cx of interior rows kS + seg, kS + seg + kSeg, …
        const bool xin = gx < W;
        int64_t off = (int64_t)(y0 + kS + seg) * W + gx;
#pragma unroll
        for (int j = 0; j < kTY / kSeg; ++j) {
          const int ry = kS + seg + j * kSeg;
          const bool in = xin && y0 + ry < H;
          cp_async8(dst + ry * kRX + cx, in ? zold + off : zold, in);
          off += (int64_t)kSeg * W;
        }
      }
      cp_async_wait_all();
      __syncthreads();
    }
    if (cx >= xlo && cx < xhi && col_in) {
      // this thread's rows of the step, clipped to the grid (rows off it are never read)
      const int ya = max(max(seg * kSegRows, ylo), -y0);
      const int yb = min(min(min(seg * kSegRows + kSegRows, kRY), yhi), H - y0);
      if (ya < yb) {
        if (uniform) bad |= sweep<S, MODE, true>(src, dst, code, spat, uc, cx, ya, yb, y0, gx, W, theta, last, out);
        else bad |= sweep<S, MODE, false>(src, dst, code, spat, uc, cx, ya, yb, y0, gx, W, theta, last, out);
      }
    }
    if (!last) __syncthreads();
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// rows on the grid's edges whose pattern reaches across it (x wrap or out of range)
// (a row slab checks its top / bottom rows only where they are the grid's: check_top/bottom)
__global__ void stencil_edge_check(const uint8_t* __restrict__ rcode, const StPat* __restrict__ pats, int W, int H,
                                   int* __restrict__ bad, int check_top, int check_bottom) {
  const int64_t per = 2LL * W + 2LL * H;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x) {
    int x, y, forbid;
    if (i < W) { x = (int)i; y = 0; forbid = check_top ? 1 : 0; }                        // top row: no −W
    else if (i < 2LL * W) { x = (int)(i - W); y = H - 1; forbid = check_bottom ? 16 : 0; }  // bottom row: no +W
    else if (i < 2LL * W + H) { x = 0; y = (int)(i - 2LL * W); forbid = 2; }  // left column: no −1
    else { x = W - 1; y = (int)(i - 2LL * W - H); forbid = 8; }          // right column: no +1
    const int m = pats[rcode[(int64_t)y * W + x]].mask;
    if (m & forbid) atomicOr(bad, 1);
  }
}

}  // namespace

int stencil_patterns_host(const double2* hp, const uint8_t* hl, int npat, int width, int64_t* W_out,
                          std::vector<StencilPattern>& tab) {
  static_assert(sizeof(StencilPattern) == sizeof(StPat), "host and device pattern layouts");
  *W_out = 0;
  tab.clear();
  if (npat < 1 || npat > kRowDictMax || width < 1 || width > kEllMaxWidth) return 0;
  int64_t w = 0;
  for (int p = 0; p < npat; ++p)
    for (int i = 0; i < hl[p]; ++i) {
      int64_t d;
      std::memcpy(&d, &hp[(size_t)p * width + i].y, 8);
      if (d != 0 && d != 1 && d != -1) {
        if (w && std::llabs(d) != w) return 0;
        w = std::llabs(d);
      }
    }
  if (w < 4 || w % 4 != 0 || w > INT32_MAX) return 0;
  std::vector<StencilPattern> t(npat);
  for (int p = 0; p < npat; ++p) {
    StencilPattern sp{};
    int last_dir = -1;
    for (int i = 0; i < hl[p]; ++i) {
      int64_t d;
      std::memcpy(&d, &hp[(size_t)p * width + i].y, 8);
      const int dir = d == -w ? 0 : d == -1 ? 1 : d == 0 ? 2 : d == 1 ? 3 : 4;
      if (dir <= last_dir) return 0;  // repeated or out-of-order entries: not the CSR order assumed
      last_dir = dir;
      sp.v[dir] = hp[(size_t)p * width + i].x;
      sp.mask |= 1 << dir;
    }
    t[p] = sp;
  }
  tab.swap(t);
  *W_out = w;
  return 0;
}

int stencil_patterns(const double2* pat, const uint8_t* plen, int npat, int width, int64_t* W_out,
                     std::vector<StencilPattern>& tab, cudaStream_t s) {
  *W_out = 0;
  tab.clear();
  if (npat < 1 || npat > kRowDictMax || width < 1 || width > kEllMaxWidth) return 0;
  std::vector<double2> hp((size_t)npat * width);
  std::vector<uint8_t> hl(npat);
  NNB_CUDA(cudaMemcpyAsync(hp.data(), pat, sizeof(double2) * hp.size(), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaMemcpyAsync(hl.data(), plen, npat, cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  return stencil_patterns_host(hp.data(), hl.data(), npat, width, W_out, tab);
}

int stencil_edges_ok(const uint8_t* rcode, const StencilPattern* table_dev, int W, int H, bool top, bool bottom,
                     bool* ok, cudaStream_t s) {
  DevBuf b;
  NNB_TRY(b.alloc(sizeof(int), s));
  NNB_CUDA(cudaMemsetAsync(b.p, 0, sizeof(int), s));
  stencil_edge_check<<<148, 256, 0, s>>>(rcode, reinterpret_cast<const StPat*>(table_dev), W, H, b.as<int>(),
                                         top ? 1 : 0, bottom ? 1 : 0);
  count_launch();
  int hbad = 1;
  NNB_CUDA(cudaMemcpyAsync(&hbad, b.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  *ok = hbad == 0;
  return 0;
}

namespace {
// the device pattern table from the row dictionary's patterns (the host checked them)
__global__ void stencil_table_kernel(const double2* __restrict__ pat, const uint8_t* __restrict__ plen, int npat,
                                     int width, long long W, StPat* __restrict__ tab) {
  for (int p = threadIdx.x; p < npat; p += blockDim.x) {
    StPat sp{};
    for (int i = 0; i < plen[p]; ++i) {
      const long long d = __double_as_longlong(pat[(size_t)p * width + i].y);
      const int dir = d == -W ? 0 : d == -1 ? 1 : d == 0 ? 2 : d == 1 ? 3 : 4;
      sp.v[dir] = pat[(size_t)p * width + i].x;
      sp.mask |= 1 << dir;
    }
    tab[p] = sp;
  }
}
}  // namespace

int stencil_plan(int64_t n, const uint8_t* rcode, const double2* pat, const uint8_t* plen, int npat, int width,
                 DevBuf& table, int* W_out, int* H_out, bool* ok, cudaStream_t s, const double2* pat_host,
                 const uint8_t* plen_host, int* edge_bad_dev) {
  *ok = false;
  if (n < 4) return 0;
  int64_t w = 0;
  std::vector<StencilPattern> tab;
  if (pat_host && plen_host) NNB_TRY(stencil_patterns_host(pat_host, plen_host, npat, width, &w, tab));
  else NNB_TRY(stencil_patterns(pat, plen, npat, width, &w, tab, s));
  if (!w || n % w != 0 || n / w > INT32_MAX) return 0;
  NNB_TRY(table.alloc(sizeof(StPat) * npat, s));
  const int W = (int)w, H = (int)(n / w);
  if (pat_host && plen_host) {  // built on the device: no host round trip
    stencil_table_kernel<<<1, 256, 0, s>>>(pat, plen, npat, width, w, table.as<StPat>());
    count_launch();
  } else {
    NNB_CUDA(cudaMemcpyAsync(table.p, tab.data(), sizeof(StPat) * npat, cudaMemcpyHostToDevice, s));
  }
  if (edge_bad_dev) {  // the caller reads the edge verdict with its own results
    stencil_edge_check<<<148, 256, 0, s>>>(rcode, table.as<StPat>(), W, H, edge_bad_dev, 1, 1);
    count_launch();
    NNB_CUDA(cudaGetLastError());
  } else {
    bool eok = false;
    NNB_TRY(stencil_edges_ok(rcode, table.as<StencilPattern>(), W, H, true, true, &eok, s));
    if (!eok) return 0;
  }
  *W_out = W;
  *H_out = H;
  *ok = true;
  return 0;
}

int stencil_tile_rows(int depth) { return depth == kStencilDepthSlab ? Tile<kStencilDepthSlab>::TY : Tile<kStencilDepthSolo>::TY; }

namespace {
template <int S>
int pass_launch(const double* tin, const uint8_t* rcode, const double* zold, double* out, const StPat* pats, int npat,
                int W, int H, int steps, int mode, double theta, int* flag, cudaStream_t s, int ty0, int ty1,
                int y_off, int out_rows) {
  using T = Tile<S>;
  NNB_TRY((ensure_smem<stencil_tb_kernel<S, kInner>>(T::Smem)));
  NNB_TRY((ensure_smem<stencil_tb_kernel<S, kFactorEnd>>(T::Smem)));
  NNB_TRY((ensure_smem<stencil_tb_kernel<S, kFinal>>(T::Smem)));
  const int tiles_y = ((out_rows < 0 ? H : out_rows) + T::TY - 1) / T::TY;
  if (ty1 < 0 || ty1 > tiles_y) ty1 = tiles_y;
  if (ty0 >= ty1) return 0;
  const dim3 grid((unsigned)((W + kTX - 1) / kTX), (unsigned)(ty1 - ty0));
  const int sm = T::smem(npat);
  switch (mode) {
    case kInner:
      stencil_tb_kernel<S, kInner><<<grid, T::Threads, sm, s>>>(tin, rcode, zold, out, pats, npat, W, H, steps, theta,
                                                                flag, ty0, y_off);
      break;
    case kFactorEnd:
      stencil_tb_kernel<S, kFactorEnd><<<grid, T::Threads, sm, s>>>(tin, rcode, zold, out, pats, npat, W, H, steps,
                                                                    theta, flag, ty0, y_off);
      break;
    default:
      stencil_tb_kernel<S, kFinal><<<grid, T::Threads, sm, s>>>(tin, rcode, zold, out, pats, npat, W, H, steps, theta,
                                                                flag, ty0, y_off);
  }
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}
}  // namespace

int stencil_pass(const double* tin, const uint8_t* rcode, const double* zold, double* out,
                 const StencilPattern* table_dev, int npat, int W, int H, int steps, int mode, double theta, int* flag,
                 int depth, cudaStream_t s, int ty0, int ty1, int y_off, int out_rows) {
  const StPat* pats = reinterpret_cast<const StPat*>(table_dev);
  if (depth == kStencilDepthSlab) {
    if (steps < 1 || steps > kStencilDepthSlab) return fail(NNB_ERR_DOMAIN, "stencil pass: steps outside 1..8");
    return pass_launch<kStencilDepthSlab>(tin, rcode, zold, out, pats, npat, W, H, steps, mode, theta, flag, s, ty0,
                                          ty1, y_off, out_rows);
  }
  if (depth != kStencilDepthSolo || steps < 1 || steps > kStencilDepthSolo)
    return fail(NNB_ERR_DOMAIN, "stencil pass: depth not 4 / 8 or steps beyond it");
  return pass_launch<kStencilDepthSolo>(tin, rcode, zold, out, pats, npat, W, H, steps, mode, theta, flag, s, ty0,
                                        ty1, y_off, out_rows);
}

double stencil_region_ratio(int depth) {
  const int S = depth == kStencilDepthSlab ? kStencilDepthSlab : kStencilDepthSolo;
  const int TY = stencil_tile_rows(depth);
  return (double)(kTX + 2 * S) * (TY + 2 * S) / ((double)kTX * TY);
}

int stencil_factors(const uint8_t* rcode, const DevBuf& table, int npat, int W, int H, const double* B,
                    int s_factors, double theta, double* X, double* z[2], double* tb[2], int* flags,
                    int64_t* bytes_moved, cudaStream_t s) {
  int depth = kStencilDepthSolo;
  if (const char* e = debug_env("NNB_STENCIL_DEPTH")) depth = std::atoi(e) == 8 ? 8 : 4;  // A/B only
  const double n = (double)W * H;
  const double halo = stencil_region_ratio(depth);  // region cells read per output cell
  double moved = 0.0;
  const double* zcur = B;
  int zi = 0;
  for (int f = 0; f < s_factors; ++f) {
    int64_t left = int64_t(1) << f;
    const double* tin = zcur;
    int ti = 0;
    while (left > 0) {
      const int steps = (int)std::min<int64_t>(depth, left);
      left -= steps;
      const int mode = left > 0 ? kInner : (f == s_factors - 1 ? kFinal : kFactorEnd);
      double* out = mode == kInner ? tb[ti] : (mode == kFinal ? X : z[zi]);
      NNB_TRY(stencil_pass(tin, rcode, zcur, out, table.as<StencilPattern>(), npat, W, H, steps, mode, theta,
                           flags + f, depth, s));
      moved += n * (halo * (8.0 + 1.0) + 8.0 + (mode == kInner ? 0.0 : 8.0));
      if (mode == kInner) {
        tin = tb[ti];
        ti ^= 1;
      } else if (mode == kFactorEnd) {
        zcur = z[zi];
        zi ^= 1;
      }
    }
  }
  if (bytes_moved) *bytes_moved = (int64_t)moved;
  return 0;
}

}  // namespace nnb
