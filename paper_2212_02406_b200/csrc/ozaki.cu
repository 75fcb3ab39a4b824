// FP64 products emulated on the int8 tensor cores (tcgen05.mma kind::i8):
// the Ozaki scheme II, NNB_ARITH_OZAKI.  sm_100a has no FP64 tcgen05 kind, and
// its DMMA pipe peaks at 37 TFLOP/s; the int8 pipe runs ~120x faster, so an
// FP64 product that costs s int8 GEMMs (s = 16 moduli) plus O(N^2) passes
// beats DMMA by several times at large N.  Every product of the chain
// (proj/src/kernels.cpp:137-162, the reference's nn::matmul) goes through it
// when the mode is on; the chain logic, its epilogue contract (α·A·B + β·D +
// γ·I, deterministic Σ C², non-finite count) and its stop rules are unchanged.
//
// The scheme, for C = A·B with A m×k and B k×n:
//   1. Scale.  Row i of A by 2^ea_i and column j of B by 2^eb_j so that the
//      largest magnitude of each lands in [2^52, 2^53); round to integers
//      A' = rint(2^ea·A), B' = rint(B·2^eb) (|A'|, |B'| <= 2^53).  This is the
//      only rounding of the scheme: each entry keeps its bits down to 2^-53
//      of its row's (column's) largest entry.
//   2. Residues.  For pairwise coprime moduli m_1..m_s <= 256 (M = Πm_l),
//      A'_l = A' mod m_l and B'_l = B' mod m_l as signed int8 (symmetric).
//   3. s int8 GEMMs on tcgen05: C_l = A'_l·B'_lᵀ accumulates exactly in int32
//      (|A'_l|,|B'_l| <= 128, k < 2^17), stored as C_l mod m_l (uint8).
//   4. Reconstruction.  The CRT sum C' = Σ_l r_l·W_l − q·M over the s residues in
//      FP64 with the weights split so the large terms cancel exactly (k·2^106 < M/8,
//      so the nearest multiple of M is the one to remove), rounded once; the scaling
//      back by 2^-(ea_i+eb_j), and the chain's epilogue.
// The integer product A'·B' is exact, so the error is step 1's truncation
// only: |C − fl(C)| <= 2^-53·k·max_i|a_i·|·max_j|b_·j| per element, the same
// order as a DGEMM's u·k·|a||b| bound.  Parity against the reference is
// therefore the same gate as the DMMA path: X within 1e-10 and identical nest
// counts (tests/test_gpu_ozaki.py).
//
// The int8 GEMM (oz_gemm_kernel): one CTA per 128×256 output tile and modulus,
// warp-specialised — warp 0 lane 0 drives a 4-stage TMA ring (A 128×128 B,
// B 256×128 B, 128B swizzle, K-major), warp 1 lane 0 issues tcgen05.mma
// (M=128, N=256, K=32 per instruction) into a 256-column TMEM accumulator and
// frees each stage with tcgen05.commit, warps 2-5 drain TMEM (tcgen05.ld
// 32x32b), reduce mod m_l and store uint8 residues.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "engine.cuh"

namespace nnb {
namespace {

constexpr int kMaxMod = 20;
constexpr int kModuli[kMaxMod] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227,
                                  223, 217, 211, 199, 197, 193, 191, 181, 179, 173};
constexpr int kAlpha = 53;                  // bits kept per row (column) of an operand
constexpr int kBadExp = INT_MIN / 4;        // exponent marking a row/column with a non-finite entry
constexpr int64_t kMaxK = 131071;           // 128·128·k < 2^31: exact int32 accumulation
constexpr int kColRows = 64;                // rows per block of the column-statistics passes

// Moduli constants for the first s moduli (host-computed, passed by value).
struct OzConst {
  int s;
  int mi[kMaxMod];
  unsigned magic[kMaxMod];   // floor(2^32 / m): the epilogue's integer reduction mod m
  unsigned offset[kMaxMod];  // m·ceil(2^31 / m): a + offset >= 0 for every int32 accumulator a
  // CRT weights of the residue pairs (moduli p_i = m_2i·m_2i+1; the last alone for odd s):
  // W_i = (M/p_i)·((M/p_i)^-1 mod p_i) < M split at 2^e (e = bits(M) − 34) into
  // pwhi = floor(W_i / 2^e)·2^e (exact, < 2^34 units of 2^e) and pwlo = W_i mod 2^e
  // (rounded); the same split of M, and 1/M for the quotient
  double pwhi[kMaxMod / 2 + 1];
  double pwlo[kMaxMod / 2 + 1];
  double pmhi, pmlo, inv_m;
};

// The moduli at compile time (template parameters -> immediates in the split kernels).
constexpr int kMod(int j) {
  return j == 0 ? 256 : j == 1 ? 255 : j == 2 ? 253 : j == 3 ? 251 : j == 4 ? 247 : j == 5 ? 241 : j == 6 ? 239
       : j == 7 ? 233 : j == 8 ? 229 : j == 9 ? 227 : j == 10 ? 223 : j == 11 ? 217 : j == 12 ? 211
       : j == 13 ? 199 : j == 14 ? 197 : j == 15 ? 193 : j == 16 ? 191 : j == 17 ? 181 : j == 18 ? 179 : 173;
}
// Packed FP32 (FFMA2/FADD2/FMUL2 on sm_100a; constants become broadcast immediates):
// two entries per instruction in the residue splits, which are issue-bound.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long bc2(float c) { return pk2(c, c); }
int inv_mod(int a, int m) {
  a %= m;
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return 0;
}

// Little-endian base-2^32 integers, just wide enough for M = Π m_l (< 2^173) and the
// CRT weights (host only).
struct BigU {
  uint32_t w[6] = {0, 0, 0, 0, 0, 0};
};
BigU big_mul(const BigU& a, uint32_t m) {
  BigU r;
  uint64_t c = 0;
  for (int i = 0; i < 6; ++i) {
    const uint64_t t = static_cast<uint64_t>(a.w[i]) * m + c;
    r.w[i] = static_cast<uint32_t>(t);
    c = t >> 32;
  }
  return r;
}
BigU big_div(const BigU& a, uint32_t m) {  // exact quotient (m divides a)
  BigU r;
  uint64_t rem = 0;
  for (int i = 5; i >= 0; --i) {
    const uint64_t t = (rem << 32) | a.w[i];
    r.w[i] = static_cast<uint32_t>(t / m);
    rem = t % m;
  }
  return r;
}
int big_bits(const BigU& a) {
  for (int i = 5; i >= 0; --i)
    if (a.w[i]) return 32 * i + 32 - __builtin_clz(a.w[i]);
  return 0;
}
bool big_bit(const BigU& a, int i) { return i >= 0 && i < 192 && ((a.w[i >> 5] >> (i & 31)) & 1u); }
// Σ_{lo <= i < hi} bit_i·2^i as a double (exact when hi − lo <= 53, else rounded once per
// 53-bit window from the top)
double big_range(const BigU& a, int lo, int hi) {
  double v = 0.0;
  for (int top = hi; top > lo; top -= 53) {
    const int b0 = std::max(lo, top - 53);
    uint64_t u = 0;
    for (int i = top - 1; i >= b0; --i) u = (u << 1) | (big_bit(a, i) ? 1u : 0u);
    v += std::ldexp(static_cast<double>(u), b0);
  }
  return v;
}

OzConst make_const(int s) {
  OzConst c{};
  c.s = s;
  BigU M;
  M.w[0] = 1;
  for (int j = 0; j < s; ++j) {
    const int m = kModuli[j];
    c.mi[j] = m;
    c.magic[j] = static_cast<unsigned>((1ull << 32) / static_cast<unsigned long long>(m));
    c.offset[j] = static_cast<unsigned>(static_cast<unsigned long long>(m) * (((1ull << 31) + m - 1) / m));
    M = big_mul(M, static_cast<uint32_t>(m));
  }
  // e: Σ_i u_i·pwhi_i (|u_i| < 2^15.1, <= 10 terms, pwhi < 2^34 units) and q·pmhi (q < 2^18.5)
  // stay below 2^53 units of 2^e, so both are exact in FP64
  const int B = big_bits(M);
  c.inv_m = 1.0 / big_range(M, 0, B);
  const int e2 = B - 34;  // e
  for (int i = 0; 2 * i < s; ++i) {
    const int64_t mod = 2 * i + 1 < s ? static_cast<int64_t>(kModuli[2 * i]) * kModuli[2 * i + 1] : kModuli[2 * i];
    const BigU Mj = big_div(M, static_cast<uint32_t>(mod));
    int64_t mj_mod = 0;
    for (int k = 5; k >= 0; --k) mj_mod = static_cast<int64_t>(((static_cast<uint64_t>(mj_mod) << 32) | Mj.w[k]) % mod);
    int64_t inv = 0;  // (M/mod)^-1 mod mod by extended Euclid
    {
      int64_t r0 = mod, r1 = mj_mod, t0 = 0, t1 = 1;
      while (r1) {
        const int64_t qq = r0 / r1;
        std::tie(r0, r1) = std::make_tuple(r1, r0 - qq * r1);
        std::tie(t0, t1) = std::make_tuple(t1, t0 - qq * t1);
      }
      inv = (t0 % mod + mod) % mod;
    }
    const BigU W = big_mul(Mj, static_cast<uint32_t>(inv));  // < M
    c.pwhi[i] = big_range(W, e2, B);
    c.pwlo[i] = big_range(W, 0, e2);
  }
  c.pmhi = big_range(M, e2, B);
  c.pmlo = big_range(M, 0, e2);
  return c;
}

// moduli needed so that k·2^(2·53) < M/8 (exact, sign decided by the top digit)
int moduli_for(int64_t k) {
  const double need = 2.0 * kAlpha + std::ceil(std::log2(static_cast<double>(std::max<int64_t>(k, 2)))) + 3.0;
  double have = 0.0;
  for (int s = 0; s < kMaxMod; ++s) {
    have += std::log2(static_cast<double>(kModuli[s]));
    if (have >= need) return s + 1;
  }
  return kMaxMod;
}

// ---------------------------------------------------------------- tcgen05 wrappers
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` once every tcgen05.mma this thread issued so far has completed
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 lanes × 32 consecutive 32-bit TMEM columns -> 32 registers per thread (row = lane)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// K-major operand tile, 128B swizzle (rows of 128 bytes, 8-row groups 1024 B apart):
// start address >> 4, LBO 1 (unused for swizzled K-major), SBO 1024 B, version 1, SWIZZLE_128B
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// ---------------------------------------------------------------- the int8 GEMM
constexpr int kBM = 128, kBN = 256, kBK = 128, kStages = 4;
constexpr int kABytes = kBM * kBK;  // 16 KB
constexpr int kBBytes = kBN * kBK;  // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kGemmSmem = kStages * kStageBytes + 1024 + 256;
constexpr uint32_t kIdesc = (2u << 4) |            // D: s32
                            (1u << 7) | (1u << 10) |  // A, B: signed int8
                            ((uint32_t)(kBN >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);  // K-major both

constexpr int kAccBufs = 2;    // TMEM accumulators: 2 × 256 columns (the whole 512)
constexpr int kEpiWarps = 4;
constexpr int kGroupM = 16;    // rasterisation: 16 tile-rows per group (measured best of 4..32: DRAM 72 vs 106 GB at N=16384 for 8)

struct TileCoord {
  int l, mt, nt;
};
__device__ __forceinline__ TileCoord tile_of(int t, int tiles_m, int tiles_n, int group_m = kGroupM) {
  // group_m tile-rows per group; each group is walked column by column
  const int per = tiles_m * tiles_n;
  TileCoord c;
  c.l = t / per;
  const int r = t - c.l * per;
  const int group = r / (group_m * tiles_n);
  const int first_m = group * group_m;
  const int gm = min(tiles_m - first_m, group_m);
  const int w = r - group * group_m * tiles_n;
  c.mt = first_m + w % gm;
  c.nt = w / gm;
  return c;
}

// cluster helpers (kC = 2: B multicast across a CTA pair)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the box lands at the same shared-memory offset in every CTA of `mask`; each CTA's mbarrier
// at `bar`'s offset receives complete_tx for the bytes delivered to it
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                               int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// TMA load with an L2 eviction-priority hint (createpolicy): the int8 GEMM's A panels are
// re-read by every tile of a raster group (evict_last), its B panels pass once per group
// (evict_first)
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                 int32_t c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// arrive on `bar` in every CTA of `mask` once this thread's MMAs so far have completed
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// The K range of one int8 GEMM launch: `n` blocks of `nk` 128-byte k-tiles each; block b
// reads the left operand's residues from column a_k0[b] and the right operand's from row
// b_row0[b] of tma_b (the sharded K split hands several arrived residue blocks to one
// launch; a single-GPU product is one block at 0, 0).
constexpr int kMaxKBlocks = 16;
struct KSpan {
  int n = 1, nk = 0;
  int a_k0[kMaxKBlocks] = {};
  int b_row0[kMaxKBlocks] = {};
};

// Persistent: CTA b takes tiles b, b + grid, ... of the (modulus, tile-row, tile-col) space;
// out[l][row][col] = (Σ_k a_l[row][k]·b_l[col][k]) mod m_l.  a_l's rows live at l·M + row
// of tma_a, b_l's at l·N + col of tma_b.  The TMA ring runs across tile boundaries and the
// two TMEM accumulators let the epilogue of tile i overlap the MMAs of tile i+1.
// kC = 2: CTA pairs (clusters of 2) take vertically adjacent tiles with the same B tile;
// each CTA loads half of that B tile and multicasts it to both (tma_b's box is then
// kBN/2 rows), so B crosses L2→SM once per pair; a stage is refilled only after both
// CTAs' MMAs released it (empty barriers count kC commits, multicast by each MMA issuer).
template <int kC>
__global__ void __launch_bounds__(192, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, int M, int N,
                   int64_t ldr, uint8_t* __restrict__ out, const OzConst cst, int tiles_m, int tiles_n,
                   int group_m, const KSpan ks, int accumulate, const uint32_t* __restrict__ tile_list, int list_len,
                   int hints) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + kAccBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAccBufs);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = ks.n * ks.nk;  // k-tiles per output tile over all K blocks
  const uint32_t crank = kC > 1 ? cluster_ctarank() : 0u;
  const int unit = static_cast<int>(blockIdx.x) / kC, nunits = static_cast<int>(gridDim.x) / kC;
  const int tiles_mu = (tiles_m + kC - 1) / kC;  // tile-rows in units of kC
  const int group_u = max(1, group_m / kC);
  // a tile list (symmetric products: the tiles that meet the upper triangle, in raster
  // order) replaces the full (tile-row, tile-col) space
  const int per = tile_list ? list_len : tiles_mu * tiles_n;
  const int total = per * cst.s;
  const auto coord = [&](int t) -> TileCoord {
    if (!tile_list) return tile_of(t, tiles_mu, tiles_n, group_u);
    TileCoord c;
    c.l = t / per;
    const uint32_t code = __ldg(tile_list + (t - c.l * per));
    c.mt = static_cast<int>(code >> 16);
    c.nt = static_cast<int>(code & 0xffffu);
    return c;
  };
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << kC) - 1u);

  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kC);
    }
    for (int b = 0; b < kAccBufs; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kBN * kAccBufs);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (kC > 1) cluster_sync_all();  // the peer's barriers exist before any multicast
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      tma_prefetch_desc(&tma_a);
      tma_prefetch_desc(&tma_b);
      const uint64_t pol_a = l2_policy_evict_last(), pol_b = l2_policy_evict_first();
      int it = 0;
      for (int t = unit; t < total; t += nunits) {
        const TileCoord tc = coord(t);
        const int mt = tc.mt * kC + static_cast<int>(crank);
        const int arow = tc.l * M + mt * kBM, brow = tc.l * N + tc.nt * kBN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int st = it % kStages;
          if (it >= kStages) mbar_wait(&empty[st], ((it / kStages) & 1) ^ 1);
          uint8_t* sa = smem + st * kStageBytes;
          mbar_arrive_expect_tx(&full[st], kStageBytes);
          const int blk = kb / ks.nk, kt = kb - blk * ks.nk;
          if (hints & 1) tma_load_2d_hint(sa, &tma_a, &full[st], ks.a_k0[blk] + kt * kBK, arow, pol_a);
          else tma_load_2d(sa, &tma_a, &full[st], ks.a_k0[blk] + kt * kBK, arow);
          if constexpr (kC == 1) {
            if (hints & 2) tma_load_2d_hint(sa + kABytes, &tma_b, &full[st], kt * kBK, ks.b_row0[blk] + brow, pol_b);
            else tma_load_2d(sa + kABytes, &tma_b, &full[st], kt * kBK, ks.b_row0[blk] + brow);
          } else {
            tma_load_2d_mc(sa + kABytes + crank * (kBBytes / kC), &tma_b, &full[st], kt * kBK,
                           ks.b_row0[blk] + brow + static_cast<int>(crank) * (kBN / kC), kMask);
          }
        }
      }
      if constexpr (kC > 1) {
        // drain: every stage's last release (both CTAs' commits) has arrived before teardown,
        // so no commit from the peer targets this CTA's barriers after it exits
        for (int j = 0; j < kStages; ++j, ++it)
          if (it >= kStages) mbar_wait(&empty[it % kStages], ((it / kStages) & 1) ^ 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int it = 0, n_t = 0;
      for (int t = unit; t < total; t += nunits, ++n_t) {
        const int acc = n_t & 1;
        if (n_t >= kAccBufs) mbar_wait(&tempty[acc], ((n_t >> 1) & 1) ^ 1);  // epilogue drained it
        tc_fence_after();
        const uint32_t tacc = tbase + acc * kBN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int st = it % kStages;
          mbar_wait(&full[st], (it / kStages) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + st * kStageBytes), b_addr = a_addr + kABytes;
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k)
            mma_i8(tacc, sw128_desc(a_addr + 32 * k), sw128_desc(b_addr + 32 * k), kIdesc, (kb | k) != 0);
          if constexpr (kC == 1) mma_commit(&empty[st]);  // the stage is free once these MMAs have read it
          else mma_commit_mc(&empty[st], kMask);           // ... in both CTAs (the peer refills it too)
        }
        mma_commit(&tfull[acc]);  // the accumulator is complete
      }
    }
  } else {  // epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
    const int q = warp & 3;
    int n_t = 0;
    for (int t = unit; t < total; t += nunits, ++n_t) {
      const TileCoord tc = coord(t);
      const int mt = tc.mt * kC + static_cast<int>(crank);
      const int acc = n_t & 1;
      mbar_wait(&tfull[acc], (n_t >> 1) & 1);
      tc_fence_after();
      const int row = mt * kBM + 32 * q + lane;
      const unsigned m = static_cast<unsigned>(cst.mi[tc.l]);
      const unsigned magic = cst.magic[tc.l], off = cst.offset[tc.l];
      uint8_t* orow = out + ((int64_t)tc.l * M + row) * ldr;
#pragma unroll 1
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + acc * kBN + (static_cast<uint32_t>(32 * q) << 16) + 32 * c, v);
        const int col = tc.nt * kBN + 32 * c;
        if (row < M && col < ldr) {
          uint32_t packed[8];
          uint4* dst = reinterpret_cast<uint4*>(orow + col);
          uint32_t prev[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          if (accumulate) {  // K-split in residue space: this block's product is added mod m_l
            const uint4 p0 = dst[0];
            prev[0] = p0.x, prev[1] = p0.y, prev[2] = p0.z, prev[3] = p0.w;
            if (col + 16 < ldr) {
              const uint4 p1 = dst[1];
              prev[4] = p1.x, prev[5] = p1.y, prev[6] = p1.z, prev[7] = p1.w;
            }
          }
          // a mod m in integer arithmetic (the FP64 form made this epilogue FP64-pipe bound
          // once K blocks got short): |a| < 2^14·K < 2^31 − 2^14, so u = a + offset is in
          // [0, 2^32) and u ≡ a (mod m); q = umulhi(u, floor(2^32/m)) is floor(u/m) or one
          // less, so u − q·m is in [0, 2m) and one unsigned min brings it into [0, m)
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            uint32_t word = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const unsigned u = v[4 * w + b] + off;
              unsigned r = u - __umulhi(u, magic) * m;
              r = min(r, r - m);
              r += (prev[w] >> (8 * b)) & 0xffu;  // K-split: add the earlier blocks' residue
              r = min(r, r - m);
              word |= r << (8 * b);
            }
            packed[w] = word;
          }
          dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          if (col + 16 < ldr) dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        }
      }
      tc_fence_before();  // this warp's TMEM reads are ordered before the release
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kC > 1) cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, kBN * kAccBufs);
  }
}

// ---------------------------------------------------------------- operand splits
__device__ __forceinline__ int exp_for(double amax) {
  // 2^e·amax in [2^52, 2^53)
  return amax == 0.0 ? 0 : kAlpha - 1 - ilogb(amax);
}

// x·2^e as scalbn(x, e) computes it (one correctly rounded multiply) while 2^e is a normal
// double — one DMUL instead of scalbn's range-reduction sequence (6 DMULs) — else scalbn
__device__ __forceinline__ bool pow2_normal(int e) { return e >= -1022 && e <= 1023; }
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double(static_cast<long long>(1023 + e) << 52); }
__device__ __forceinline__ double scale2(double x, int e) { return pow2_normal(e) ? x * pow2(e) : scalbn(x, e); }

// Round-to-nearest by the 1.5·2^52 shifter (exact for |x| < 2^51): one DFMA and one DADD
// instead of FRND.F64; and the low word of (r + 1.5·2^52) is r in two's complement, so
// the residue leaves the FP64 pipe without an F2I conversion.
constexpr double kShift52 = 6755399441055744.0;
__device__ __forceinline__ int resid(double a, double m, double inv_m) {
  const double q = fma(a, inv_m, kShift52) - kShift52;  // |a·inv_m| < 2^46: rint(a/m) up to one
  const double r = fma(-q, m, a);                          // exact: a small integer
  int ri = __double2loint(r + kShift52);
  const int mi = static_cast<int>(m);
  ri -= (ri > 127) ? mi : 0;   // q one off near a half-integer: bring r into int8 range
  ri += (ri < -128) ? mi : 0;
  return ri;
}

// ---- residues in packed FP32, two entries per instruction (FFMA2) ------------------
// An entry a' (integer-valued, |a'| < 2^53) becomes five 12-bit limbs a' = Σ_i L_i·2^(12i)
// (L_0..3 in [0, 4096), L_4 = a' >> 48 signed), each an exact float built from its bits.
// For modulus m: t = Σ_i L_i·(2^(12i) mod m) is an exact FP32 integer (|t| < 2^22.1), and
// r = t − m·rint(t·(1/m)) is exact; the float quotient can be one off near a half-integer,
// so |r| <= m/2 + 1, inside [−128, 127] for every modulus below 254 — 256 and 255 fold
// r = 128 to r − m.  r + 1.5·2^23 carries r's two's-complement byte in its low bits.  The
// moduli and the limb weights are template constants (immediates), so a residue costs
// about 4 FFMA2 + 4 more FP32 ops per two entries, against ~17 instructions per entry
// for the FP64 form above (the splits were issue-bound on those).
__device__ __forceinline__ float limb_f(uint32_t v) { return __uint_as_float(0x4B000000u | v) - 8388608.0f; }
__device__ __forceinline__ void limbs_of(double a, float (&L)[5]) {
  const long long ai = __double2ll_rn(a);
  const uint32_t lo = static_cast<uint32_t>(ai), hi = static_cast<uint32_t>(static_cast<unsigned long long>(ai) >> 32);
  L[0] = limb_f(lo & 0xFFFu);
  L[1] = limb_f((lo >> 12) & 0xFFFu);
  L[2] = limb_f(__funnelshift_r(lo, hi, 24) & 0xFFFu);
  L[3] = limb_f((hi >> 4) & 0xFFFu);
  L[4] = __uint_as_float(0x4B000000u | static_cast<uint32_t>((static_cast<int>(hi) >> 16) + 0x400000)) - 12582912.0f;
}
constexpr int pow2_mod(int e, int m) {
  long long r = 1;
  for (int i = 0; i < e; ++i) r = (r * 2) % m;
  return static_cast<int>(r);
}
// packed residues of two entries for modulus L: the bytes sit in bits 0-7 of each half
template <int L>
__device__ __forceinline__ unsigned long long resid2(const unsigned long long (&lp)[5]) {
  constexpr int m = kMod(L);
  constexpr float c1 = pow2_mod(12, m), c2 = pow2_mod(24, m), c3 = pow2_mod(36, m), c4 = pow2_mod(48, m);
  unsigned long long t = fma2(lp[1], bc2(c1), lp[0]);
  t = fma2(lp[2], bc2(c2), t);
  t = fma2(lp[3], bc2(c3), t);
  t = fma2(lp[4], bc2(c4), t);
  const unsigned long long q = add2(fma2(t, bc2(1.0f / m), bc2(12582912.0f)), bc2(-12582912.0f));
  unsigned long long r = fma2(q, bc2(-static_cast<float>(m)), t);
  if constexpr (m >= 254) {
    float r0, r1;
    upk2(r, r0, r1);
    r0 = r0 > 127.5f ? r0 - m : r0;
    r1 = r1 > 127.5f ? r1 - m : r1;
    r = pk2(r0, r1);
  }
  return add2(r, bc2(12582912.0f));
}
// 4 bytes (byte 0 of each 32-bit half of two packed pairs)
__device__ __forceinline__ uint32_t bytes4(unsigned long long p, unsigned long long q) {
  const uint32_t w0 = __byte_perm(static_cast<uint32_t>(p), static_cast<uint32_t>(p >> 32), 0x0040);
  const uint32_t w1 = __byte_perm(static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32), 0x0040);
  return __byte_perm(w0, w1, 0x5410);
}
// residues of P packed pairs (2P consecutive entries) for moduli L..S−1, plane stride `ps`
template <int L, int S, int P>
__device__ __forceinline__ void store_residues(const unsigned long long (&lp)[P][5], int8_t* out, int64_t ps) {
  if constexpr (L < S) {
    unsigned long long b[P];
#pragma unroll
    for (int p = 0; p < P; ++p) b[p] = resid2<L>(lp[p]);
    if constexpr (P == 4) {
      *reinterpret_cast<uint2*>(out + L * ps) = make_uint2(bytes4(b[0], b[1]), bytes4(b[2], b[3]));
    } else {
      static_assert(P == 8, "8 or 16 entries per thread");
      *reinterpret_cast<uint4*>(out + L * ps) =
          make_uint4(bytes4(b[0], b[1]), bytes4(b[2], b[3]), bytes4(b[4], b[5]), bytes4(b[6], b[7]));
    }
    store_residues<L + 1, S, P>(lp, out, ps);
  }
}
template <int P>
__device__ __forceinline__ void pack_limbs(const double (&a)[2 * P], unsigned long long (&lp)[P][5]) {
#pragma unroll
  for (int p = 0; p < P; ++p) {
    float x[5], y[5];
    limbs_of(a[2 * p], x);
    limbs_of(a[2 * p + 1], y);
#pragma unroll
    for (int i = 0; i < 5; ++i) lp[p][i] = pk2(x[i], y[i]);
  }
}

// Left operand, pass 1: one 256-thread block per row: the row's exponent (exps[row])
// and its L1/max ratio, folded into *ratio (float bits, atomic max): Σ_k |a'_ik| <=
// ratio·2^53 bounds the integer product (the moduli count follows from it).
// ratio[0]: max L1/max, ratio[2]: max L2/max (float bits, atomic max); the caller
// interleaves two operands' slots (ratio + 0 / + 1)
__global__ void __launch_bounds__(256) oz_rowstat_kernel(const double* __restrict__ X, int64_t ld, int rows, int k,
                                                         int* __restrict__ exps, unsigned* __restrict__ ratio) {
  __shared__ double smax[8], ssum[8], ssq[8];
  __shared__ int sbad[8];
  const int row = blockIdx.x;
  const double* xr = X + (int64_t)row * ld;
  double mx = 0.0, sum = 0.0, sq = 0.0;
  int bad = 0;
  for (int c = threadIdx.x; c < k; c += 256) {
    const double v = xr[c];
    bad |= !isfinite(v);
    mx = fmax(mx, fabs(v));
    sum += fabs(v);
    sq = fma(v, v, sq);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    smax[threadIdx.x >> 5] = mx;
    ssum[threadIdx.x >> 5] = sum;
    ssq[threadIdx.x >> 5] = sq;
    sbad[threadIdx.x >> 5] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mx = 0.0;
    sum = 0.0;
    sq = 0.0;
    bad = 0;
    for (int w = 0; w < 8; ++w) {
      mx = fmax(mx, smax[w]);
      sum += ssum[w];
      sq += ssq[w];
      bad |= sbad[w];
    }
    exps[row] = bad ? kBadExp : exp_for(mx);
    if (!bad && mx > 0.0) {
      atomicMax(ratio, __float_as_uint(static_cast<float>(sum / mx) * 1.0001f));
      atomicMax(ratio + 2, __float_as_uint(static_cast<float>(sqrt(sq) / mx) * 1.0001f));
    }
  }
}

// Left operand, pass 2: out[l][row][kp] int8 residues for S moduli (zero-padded from k).
template <int S>
__global__ void __launch_bounds__(256) oz_split_rows_kernel(const double* __restrict__ X, int64_t ld, int rows,
                                                            int k, int64_t kp, int8_t* __restrict__ out,
                                                            const int* __restrict__ exps) {
  const int row = blockIdx.x;
  const double* xr = X + (int64_t)row * ld;
  const int e = exps[row];
  const bool bad = e == kBadExp;
  for (int64_t c0 = threadIdx.x * 8; c0 < kp; c0 += 256 * 8) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t c = c0 + j;
      a[j] = (c < k && !bad) ? rint(scale2(xr[c], e)) : 0.0;
    }
    unsigned long long lp[4][5];
    pack_limbs<4>(a, lp);
    store_residues<0, S, 4>(lp, out + (int64_t)row * kp + c0, (int64_t)rows * kp);
  }
}

// Right operand, pass 1: per-column max |b| (as ordered bits) and non-finite flags.
__global__ void __launch_bounds__(256) oz_colmax_kernel(const double* __restrict__ B, int64_t ld, int k, int n,
                                                        unsigned long long* __restrict__ colmax,
                                                        double* __restrict__ colsum, double* __restrict__ colsq,
                                                        int* __restrict__ colbad) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= n) return;
  const int r0 = blockIdx.y * kColRows, r1 = min(k, r0 + kColRows);
  double mx = 0.0, sum = 0.0, sq = 0.0;
  int bad = 0;
  for (int r = r0; r < r1; ++r) {
    const double v = B[(int64_t)r * ld + c];
    bad |= !isfinite(v);
    mx = fmax(mx, fabs(v));
    sum += fabs(v);
    sq = fma(v, v, sq);
  }
  if (mx > 0.0) atomicMax(colmax + c, static_cast<unsigned long long>(__double_as_longlong(mx)));
  // per-kColRows-row partial sums, added in row-block order by oz_colratio_kernel: the bound,
  // and so the moduli count, is the same on every run (no floating-point atomics)
  colsum[(int64_t)blockIdx.y * n + c] = sum;
  colsq[(int64_t)blockIdx.y * n + c] = sq;
  if (bad) atomicOr(colbad + c, 1);
}

// Right operand, pass 1b: column exponents and the L1/max ratio bound (as rows above)
__global__ void __launch_bounds__(256) oz_colratio_kernel(const unsigned long long* __restrict__ colmax,
                                                          const double* __restrict__ colsum,
                                                          const double* __restrict__ colsq,
                                                          const int* __restrict__ colbad, int n, int kblocks,
                                                          int* __restrict__ exps, unsigned* __restrict__ ratio) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  float r = 0.0f, r2 = 0.0f;
  if (c < n) {
    const double mx = __longlong_as_double(static_cast<long long>(colmax[c]));
    const bool bad = colbad[c] != 0;
    exps[c] = bad ? kBadExp : exp_for(mx);
    if (!bad && mx > 0.0) {
      double sum = 0.0, sq = 0.0;
      for (int b = 0; b < kblocks; ++b) {
        sum += colsum[(int64_t)b * n + c];
        sq += colsq[(int64_t)b * n + c];
      }
      r = static_cast<float>(sum / mx) * 1.0001f;
      r2 = static_cast<float>(sqrt(sq) / mx) * 1.0001f;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, o));
    r2 = fmaxf(r2, __shfl_xor_sync(0xffffffffu, r2, o));
  }
  if ((threadIdx.x & 31) == 0 && r > 0.0f) {
    atomicMax(ratio, __float_as_uint(r));
    atomicMax(ratio + 2, __float_as_uint(r2));
  }
}

// Row-sharded right operand (sharded.cu): per-column statistics of one rank's row block,
// combined over the ranks in rank order.  part[y][3][n] per kColRows-row block y: max|x| (+inf
// when the block holds a non-finite entry), Σ|x|, Σx².
__global__ void __launch_bounds__(256) oz_colpart_kernel(const double* __restrict__ B, int64_t ld, int k, int n,
                                                         double* __restrict__ part) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= n) return;
  const int r0 = blockIdx.y * kColRows, r1 = min(k, r0 + kColRows);
  double mx = 0.0, sum = 0.0, sq = 0.0;
  int bad = 0;
  for (int r = r0; r < r1; ++r) {
    const double v = B[(int64_t)r * ld + c];
    bad |= !isfinite(v);
    mx = fmax(mx, fabs(v));
    sum += fabs(v);
    sq = fma(v, v, sq);
  }
  double* o = part + (int64_t)blockIdx.y * 3 * n + c;
  o[0] = bad ? INFINITY : mx;
  o[n] = sum;
  o[2 * (int64_t)n] = sq;
}
// out[3][n] = the rank's column statistics: the kColRows-row block partials in block order
// (for one rank: the same sums oz_colratio_kernel forms for the whole operand)
__global__ void __launch_bounds__(256) oz_colpart_sum_kernel(const double* __restrict__ part, int kblocks, int n,
                                                             double* __restrict__ out) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= n) return;
  double mx = 0.0, sum = 0.0, sq = 0.0;
  for (int y = 0; y < kblocks; ++y) {
    const double* o = part + (int64_t)y * 3 * n + c;
    mx = fmax(mx, o[0]);
    sum += o[n];
    sq += o[2 * (int64_t)n];
  }
  out[c] = mx;
  out[n + c] = sum;
  out[2 * (int64_t)n + c] = sq;
}
// gathered[g][3][n] (g in rank order) -> global column exponents and the L1/L2 ratio bounds
// (ratio[0], ratio[2], as oz_colratio_kernel); identical on every rank
__global__ void __launch_bounds__(256) oz_colcombine_kernel(const double* __restrict__ gathered, int world, int n,
                                                            int64_t stride, int* __restrict__ exps,
                                                            unsigned* __restrict__ ratio) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  float r = 0.0f, r2 = 0.0f;
  if (c < n) {
    double mx = 0.0, sum = 0.0, sq = 0.0;
    bool bad = false;
    for (int g = 0; g < world; ++g) {
      const double* o = gathered + (int64_t)g * stride;
      bad |= isinf(o[c]);
      mx = fmax(mx, o[c]);
      sum += o[n + c];
      sq += o[2 * (int64_t)n + c];
    }
    exps[c] = bad ? kBadExp : exp_for(mx);
    if (!bad && mx > 0.0) {
      r = static_cast<float>(sum / mx) * 1.0001f;
      r2 = static_cast<float>(sqrt(sq) / mx) * 1.0001f;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, o));
    r2 = fmaxf(r2, __shfl_xor_sync(0xffffffffu, r2, o));
  }
  if ((threadIdx.x & 31) == 0 && r > 0.0f) {
    atomicMax(ratio, __float_as_uint(r));
    atomicMax(ratio + 2, __float_as_uint(r2));
  }
}

// Right operand, pass 2: 64(k)×64(n) tiles transposed through shared memory into
// K-major residues out[l][col][kp].  Thread (column nn, 8-entry k segment 8g): the 8
// threads of a column write its 64 residue bytes per plane contiguously.  The tile's
// column index is XOR-swizzled by bit 4 of the row (phys = nn ^ 4·((kk >> 4) & 1)), so a
// warp's reads (4 columns × 8 segments) fall on 16 distinct double banks — the
// 2-wavefront minimum (unswizzled, segments 16 rows apart share banks: 4-way conflicts).
template <int S>
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const double* __restrict__ B, int64_t ld, int k, int n,
                                                            int64_t kp, int8_t* __restrict__ out,
                                                            const int* __restrict__ exps) {
  __shared__ double tile[64][65];
  const int n0 = blockIdx.x * 64, k0 = blockIdx.y * 64;
  for (int i = threadIdx.x; i < 64 * 64; i += 256) {
    const int kk = i >> 6, nn = i & 63;
    const int r = k0 + kk, c = n0 + nn;
    tile[kk][nn ^ (((kk >> 4) & 1) << 2)] = (r < k && c < n) ? B[(int64_t)r * ld + c] : 0.0;
  }
  __syncthreads();
  const int kc = (threadIdx.x & 7) * 8;
  if (k0 + kc >= kp) return;
  const int sw = ((kc >> 4) & 1) << 2;
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    const int nn = (threadIdx.x >> 3) + 32 * half;
    const int col = n0 + nn;
    if (col >= n) break;
    const int e = exps[col];
    const bool bad = e == kBadExp;
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = bad ? 0.0 : rint(scale2(tile[kc + j][nn ^ sw], e));
    unsigned long long lp[4][5];
    pack_limbs<4>(a, lp);
    store_residues<0, S, 4>(lp, out + (int64_t)col * kp + k0 + kc, (int64_t)n * kp);
  }
}

// launchers for the moduli counts the emulation uses (14..17)
int split_rows_launch(int s, const double* X, int64_t ld, int rows, int k, int64_t kp, int8_t* out, const int* exps,
                      cudaStream_t st) {
  switch (s) {
#define NNB_OZ_SR(S)                                                                          \
  case S:                                                                                     \
    oz_split_rows_kernel<S><<<static_cast<unsigned>(rows), 256, 0, st>>>(X, ld, rows, k, kp, out, exps); \
    break;
    NNB_OZ_SR(14)
    NNB_OZ_SR(15)
    NNB_OZ_SR(16)
    NNB_OZ_SR(17)
#undef NNB_OZ_SR
    default:
      return fail(7, "ozaki: unsupported moduli count " + std::to_string(s));
  }
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}
int split_cols_launch(int s, const double* B, int64_t ld, int k, int n, int64_t kp, int8_t* out, const int* exps,
                      cudaStream_t st) {
  const dim3 grid((unsigned)((n + 63) / 64), (unsigned)((kp + 63) / 64));
  switch (s) {
#define NNB_OZ_SC(S)                                                                  \
  case S:                                                                             \
    oz_split_cols_kernel<S><<<grid, 256, 0, st>>>(B, ld, k, n, kp, out, exps);       \
    break;
    NNB_OZ_SC(14)
    NNB_OZ_SC(15)
    NNB_OZ_SC(16)
    NNB_OZ_SC(17)
#undef NNB_OZ_SC
    default:
      return fail(7, "ozaki: unsupported moduli count " + std::to_string(s));
  }
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------- reconstruction
// C' from its residues by the CRT sum.  Residue pairs first: u ≡ r_a (mod a), u ≡ r_b
// (mod b) as u = r_a + a·v, v = (r_b − r_a)·a^-1 mod b (balanced: |u| <= 255 + 256·129 < 2^15.1), in packed
// FP32 for the thread's two elements at once (the bytes enter as 1.5·2^23 + r, bits
// 0x4B4000rr, and u leaves the same way, one DADD from a double).  Then, over the P =
// ceil(s/2) pair moduli, C' ≡ Σ_i u_i·W_i (mod M) with W_i = (M/p_i)·((M/p_i)^-1 mod p_i)
// < M, and |C'| < M/8 (the moduli count) makes C' = Σ u_i·W_i − q·M for q = rint(Σ/M).
// Each weight is split at 2^e (e = bits(M) − 34): the high parts' sum and q·mhi stay
// below 2^53 units of 2^e, so both and their difference are exact; the low parts' sum
// (< 2^(e+19)) carries ~10 roundings of 2^(e−34), i.e. below M·2^-66 — under the scheme's
// truncation error (>= M·2^-56) by far; the result is rounded once (the final add).
// 3 FP64 ops per pair against Garner's O(s^2) small-integer recurrence (round 2's first
// form): the reconstruction was issue-bound on that.
constexpr int cinv(int a, int m) {
  for (int x = 1; x < m; ++x)
    if ((a % m) * x % m == 1) return x;
  return 0;
}
template <int S, int I>
__device__ __forceinline__ void crt_pairs(const uint32_t (&w)[S], int b, const OzConst& c, double& sh0, double& sl0,
                                          double& sh1, double& sl1) {
  if constexpr (2 * I < S) {
    constexpr float kOff = 12582912.0f;  // 1.5·2^23
    const unsigned long long fa = pk2(__uint_as_float(__byte_perm(w[2 * I], 0x4B40u, 0x5460u + b)),
                                      __uint_as_float(__byte_perm(w[2 * I], 0x4B40u, 0x5460u + b + 1)));
    unsigned long long u = fa;
    if constexpr (2 * I + 1 < S) {
      constexpr int ma = kMod(2 * I), mb = kMod(2 * I + 1);
      const unsigned long long fb = pk2(__uint_as_float(__byte_perm(w[2 * I + 1], 0x4B40u, 0x5460u + b)),
                                        __uint_as_float(__byte_perm(w[2 * I + 1], 0x4B40u, 0x5460u + b + 1)));
      const unsigned long long t = mul2(add2(fb, mul2(fa, bc2(-1.0f))), bc2(static_cast<float>(cinv(ma, mb))));
      const unsigned long long q = add2(fma2(t, bc2(1.0f / mb), bc2(kOff)), bc2(-kOff));
      const unsigned long long v = fma2(q, bc2(-static_cast<float>(mb)), t);
      u = fma2(v, bc2(static_cast<float>(ma)), fa);
    }
    float u0, u1;
    upk2(u, u0, u1);
    constexpr double kBias = 4503599627370496.0 + 1262485504.0;  // 2^52 + 0x4B400000
    const double d0 = __hiloint2double(0x43300000, static_cast<int>(__float_as_uint(u0))) - kBias;
    const double d1 = __hiloint2double(0x43300000, static_cast<int>(__float_as_uint(u1))) - kBias;
    sh0 = fma(d0, c.pwhi[I], sh0);
    sl0 = fma(d0, c.pwlo[I], sl0);
    sh1 = fma(d1, c.pwhi[I], sh1);
    sl1 = fma(d1, c.pwlo[I], sl1);
    crt_pairs<S, I + 1>(w, b, c, sh0, sl0, sh1, sl1);
  }
}
// C' of the elements in bytes b and b+1 of the residue words w
template <int S>
__device__ __forceinline__ void crt_value_pair(const uint32_t (&w)[S], int b, const OzConst& c, double& x0,
                                               double& x1) {
  double sh0 = 0.0, sl0 = 0.0, sh1 = 0.0, sl1 = 0.0;
  crt_pairs<S, 0>(w, b, c, sh0, sl0, sh1, sl1);
  const double q0 = fma(sh0 + sl0, c.inv_m, kShift52) - kShift52;  // |Σ/M| < 2^19: rint by the shifter
  const double q1 = fma(sh1 + sl1, c.inv_m, kShift52) - kShift52;
  x0 = fma(-q0, c.pmhi, sh0) + fma(-q0, c.pmlo, sl0);
  x1 = fma(-q1, c.pmhi, sh1) + fma(-q1, c.pmlo, sl1);
}

// One block: 16 rows × 16·CPT columns; thread t: row t/16, CPT consecutive columns.
template <int S, int CPT>
__device__ __forceinline__ void recon_body(const uint8_t* __restrict__ res, int64_t ldr, int M, int N,
                                           const int* __restrict__ ea, const int* __restrict__ eb,
                                           const GemmEpilogue& ep, const OzConst& cst) {
  static_assert(CPT == 8 || CPT == 4, "8 or 4 columns per thread");
  using RV = typename std::conditional<CPT == 8, uint2, uint32_t>::type;
  __shared__ double red[8];
  __shared__ int redi[8];
  __shared__ int last_flag;
  const int row = blockIdx.y * 16 + (threadIdx.x >> 4);
  const int c0 = blockIdx.x * (16 * CPT) + (threadIdx.x & 15) * CPT;
  double ss = 0.0;
  int nf = 0;
  const bool want_red = ep.ss_partial != nullptr;
  // symmetric products (ep.sym): only the elements r <= c exist in the residues (the GEMM
  // ran the upper-triangle tiles); each is stored with its mirror and counted twice in
  // the Σ C² / non-finite reduction, as the DMMA epilogue does
  const bool sym = ep.sym != 0;
  if (row < M && c0 < N && !(sym && c0 + CPT - 1 < row)) {
    RV rv[S];
#pragma unroll
    for (int l = 0; l < S; ++l) rv[l] = *reinterpret_cast<const RV*>(res + ((int64_t)l * M + row) * ldr + c0);
    const int era = ea[row];
    // β·D of the thread's columns, loaded with the residues (more loads in flight)
    double dv[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int cc = c0 + j;
      dv[j] = (ep.D && cc < N && !(sym && row > cc)) ? ep.D[(int64_t)row * ep.ldd + cc] : 0.0;
    }
#pragma unroll
    for (int jp = 0; jp < CPT / 2; ++jp) {
      const int c = c0 + 2 * jp;
      if (c >= N) break;
      const bool two = c + 1 < N;
      double out2[2];
      double xp[2];
      {
        uint32_t w[S];
#pragma unroll
        for (int l = 0; l < S; ++l) {
          if constexpr (CPT == 8) w[l] = (jp < 2) ? rv[l].x : rv[l].y;
          else w[l] = rv[l];
        }
        crt_value_pair<S>(w, (2 * jp) & 3, cst, xp[0], xp[1]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double x = xp[h];
        // scale back by 2^-(ea+eb), then the chain's epilogue
        const int cc = c + h;
        const int e = (cc < N) ? eb[cc] : 0;
        double cv;
        if (era == kBadExp || e == kBadExp) cv = __longlong_as_double(0x7ff8000000000000LL);
        else cv = scale2(x, -(era + e));
        double o = ep.alpha * cv;
        if (ep.D && cc < N && !(sym && row > cc)) o = fma(ep.beta, dv[2 * jp + h], o);
        if ((int64_t)row + ep.diag_offset == cc) o += ep.gamma;
        out2[h] = o;
      }
      if (sym) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = c + h;
          if (cc >= N || row > cc) continue;
          ep.C[(int64_t)row * ep.ldc + cc] = out2[h];
          if (row < cc) ep.C[(int64_t)cc * ep.ldc + row] = out2[h];
          if (want_red) {
            const double w = row < cc ? 2.0 : 1.0;
            ss = fma(w * out2[h], out2[h], ss);
            nf += (row < cc ? 2 : 1) * !isfinite(out2[h]);
          }
        }
        continue;
      }
      double* cp = ep.C + (int64_t)row * ep.ldc + c;
      if (two) {
        *reinterpret_cast<double2*>(cp) = make_double2(out2[0], out2[1]);
      } else {
        cp[0] = out2[0];
      }
      if (want_red) {
        ss = fma(out2[0], out2[0], ss);
        nf += !isfinite(out2[0]);
        if (two) {
          ss = fma(out2[1], out2[1], ss);
          nf += !isfinite(out2[1]);
        }
      }
    }
  }
  if (!want_red) return;
  // deterministic reduction: fixed shuffle tree, fixed warp order, last block sums the
  // block partials in index order (the DMMA epilogue's scheme, gemm_f64.cuh)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ss = warp_sum(ss);
  nf = warp_sum_i(nf);
  if (lane == 0) {
    red[warp] = ss;
    redi[warp] = nf;
  }
  __syncthreads();
  const int pid = blockIdx.y * gridDim.x + blockIdx.x;
  const int nblocks = gridDim.x * gridDim.y;
  if (threadIdx.x == 0) {
    double tss = 0.0;
    int tnf = 0;
    for (int w = 0; w < 8; ++w) {
      tss += red[w];
      tnf += redi[w];
    }
    ep.ss_partial[pid] = tss;
    ep.nf_partial[pid] = tnf;
    __threadfence();
    const unsigned done = atomicAdd(ep.tile_counter, 1u);
    last_flag = (done == (unsigned)(nblocks - 1));
  }
  __syncthreads();
  if (!last_flag) return;
  __threadfence();
  double s2 = 0.0;
  int n2 = 0;
  for (int k = threadIdx.x; k < nblocks; k += 256) {
    s2 += __ldcg(ep.ss_partial + k);
    n2 += __ldcg(ep.nf_partial + k);
  }
  s2 = warp_sum(s2);
  n2 = warp_sum_i(n2);
  __syncthreads();
  if (lane == 0) {
    red[warp] = s2;
    redi[warp] = n2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    int ntot = 0;
    for (int w = 0; w < 8; ++w) {
      tot += red[w];
      ntot += redi[w];
    }
    if (ep.ss_out) *ep.ss_out = tot;
    if (ep.nf_out) *ep.nf_out = ntot;
    if (ep.eps_out) *ep.eps_out = sqrt(tot) * ep.eps_scale;
    *ep.tile_counter = 0u;
  }
}

// 8 columns per thread, 3 blocks per SM (85 registers; the CRT weights are kernel-parameter
// constants).  A/B at N=32768 under the power cap (tools/recon_ab.sh): 2 blocks per SM with
// D read in the column loop 16.0 ms, 3 blocks 15.7, D hoisted 14.0, both 13.1.
template <int S>
__global__ void __launch_bounds__(256, 3) oz_recon_kernel(const uint8_t* __restrict__ res, int64_t ldr, int M, int N,
                                                       const int* __restrict__ ea, const int* __restrict__ eb,
                                                       GemmEpilogue ep, const OzConst cst) {
  recon_body<S, 8>(res, ldr, M, N, ea, eb, ep, cst);
}

// Live per-kernel timing for bench.py's roofline (nnb_ozaki_profile / nnb_ozaki_stats):
// while enabled, each int8 GEMM, split and reconstruction launch is bracketed by CUDA
// events on its own stream; the sums are read (and the events drained) on request.
struct OzStats {
  std::mutex mu;
  bool on = false;
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    double work;
  };
  std::vector<Rec> pending;
  double ms[3] = {0, 0, 0}, work[3] = {0, 0, 0};
  int64_t n[3] = {0, 0, 0};
};
OzStats& stats() {
  static OzStats s;
  return s;
}
struct Timed {
  int cls;
  double work;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Timed(int c, double w, cudaStream_t s) : cls(c), work(w), st(s) {
    OzStats& S = stats();
    std::lock_guard<std::mutex> g(S.mu);
    if (!S.on) return;
    cudaEventCreate(&a);
    cudaEventRecord(a, st);
  }
  ~Timed() {
    if (!a) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, st);
    OzStats& S = stats();
    std::lock_guard<std::mutex> g(S.mu);
    S.pending.push_back({cls, a, b, work});
  }
};

// ---------------------------------------------------------------- host side
struct OzOperand {
  DevBuf res;   // int8 [s][rows][kp]
  DevBuf exps;  // int [rows]
  int64_t rows = 0, k = 0, kp = 0;
  int s = 0;
};

// Pass 1 of an operand: exponents and the L1/max ratio (into *ratio on the device).
// `left`: per-row scaling of a rows×k row-major operand; else per-column scaling of a
// k×n row-major right operand (n = rows of its K-major residues).
int operand_stats(const double* X, int64_t ld, int64_t rows, int64_t k, bool left, OzOperand& o, unsigned* ratio,
                  cudaStream_t st) {
  o.rows = rows;
  o.k = k;
  o.kp = (k + 15) / 16 * 16;
  o.s = 0;
  NNB_TRY(o.exps.alloc(sizeof(int) * std::max<int64_t>(rows, 1), st));
  Timed tm(1, (double)rows * k * 8.0, st);  // one read of the operand
  if (left) {
    oz_rowstat_kernel<<<static_cast<unsigned>(rows), 256, 0, st>>>(X, ld, (int)rows, (int)k, o.exps.as<int>(),
                                                                    ratio);
    count_launch();
  } else {
    const int64_t n = rows;
    DevBuf cm;
    const int64_t kb = (k + kColRows - 1) / kColRows;
    NNB_TRY(cm.alloc((sizeof(unsigned long long) + sizeof(int)) * n + 8 + 2 * sizeof(double) * kb * n, st));
    unsigned long long* colmax = cm.as<unsigned long long>();
    int* colbad = reinterpret_cast<int*>(colmax + n);
    double* colsum = reinterpret_cast<double*>(colbad + n + (n & 1));  // [kb][n] partials
    double* colsq = colsum + kb * n;
    NNB_CUDA(cudaMemsetAsync(cm.p, 0, (sizeof(unsigned long long) + sizeof(int)) * n, st));
    oz_colmax_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)kb), 256, 0, st>>>(X, ld, (int)k, (int)n, colmax,
                                                                                    colsum, colsq, colbad);
    oz_colratio_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(colmax, colsum, colsq, colbad, (int)n, (int)kb,
                                                                   o.exps.as<int>(), ratio);
    count_launch(2);
  }
  NNB_CUDA(cudaGetLastError());
  return 0;
}

// Pass 2: residues for c.s moduli (the operand's exponents from pass 1).
int operand_residues(const double* X, int64_t ld, bool left, const OzConst& c, OzOperand& o, cudaStream_t st) {
  NNB_TRY(o.res.alloc((size_t)c.s * o.rows * o.kp, st));
  o.s = c.s;
  Timed tm(1, (double)o.rows * o.k * (8.0 + c.s), st);  // 8 B in, s B out per entry
  if (left) return split_rows_launch(c.s, X, ld, (int)o.rows, (int)o.k, o.kp, o.res.as<int8_t>(), o.exps.as<int>(), st);
  return split_cols_launch(c.s, X, ld, (int)o.k, (int)o.rows, o.kp, o.res.as<int8_t>(), o.exps.as<int>(), st);
}

// moduli for |C'| <= ratio·2^106 < M/8 (the balanced Garner value is then C' itself)
__global__ void oz_ratio_out_kernel(const unsigned* __restrict__ rd, unsigned* out, unsigned seq) {
  if (threadIdx.x < 4) out[threadIdx.x] = rd[threadIdx.x];
  __threadfence_system();
  __syncwarp();
  if (threadIdx.x == 0) {
    *reinterpret_cast<volatile unsigned*>(out + 4) = seq;  // published after the ratios
    __threadfence_system();
  }
}

// The 4 ratio slots of `rd` on the host, the moment the stream reaches them: a one-warp
// kernel writes them and then a sequence number to mapped host memory, and the host polls
// that word instead of synchronising the stream (cudaStreamSynchronize returned ~0.14 ms
// after the GPU got there, an idle gap before every product's split at N=4096);
// cudaStreamQuery every 16384 polls surfaces any error of the stream.
int read_ratios_mapped(const unsigned* rd, unsigned out[4], cudaStream_t st) {
  static thread_local unsigned* host = nullptr;
  static thread_local unsigned* mapped = nullptr;
  static thread_local unsigned seq = 0;
  if (!host) {
    NNB_CUDA(cudaHostAlloc(&host, sizeof(unsigned) * 8, cudaHostAllocMapped));
    NNB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped), host, 0));
    host[4] = 0;
  }
  ++seq;
  oz_ratio_out_kernel<<<1, 32, 0, st>>>(rd, mapped, seq);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  volatile unsigned* flag = host + 4;
  for (int spins = 0; *flag != seq; ++spins) {
    if ((spins & 16383) == 16383) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) break;  // everything enqueued so far (the ratio kernel too) is done
      if (q != cudaErrorNotReady) NNB_CUDA(q);
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  for (int i = 0; i < 4; ++i) out[i] = reinterpret_cast<volatile unsigned*>(host)[i];
  return 0;
}

int moduli_for_ratio(double ratio) {
  const double need = 2.0 * kAlpha + std::log2(std::max(ratio, 1.0)) + 3.0;
  double have = 0.0;
  for (int s = 0; s < kMaxMod; ++s) {
    have += std::log2(static_cast<double>(kModuli[s]));
    if (have >= need) return s + 1;
  }
  return kMaxMod;
}

int launch_recon(int s, const uint8_t* res, int64_t ldr, int M, int N, const int* ea, const int* eb,
                 const GemmEpilogue& ep, const OzConst& c, cudaStream_t st) {
  const dim3 grid((unsigned)((N + 127) / 128), (unsigned)((M + 15) / 16));
  Timed tm(2, (double)M * N * (s + (ep.D ? 16.0 : 8.0)), st);  // s residue bytes (+ D) in, 8 B out
  switch (s) {
#define NNB_OZ_RECON(S)                                                                     \
  case S:                                                                                   \
    oz_recon_kernel<S><<<grid, 256, 0, st>>>(res, ldr, M, N, ea, eb, ep, c);                \
    break;
    NNB_OZ_RECON(14)
    NNB_OZ_RECON(15)
    NNB_OZ_RECON(16)
    NNB_OZ_RECON(17)
#undef NNB_OZ_RECON
    default:
      return fail(7, "ozaki: unsupported moduli count " + std::to_string(s));
  }
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

// Operand pinned by the chain for its whole run (A never changes between nests):
// its split is computed once per role and reused.
struct Pinned {
  const double* p = nullptr;
  int64_t ld = 0, rows = 0, cols = 0;
  OzOperand left, right;
  bool have_left = false, have_right = false;  // exponents and ratios formed
  float ratio_left = 0.0f, ratio_right = 0.0f, ratio_left2 = 0.0f, ratio_right2 = 0.0f;
};
thread_local std::vector<Pinned*> g_pins;  // at most a few: the chain's A, a chunked product's B

}  // namespace

bool oz_pin(const double* p, int64_t ld, int64_t rows, int64_t cols) {
  for (Pinned* q : g_pins)
    if (q->p == p) return false;  // already pinned by an enclosing scope: keep its splits
  Pinned* q = new Pinned();
  q->p = p;
  q->ld = ld;
  q->rows = rows;
  q->cols = cols;
  g_pins.push_back(q);
  return true;
}

void oz_unpin(const double* p) {
  for (size_t i = 0; i < g_pins.size(); ++i)
    if (g_pins[i]->p == p) {
      delete g_pins[i];
      g_pins.erase(g_pins.begin() + i);
      return;
    }
}

int make_tmap_u8(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                 int box_cols);

// s int8 GEMMs out[l] = (a_l[:, a_k0 : a_k0+K] · b_lᵀ) mod m_l (+ out[l] mod m_l when
// `accumulate`): a_l = a_res[l·M .. l·M+M) (row stride a_kp), b_l = b_res[l·N .. l·N+N)
// (row stride b_kp, zero beyond b_kp).  a_k0 > 0 multiplies a column block of the left
// operand's residues with a row block of the right operand's (the sharded K split);
// the left operand's columns past the block meet the right block's zeros.
// The tiles (128-row tile-row mt, 256-column tile-col nt) of an n×n product that meet its
// upper triangle (128·mt <= 256·nt + 255), in the grouped raster order of tile_of, packed
// mt << 16 | nt — built once per shape and device and kept.
const uint32_t* upper_tile_list(int tiles_m, int tiles_n, int group_m, int* len, cudaStream_t st) {
  static std::mutex mu;
  static std::vector<std::tuple<int, int, int, int, uint32_t*, int>> cache;  // dev, tm, tn, gm, list, len
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  for (auto& e : cache)
    if (std::get<0>(e) == dev && std::get<1>(e) == tiles_m && std::get<2>(e) == tiles_n && std::get<3>(e) == group_m) {
      *len = std::get<5>(e);
      return std::get<4>(e);
    }
  std::vector<uint32_t> h;
  for (int r = 0; r < tiles_m * tiles_n; ++r) {  // tile_of's raster, host side
    const int group = r / (group_m * tiles_n), first_m = group * group_m;
    const int gm = std::min(tiles_m - first_m, group_m), w = r - group * group_m * tiles_n;
    const int mt = first_m + w % gm, nt = w / gm;
    if (128LL * mt <= 256LL * nt + 255) h.push_back(static_cast<uint32_t>(mt) << 16 | static_cast<uint32_t>(nt));
  }
  uint32_t* d = nullptr;
  if (cudaMalloc(&d, sizeof(uint32_t) * h.size()) != cudaSuccess) return nullptr;
  if (cudaMemcpyAsync(d, h.data(), sizeof(uint32_t) * h.size(), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return nullptr;
  cache.emplace_back(dev, tiles_m, tiles_n, group_m, d, static_cast<int>(h.size()));
  *len = static_cast<int>(h.size());
  return d;
}

// b_rows: rows of the right operand's residue array (s·N for one block; the sharded
// gather holds G blocks of fs·N rows)
int launch_oz_gemm(const int8_t* a_res, int64_t M, int64_t a_kp, const int8_t* b_res, int64_t N, int64_t b_rows,
                   int64_t b_kp, const KSpan& ks, const OzConst& c, uint8_t* out, int64_t ldr, bool accumulate,
                   cudaStream_t st, int reserve_sms = 0, bool upper = false) {
  if (ks.n < 1 || ks.n > kMaxKBlocks) return fail(7, "ozaki: K block count out of range");
  const int64_t K = (int64_t)ks.n * ks.nk * kBK;  // work accounting: the padded K of the launch
  const int s = c.s;
  // NNB_DEBUG=1 NNB_OZ_CLUSTER=2: B multicast across CTA pairs (oz_gemm_kernel<2>)
  static const int kc_env = debug_env("NNB_OZ_CLUSTER") && std::atoi(debug_env("NNB_OZ_CLUSTER")) == 2 ? 2 : 1;
  const int kc = upper ? 1 : kc_env;
  CUtensorMap ta, tb;
  NNB_TRY(make_tmap_u8(&ta, a_res, (int64_t)s * M, a_kp, a_kp, kBM, kBK));
  NNB_TRY(make_tmap_u8(&tb, b_res, b_rows, b_kp, b_kp, kBN / kc, kBK));
  NNB_TRY(ensure_smem<oz_gemm_kernel<1>>(kGemmSmem));
  NNB_TRY(ensure_smem<oz_gemm_kernel<2>>(kGemmSmem));
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    NNB_CUDA(cudaGetDevice(&dev));
    NNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int tiles_m = (int)((M + kBM - 1) / kBM), tiles_n = (int)((N + kBN - 1) / kBN);
  static const int gm = debug_env("NNB_OZ_GROUP") ? std::atoi(debug_env("NNB_OZ_GROUP")) : kGroupM;
  // NNB_DEBUG=1 NNB_OZ_HINTS=bits: L2 eviction hints on the operand loads (1: A evict_last,
  // 2: B evict_first; both together measured 1.7x slower at N=32768: B panels serve a whole
  // raster group and evict_first lost them)
  static const int hints = debug_env("NNB_OZ_HINTS") ? std::atoi(debug_env("NNB_OZ_HINTS")) : 0;
  int list_len = 0;
  const uint32_t* list = nullptr;
  if (upper) {
    list = upper_tile_list(tiles_m, tiles_n, gm, &list_len, st);
    if (!list) return fail(7, "ozaki: upper-triangle tile list");
  }
  const int64_t total = (upper ? (int64_t)list_len : (int64_t)((tiles_m + kc - 1) / kc) * tiles_n) * s;
  if (total > INT32_MAX) return fail(7, "ozaki: too many tiles");
  Timed tm(0, 2.0 * s * (double)M * N * K * (upper ? (double)list_len / ((double)tiles_m * tiles_n) : 1.0), st);
  if (kc == 1) {
    const unsigned grid = (unsigned)std::min<int64_t>(total, std::max(1, sms - reserve_sms));
    oz_gemm_kernel<1><<<grid, 192, kGemmSmem, st>>>(ta, tb, (int)M, (int)N, ldr, out, c, tiles_m, tiles_n, gm, ks,
                                                    accumulate ? 1 : 0, list, list_len, hints);
  } else {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = kGemmSmem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static int max_clusters = 0;
    if (!max_clusters) {
      cfg.gridDim = dim3(2 * 74);
      NNB_CUDA(cudaOccupancyMaxActiveClusters(&max_clusters, oz_gemm_kernel<2>, &cfg));
      if (max_clusters < 1) return fail(7, "ozaki: no co-resident CTA pairs");
    }
    const int64_t units = std::min<int64_t>(total, std::max(1, std::min(max_clusters, (sms - reserve_sms) / 2)));
    cfg.gridDim = dim3((unsigned)(2 * units));
    NNB_CUDA(cudaLaunchKernelEx(&cfg, oz_gemm_kernel<2>, ta, tb, (int)M, (int)N, ldr, out, c, tiles_m, tiles_n, gm,
                                ks, accumulate ? 1 : 0, static_cast<const uint32_t*>(nullptr), 0, 0));
  }
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

thread_local int g_forced_s = 0;  // ozaki_force_moduli: a chunked product uses its whole product's count

int gemm_ozaki_impl(const GemmOp& op, cudaStream_t st, bool plan_only, int* s_out);

int gemm_ozaki(const GemmOp& op, cudaStream_t st) { return gemm_ozaki_impl(op, st, false, nullptr); }

// The moduli count the whole product `op` needs (its stats passes only; the operands'
// pins keep them), so that chunks of it can be formed with the same count — every
// element then rounds exactly as in the whole product.
int ozaki_plan_moduli(const GemmOp& op, cudaStream_t st, int* s_out) { return gemm_ozaki_impl(op, st, true, s_out); }
void ozaki_force_moduli(int s) { g_forced_s = s; }

int gemm_ozaki_impl(const GemmOp& op, cudaStream_t st, bool plan_only, int* s_out) {
  const int64_t M = op.M, N = op.N, K = op.K;
  if (K > kMaxK) return fail(7, "ozaki: inner dimension above 131071 (int32 accumulation bound)");
  if (op.ep.C2 || op.ep.acc_in) return fail(7, "ozaki: dual-output and K-split epilogues are DMMA-only");
  // Pass 1 of both operands: exponents, and the L1/max ratios that bound the integer
  // product (|C'| <= min(rA, rB)·2^106) — the moduli count follows from them, so a
  // product of the configs' matrices (ratios ~70) needs 15 moduli instead of the
  // worst case's 16.  One small host read per product.
  auto find = [](const double* p) -> Pinned* {
    for (Pinned* q : g_pins)
      if (q->p == p) return q;
    return nullptr;
  };
  // the ratios come back through mapped host memory written by a one-warp kernel, not
  // a copy: a device-to-host copy would queue behind any large copy on the same engine
  // (the host-buffer nest streams X out during its last product)
  DevBuf ratio_dev;  // [L1 A, L1 B, L2 A, L2 B] ratios to the row/column max
  NNB_TRY(ratio_dev.alloc(sizeof(unsigned) * 4, st));
  unsigned* rd = ratio_dev.as<unsigned>();
  NNB_CUDA(cudaMemsetAsync(rd, 0, sizeof(unsigned) * 4, st));
  OzOperand la, rb;
  OzOperand* L = &la;
  OzOperand* R = &rb;
  Pinned* pa = find(op.A);
  if (!(pa && op.lda == pa->ld && M == pa->rows && K == pa->cols)) pa = nullptr;
  Pinned* pb = find(op.B);
  if (!(pb && !op.b_kmajor && op.ldb == pb->ld && K == pb->rows && N == pb->cols)) pb = nullptr;
  if (pa) {
    L = &pa->left;
    if (!pa->have_left) NNB_TRY(operand_stats(op.A, op.lda, M, K, true, *L, rd, st));
  } else {
    NNB_TRY(operand_stats(op.A, op.lda, M, K, true, la, rd, st));
  }
  const bool right_as_rows = op.b_kmajor;  // Bᵀ given: its rows are B's columns
  if (pb) {
    R = &pb->right;
    if (!pb->have_right) NNB_TRY(operand_stats(op.B, op.ldb, N, K, false, *R, rd + 1, st));
  } else {
    NNB_TRY(operand_stats(op.B, op.ldb, N, K, right_as_rows, rb, rd + 1, st));
  }
  // A chunk of a planned product (ozaki_force_moduli) uses the whole product's count,
  // which bounds its own (its rows and columns are a subset): no host read at all.
  // Two pinned operands whose ratios are known need none either.
  const bool forced = g_forced_s > 0 && !plan_only;
  const bool known = pa && pa->have_left && pb && pb->have_right;
  double a1 = 1.0, b1 = 1.0, a2 = 1.0, b2 = 1.0;
  if (!forced && !known) {
    unsigned ratio_host[4];
    NNB_TRY(read_ratios_mapped(rd, ratio_host, st));
    trace_mark(st, "oz stats");
    const auto f = [](unsigned u) { return std::max((double)__builtin_bit_cast(float, u), 1.0); };
    a1 = f(ratio_host[0]);
    b1 = f(ratio_host[1]);
    a2 = f(ratio_host[2]);
    b2 = f(ratio_host[3]);
    if (pa && !pa->have_left) {
      pa->have_left = true;
      pa->ratio_left = (float)a1;
      pa->ratio_left2 = (float)a2;
    }
    if (pb && !pb->have_right) {
      pb->have_right = true;
      pb->ratio_right = (float)b1;
      pb->ratio_right2 = (float)b2;
    }
  }
  if (pa && pa->have_left) {
    a1 = pa->ratio_left;
    a2 = pa->ratio_left2;
  }
  if (pb && pb->have_right) {
    b1 = pb->ratio_right;
    b2 = pb->ratio_right2;
  }
  // |C'_ij| <= Σ|a'||b'| <= min(‖a'_i‖₁·max|b'|, max|a'|·‖b'_j‖₁, ‖a'_i‖₂‖b'_j‖₂)
  // (Cauchy-Schwarz) = 2^106·min(L1 ratios, product of L2 ratios); an operand with no
  // finite nonzero row/column reads 0 and its product is exact zeros
  const double ratio = std::min(std::min(a1, b1), a2 * b2);
  const int s_need = forced ? 0 : std::max(14, std::min(kMaxMod, moduli_for_ratio(std::min(ratio, (double)K))));
  if (plan_only) {
    *s_out = s_need;
    return 0;
  }
  // a forced count comes from the whole product of which this is a chunk: never fewer
  // than this chunk needs (a chunk's rows and columns are a subset of the whole's)
  const int s = std::max(s_need, g_forced_s);
  if (s > 17) return fail(7, "ozaki: more than 17 moduli needed");
  const OzConst c = make_const(s);
  // Pass 2: residues (a pinned operand keeps the planes it has when they suffice; the
  // moduli are a fixed sequence, so a prefix of its planes is the residues for s)
  if (L->s < s) NNB_TRY(operand_residues(op.A, op.lda, true, c, *L, st));
  if (R->s < s) NNB_TRY(operand_residues(op.B, op.ldb, right_as_rows, c, *R, st));
  trace_mark(st, "oz split");
  // s int8 GEMMs -> residues
  const int64_t ldr = (N + 15) / 16 * 16;
  DevBuf res;
  NNB_TRY(res.alloc((size_t)s * M * ldr, st));
  KSpan ks;
  ks.nk = (int)((K + kBK - 1) / kBK);
  NNB_TRY(launch_oz_gemm(L->res.as<int8_t>(), M, L->kp, R->res.as<int8_t>(), N, (int64_t)s * N, R->kp, ks, c,
                         res.as<uint8_t>(), ldr, false, st, 0, op.ep.sym != 0));
  trace_mark(st, "oz gemm");
  // reconstruction + the chain's epilogue
  NNB_TRY(launch_recon(s, res.as<uint8_t>(), ldr, (int)M, (int)N, L->exps.as<int>(), R->exps.as<int>(), op.ep, c,
                       st));
  trace_mark(st, "oz recon");
  return 0;
}

int ozaki_moduli_for(int64_t k) { return std::max(15, moduli_for(k)); }

void ozaki_profile(int on) {
  OzStats& S = stats();
  std::lock_guard<std::mutex> g(S.mu);
  S.on = on != 0;
}

// class 0: int8 GEMMs (work = int8 ops), 1: operand splits, 2: reconstructions (work = bytes)
void ozaki_stats(double* ms, double* work, int64_t* launches, int reset) {
  OzStats& S = stats();
  std::lock_guard<std::mutex> g(S.mu);
  for (auto& r : S.pending) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    S.ms[r.cls] += t;
    S.work[r.cls] += r.work;
    S.n[r.cls] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  S.pending.clear();
  for (int c = 0; c < 3; ++c) {
    if (ms) ms[c] = S.ms[c];
    if (work) work[c] = S.work[c];
    if (launches) launches[c] = S.n[c];
    if (reset) {
      S.ms[c] = S.work[c] = 0.0;
      S.n[c] = 0;
    }
  }
}

// ---------------------------------------------------------------- row-sharded products
// (sharded.cu drives them; see engine.cuh)
int oz_col_partials(const double* F, int64_t ld, int64_t rows, int64_t n, double* out, cudaStream_t st) {
  if (n <= 0) return 0;
  const int64_t kb = std::max<int64_t>((rows + kColRows - 1) / kColRows, 1);
  DevBuf part;
  NNB_TRY(part.alloc(sizeof(double) * 3 * kb * n, st));
  Timed tm(1, (double)rows * n * 8.0, st);
  if (rows > 0) {
    oz_colpart_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)kb), 256, 0, st>>>(F, ld, (int)rows, (int)n,
                                                                                    part.as<double>());
    oz_colpart_sum_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part.as<double>(), (int)kb, (int)n, out);
    count_launch(2);
  } else {
    NNB_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 3 * n, st));
  }
  NNB_CUDA(cudaGetLastError());
  return 0;
}

int oz_col_combine(const double* gathered, int world, int64_t stride, int64_t n, int* exps, unsigned* ratio,
                   cudaStream_t st) {
  if (n <= 0) return 0;
  oz_colcombine_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(gathered, world, (int)n, stride, exps, ratio);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

int oz_row_stats(const double* L, int64_t ld, int64_t rows, int64_t k, int* exps, unsigned* ratio, cudaStream_t st) {
  if (rows <= 0) return 0;
  Timed tm(1, (double)rows * k * 8.0, st);
  oz_rowstat_kernel<<<static_cast<unsigned>(rows), 256, 0, st>>>(L, ld, (int)rows, (int)k, exps, ratio);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

int oz_read_ratios(const unsigned* rd, double out[4], cudaStream_t st) {
  unsigned h[4];
  NNB_TRY(read_ratios_mapped(rd, h, st));
  for (int i = 0; i < 4; ++i) out[i] = std::max((double)__builtin_bit_cast(float, h[i]), 1.0);
  return 0;
}

int oz_moduli(double a1, double a2, double b1, double b2, int64_t K) {
  const double ratio = std::min(std::min(a1, b1), a2 * b2);
  return std::max(14, std::min(kMaxMod, moduli_for_ratio(std::min(ratio, (double)K))));
}

int oz_split_left(const double* L, int64_t ld, int64_t rows, int64_t k, const int* exps, int s, int8_t* out,
                  int64_t kp, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (s > 17) return fail(7, "ozaki: more than 17 moduli needed");
  const OzConst c = make_const(s);
  Timed tm(1, (double)rows * k * (8.0 + s), st);
  (void)c;
  return split_rows_launch(s, L, ld, (int)rows, (int)k, kp, out, exps, st);
}

int oz_split_right(const double* F, int64_t ld, int64_t k_rows, int64_t n, const int* exps, int s, int8_t* out,
                   int64_t kp, cudaStream_t st) {
  if (n <= 0 || kp <= 0) return 0;
  if (s > 17) return fail(7, "ozaki: more than 17 moduli needed");
  const OzConst c = make_const(s);
  Timed tm(1, (double)k_rows * n * (8.0 + s), st);
  (void)c;
  return split_cols_launch(s, F, ld, (int)k_rows, (int)n, kp, out, exps, st);
}

int oz_gemm_blocks(const int8_t* a_res, int64_t M, int64_t a_kp, const int64_t* a_k0, const int8_t* b_res, int64_t N,
                   int64_t b_rows, int64_t b_kp, const int64_t* b_row0, int nblk, int s, uint8_t* out, int64_t ldr,
                   bool accumulate, cudaStream_t st, int reserve_sms) {
  if (M <= 0 || N <= 0 || nblk <= 0) return 0;
  if (s > 17) return fail(7, "ozaki: more than 17 moduli needed");
  if (nblk > kMaxKBlocks) return fail(7, "ozaki: more than 16 K blocks in one launch");
  // a TMA box must start on a 16-byte boundary of the row (the sharded partition's 16-row
  // units guarantee it for the block origins)
  if (b_kp % 16 || a_kp % 16) return fail(7, "ozaki: residue rows not a multiple of 16 bytes");
  KSpan ks;
  ks.n = nblk;
  ks.nk = (int)((b_kp + kBK - 1) / kBK);
  for (int b = 0; b < nblk; ++b) {
    if (a_k0[b] % 16) return fail(7, "ozaki: block origin not a multiple of 16 bytes");
    ks.a_k0[b] = (int)a_k0[b];
    ks.b_row0[b] = (int)b_row0[b];
  }
  return launch_oz_gemm(a_res, M, a_kp, b_res, N, b_rows, b_kp, ks, make_const(s), out, ldr, accumulate, st,
                        reserve_sms);
}

int oz_reconstruct(int s, const uint8_t* res, int64_t ldr, int64_t M, int64_t N, const int* ea, const int* eb,
                   GemmEpilogue ep, RedWs* red, cudaStream_t st) {
  if (M <= 0 || N <= 0) return 0;
  if (red) {
    if (red->capacity < max_tiles_for(M, N)) return fail(7, "ozaki: reduction workspace too small");
    ep.ss_partial = red->ss_partial;
    ep.nf_partial = red->nf_partial;
    ep.tile_counter = red->counter;
  } else {
    ep.ss_partial = nullptr;
  }
  return launch_recon(s, res, ldr, (int)M, (int)N, ea, eb, ep, make_const(s), st);
}

}  // namespace nnb
