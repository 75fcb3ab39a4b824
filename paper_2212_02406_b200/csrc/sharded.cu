// Row-sharded Nested Neumann chain across GPUs (BASELINE config 3:
// N=32768 on 1/2/4/8 B200s) — SURVEY.md §8(e).
//
// Rank g owns the rows J_g = [row0_g, row0_g+rows_g) of A and X (16-row units,
// balanced).  Per nest, with full-size ping-pong buffers XF[2] and RF:
//   1. ring all-gather of X (NCCL send/recv on a side stream, G−1 steps);
//      overlapped with the K-split product
//        R_g = I_g − Σ_j A_g[:, J_j]·X_j,   own block first, then in ring order,
//      each partial GEMM waiting only for the ring step that delivers X_j;
//   2. eps = sqrt(Σ_g ‖R_g‖²)/√N with the per-rank partials all-gathered and
//      summed in rank order (bit-identical on every rank → identical stop
//      decisions), non-finite counts likewise;
//   3. ring all-gather of R overlapped with V_g = X_g + Σ_j X_g[:, J_j]·R_j,
//      then V_g = X_g + V_g·R (p−1 more) and X_{k+1, g} = V_g.
// p+1 local (rows_g × N × N) products per nest, 2 ring all-gathers.
// R_g is written straight into its slot of RF and the last Horner product
// straight into XF[next], so the gathers move data in place.
//
// Emulation mode runs all `world` virtual ranks in this process on one GPU:
// the buffers are shared, the ring is a no-op, and every other step (the
// partition, the K-split accumulation order, the rank-ordered eps) is the
// same code — that is how the partition logic is exercised on a 1-GPU box.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/nnb.h"
#include "comm.cuh"
#include "engine.cuh"

namespace nnb {
namespace {

// ---- NCCL, loaded at first use (reuses torch's libnccl when already loaded) ----
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define LOAD(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym))
    LOAD(getUniqueId, "ncclGetUniqueId");
    LOAD(commInitRank, "ncclCommInitRank");
    LOAD(commDestroy, "ncclCommDestroy");
    LOAD(send, "ncclSend");
    LOAD(recv, "ncclRecv");
    LOAD(allGather, "ncclAllGather");
    LOAD(groupStart, "ncclGroupStart");
    LOAD(groupEnd, "ncclGroupEnd");
    LOAD(errorString, "ncclGetErrorString");
#undef LOAD
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.send && api.recv &&
             api.allGather && api.groupStart && api.groupEnd && api.errorString;
  });
  return api;
}

#define NNB_NCCL(x)                                                                   \
  do {                                                                                \
    ncclResult_t _r = (x);                                                            \
    if (_r != ncclSuccess)                                                            \
      return fail(NNB_ERR_NCCL, std::string("NCCL error: ") + nccl().errorString(_r) + \
                                    " in " #x);                                       \
  } while (0)

int64_t pad8(int64_t c) { return (c + 7) / 8 * 8; }

__global__ void combine_ranks_kernel(const double* gathered, int world, double* eps_out,
                                     int* nf_out, double scale) {
  if (threadIdx.x == 0) {
    double ss = 0.0, nf = 0.0;
    for (int r = 0; r < world; ++r) {  // rank order: identical on every rank
      ss += gathered[2 * r];
      nf += gathered[2 * r + 1];
    }
    *eps_out = sqrt(ss) * scale;
    *nf_out = static_cast<int>(nf);
  }
}

__global__ void pack_pair_kernel(const double* ss, const int* nf, double* dst) {
  if (threadIdx.x == 0) {
    dst[0] = *ss;
    dst[1] = static_cast<double>(*nf);
  }
}

// X0 = diag(A)^-1 restricted to rows [row0, row0+rows): X[i][row0+i] = 1/A[i][row0+i].
__global__ void jacobi_rows_kernel(const double* __restrict__ A, int64_t lda, int64_t rows,
                                   int64_t row0, int64_t n, double* __restrict__ X, int64_t ldx) {
  const int64_t total = rows * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / n, c = idx % n;
    X[r * ldx + c] = (row0 + r == c) ? 1.0 / A[r * lda + c] : 0.0;
  }
}

}  // namespace

// wrappers shared with sparse_sharded.cu (comm.cuh)
ncclResult_t nccl_send(const void* buf, size_t count, int peer, nnb_comm* c, cudaStream_t s) {
  return nccl().send(buf, count, ncclDouble, peer, c->comm, s);
}
ncclResult_t nccl_recv(void* buf, size_t count, int peer, nnb_comm* c, cudaStream_t s) {
  return nccl().recv(buf, count, ncclDouble, peer, c->comm, s);
}
ncclResult_t nccl_group(bool start) { return start ? nccl().groupStart() : nccl().groupEnd(); }
ncclResult_t nccl_allgather(const void* send, void* recv, size_t count, nnb_comm* c, cudaStream_t s) {
  return nccl().allGather(send, recv, count, ncclDouble, c->comm, s);
}
const char* nccl_error(ncclResult_t r) { return nccl().errorString ? nccl().errorString(r) : "NCCL unavailable"; }

namespace {

struct Shard {
  int64_t n = 0, ld = 0;
  int world = 1;
  std::vector<int64_t> row0, rows;
  nnb_comm* comm = nullptr;  // null => emulation
  std::vector<int> local;    // ranks executed by this process
  cudaStream_t s = nullptr;
  std::vector<cudaEvent_t> ev;  // ev[q]: ring step q delivered its block
  cudaEvent_t ready = nullptr;
  RedWs red;
};

// 16-row units: every block starts at a multiple of 16 rows, so a block's columns of a
// left operand's int8 residues start on a 16-byte boundary (the TMA box origin the
// sharded int8 GEMM needs), and FP64 rows stay 16-byte aligned for the DMMA path
void partition(int64_t n, int world, std::vector<int64_t>& row0, std::vector<int64_t>& rows) {
  constexpr int64_t kUnit = 16;
  const int64_t units = (n + kUnit - 1) / kUnit;
  row0.assign(world, 0);
  rows.assign(world, 0);
  int64_t u0 = 0;
  for (int g = 0; g < world; ++g) {
    const int64_t u = units / world + (g < units % world ? 1 : 0);
    row0[g] = std::min<int64_t>(n, u0 * kUnit);
    rows[g] = std::min<int64_t>(n, (u0 + u) * kUnit) - row0[g];
    u0 += u;
  }
}

// In-place ring all-gather of the row blocks of `full` (n × ld) on the comm
// stream; ev[q] records after step q (block (me−q) mod G arrived).
int ring_allgather(Shard& sh, double* full) {
  if (!sh.comm || sh.world == 1) return 0;
  auto& api = nccl();
  const int G = sh.world, me = sh.comm->rank;
  NNB_CUDA(cudaEventRecord(sh.ready, sh.s));
  NNB_CUDA(cudaStreamWaitEvent(sh.comm->cs, sh.ready, 0));
  for (int q = 1; q < G; ++q) {
    const int send_blk = ((me - q + 1) % G + G) % G, recv_blk = ((me - q) % G + G) % G;
    NNB_NCCL(api.groupStart());
    NNB_NCCL(api.send(full + sh.row0[send_blk] * sh.ld, (size_t)(sh.rows[send_blk] * sh.ld),
                      ncclDouble, (me + 1) % G, sh.comm->comm, sh.comm->cs));
    NNB_NCCL(api.recv(full + sh.row0[recv_blk] * sh.ld, (size_t)(sh.rows[recv_blk] * sh.ld),
                      ncclDouble, (me - 1 + G) % G, sh.comm->comm, sh.comm->cs));
    NNB_NCCL(api.groupEnd());
    NNB_CUDA(cudaEventRecord(sh.ev[q], sh.comm->cs));
  }
  return 0;
}

// All-gather of the per-rank [Σ‖·‖², non-finite] pairs.  Every NCCL call of a
// communicator goes to its one communication stream (issue order = execution
// order on every rank); the compute stream hands over and waits by events.
int gather_pairs(Shard& sh, const double* pairs, double* gathered) {
  if (!sh.comm || sh.world == 1) {
    NNB_CUDA(cudaMemcpyAsync(gathered, pairs, sizeof(double) * 2 * sh.world, cudaMemcpyDeviceToDevice, sh.s));
    return 0;
  }
  NNB_CUDA(cudaEventRecord(sh.ready, sh.s));
  NNB_CUDA(cudaStreamWaitEvent(sh.comm->cs, sh.ready, 0));
  NNB_NCCL(nccl().allGather(pairs + 2 * sh.comm->rank, gathered, 2, ncclDouble, sh.comm->comm, sh.comm->cs));
  NNB_CUDA(cudaEventRecord(sh.ev[0], sh.comm->cs));  // ev[0] is free: ring events use q >= 1
  NNB_CUDA(cudaStreamWaitEvent(sh.s, sh.ev[0], 0));
  return 0;
}

// C_g = alpha·Σ_j L[:, J_j]·F_j + beta·D + gamma·I(row0_g), K split by the
// ranks' row blocks, own block first then ring order; the last partial
// carries the Σ C² / non-finite reduction when ss_out != null.
int ksplit_product(Shard& sh, int g, const double* L, int64_t ldl, const double* F, double alpha,
                   const double* D, double beta, double gamma, double* C, int64_t ldc,
                   bool wait_ring, double* ss_out, int* nf_out) {
  const int G = sh.world;
  int last = -1;  // the reduction rides on the last non-empty partial
  for (int q = 0; q < G; ++q)
    if (sh.rows[((g - q) % G + G) % G]) last = q;
  for (int q = 0; q < G; ++q) {
    const int j = ((g - q) % G + G) % G;
    if (sh.rows[j] == 0) continue;
    if (wait_ring && sh.comm && q > 0) NNB_CUDA(cudaStreamWaitEvent(sh.s, sh.ev[q], 0));
    GemmOp op;
    op.A = L + sh.row0[j];
    op.lda = ldl;
    op.B = F + sh.row0[j] * sh.ld;
    op.ldb = sh.ld;
    op.M = sh.rows[g];
    op.N = sh.n;
    op.K = sh.rows[j];
    op.ep.C = C;
    op.ep.ldc = ldc;
    op.ep.alpha = alpha;
    if (q == 0) {
      op.ep.D = D;
      op.ep.ldd = ldc;
      op.ep.beta = beta;
      op.ep.gamma = gamma;
      op.ep.diag_offset = sh.row0[g];
    } else {
      op.ep.D = C;
      op.ep.ldd = ldc;
      op.ep.beta = 1.0;
    }
    const bool reduce = (last == q) && nf_out;
    if (reduce) {
      op.ep.ss_out = ss_out;
      op.ep.nf_out = nf_out;
    }
    NNB_TRY(gemm(op, reduce ? &sh.red : nullptr, sh.s));
  }
  return 0;
}

// ---- int8 emulation of the sharded products (NNB_ARITH_FAST at large n, NNB_ARITH_OZAKI) ----
// The right operand F (X for the residual product, R for the Horner products) is gathered
// as int8 residues instead of FP64 rows:
//   1. every rank reduces its rows of F to per-column [max|x|, Σ|x|, Σx²]; the G records are
//      all-gathered and combined in rank order into F's column exponents and ratio bounds
//      (identical on every rank);
//   2. the moduli count s comes from those and the left operands' row ratios (a 16-byte
//      all-gather), the same count the single-GPU product of the whole matrices takes;
//   3. each rank splits its own block of F into K-major residues [s][n][kpb] (block g at a
//      fixed offset of one gathered buffer) and a ring all-gather moves the residue blocks;
//   4. rank g's product runs as G int8 GEMMs over the K blocks (own block first, then ring
//      order, each waiting only for its block) accumulating mod m_l, then one
//      reconstruction with the chain's epilogue.
// Every element equals the single-GPU emulated product's (same exponents, same residues, an
// exact modular sum, the same CRT reconstruction), so the sharded X matches the
// single-GPU X; FP64 traffic per nest drops to the G small records.
__global__ void max_slots_kernel(const unsigned* __restrict__ slots, int world, unsigned* __restrict__ out) {
  if (threadIdx.x < 4) {
    unsigned m = 0;
    for (int g = 0; g < world; ++g) m = max(m, slots[4 * g + threadIdx.x]);  // float bits >= 0: ordered
    out[threadIdx.x] = m;
  }
}

constexpr int kRingSms = 8;  // SMs the int8 GEMM leaves free while the residue ring runs
constexpr int kMaxGroup = 16;  // K blocks per int8 GEMM launch (ozaki.cu kMaxKBlocks)

struct OzSh {
  int64_t n = 0, kp = 0, kpb = 0, stride = 0;  // kpb: 16-padded rows of the largest block
  DevBuf stats;  // [G][stride]: 3n column statistics + 2 doubles (= 4 ratio slots)
  DevBuf ints;   // fexps[n] | aexps[n] | lexps[n] | rd[4] | rdf[4]
  DevBuf fres;   // gathered residues of F: block j at j·s·n·kpb (equal strides: one TMA map)
  int fcap = 0, fplanes = 0;
  bool fcombined = false, fknown = false;
  double fb1 = 1.0, fb2 = 1.0;
  std::vector<std::unique_ptr<DevBuf>> ares;  // pinned A: residues per local rank
  std::vector<int> aplanes;
  bool aknown = false;
  double aa1 = 1.0, aa2 = 1.0;
  DevBuf lres, out, slots;   // slots: [G][4] ratio slots
  int64_t lcap = 0, ocap = 0;
  const double* fsrc = nullptr;  // the F whose statistics were gathered last
  int* fexps() const { return ints.as<int>(); }
  int* aexps() const { return ints.as<int>() + n; }
  int* lexps() const { return ints.as<int>() + 2 * n; }
  unsigned* rd() const { return reinterpret_cast<unsigned*>(ints.as<int>() + 3 * n); }
  unsigned* rdf() const { return rd() + 4; }
};

// in-place all-gather of equal per-rank records (count doubles each) on the comm stream
int gather_records(Shard& sh, double* buf, size_t count) {
  if (!sh.comm || sh.world == 1) return 0;
  NNB_CUDA(cudaEventRecord(sh.ready, sh.s));
  NNB_CUDA(cudaStreamWaitEvent(sh.comm->cs, sh.ready, 0));
  NNB_NCCL(nccl().allGather(buf + count * sh.comm->rank, buf, count, ncclDouble, sh.comm->comm, sh.comm->cs));
  NNB_CUDA(cudaEventRecord(sh.ev[0], sh.comm->cs));
  NNB_CUDA(cudaStreamWaitEvent(sh.s, sh.ev[0], 0));
  return 0;
}

int oz_init(Shard& sh, OzSh& oz) {
  const int G = sh.world;
  oz.n = sh.n;
  oz.kp = (sh.n + 15) / 16 * 16;
  oz.kpb = 16;
  for (int j = 0; j < G; ++j) oz.kpb = std::max<int64_t>(oz.kpb, (sh.rows[j] + 15) / 16 * 16);
  oz.stride = 3 * sh.n + 2;
  NNB_TRY(oz.stats.alloc(sizeof(double) * oz.stride * G, sh.s));
  NNB_TRY(oz.ints.alloc(sizeof(int) * (3 * sh.n + 8), sh.s));
  NNB_TRY(oz.slots.alloc(sizeof(unsigned) * 4 * G, sh.s));
  oz.ares.clear();
  for (size_t i = 0; i < sh.local.size(); ++i) oz.ares.emplace_back(new DevBuf());
  oz.aplanes.assign(sh.local.size(), 0);
  return 0;
}

// step 1 for a new F (full-size buffer, rank g's rows at row0_g)
int oz_prepare_right(Shard& sh, OzSh& oz, const double* F) {
  for (int g : sh.local)
    NNB_TRY(oz_col_partials(F + sh.row0[g] * sh.ld, sh.ld, sh.rows[g], sh.n, oz.stats.as<double>() + g * oz.stride,
                            sh.s));
  NNB_TRY(gather_records(sh, oz.stats.as<double>(), (size_t)oz.stride));
  oz.fsrc = F;
  oz.fcombined = false;
  oz.fknown = false;
  oz.fplanes = 0;
  return 0;
}

// in-place ring all-gather of F's residue blocks (s planes) on the comm stream
int oz_ring(Shard& sh, OzSh& oz, int s) {
  if (!sh.comm || sh.world == 1) return 0;
  auto& api = nccl();
  const int G = sh.world, me = sh.comm->rank;
  uint8_t* base = oz.fres.as<uint8_t>();
  auto blk = [&](int j) { return base + (size_t)j * s * oz.n * oz.kpb; };
  auto bytes = [&](int j) { return sh.rows[j] ? (size_t)s * oz.n * oz.kpb : (size_t)0; };
  NNB_CUDA(cudaEventRecord(sh.ready, sh.s));
  NNB_CUDA(cudaStreamWaitEvent(sh.comm->cs, sh.ready, 0));
  for (int q = 1; q < G; ++q) {
    const int send_blk = ((me - q + 1) % G + G) % G, recv_blk = ((me - q) % G + G) % G;
    NNB_NCCL(api.groupStart());
    if (bytes(send_blk)) NNB_NCCL(api.send(blk(send_blk), bytes(send_blk), ncclUint8, (me + 1) % G, sh.comm->comm, sh.comm->cs));
    if (bytes(recv_blk)) NNB_NCCL(api.recv(blk(recv_blk), bytes(recv_blk), ncclUint8, (me - 1 + G) % G, sh.comm->comm, sh.comm->cs));
    NNB_NCCL(api.groupEnd());
    NNB_CUDA(cudaEventRecord(sh.ev[q], sh.comm->cs));
  }
  return 0;
}

// steps 2-4: C_g = ep_of(g)(L_g·F) for every local rank g; after(g) runs on the stream
// right after rank g's reconstruction.  `pinned`: L is the chain's A (splits kept).
int oz_product(Shard& sh, OzSh& oz, const std::function<const double*(int)>& left, int64_t ldl, bool pinned,
               const std::function<GemmEpilogue(int)>& ep_of, const std::function<int(int)>& after) {
  const int G = sh.world;
  const int64_t n = sh.n;
  int* lexps = pinned ? oz.aexps() : oz.lexps();
  // ---- 2. moduli count: F's column ratios (combined once per F), the left rows' ratios
  const bool need_left = !(pinned && oz.aknown);
  double a1 = oz.aa1, a2 = oz.aa2;
  if (!oz.fcombined || need_left) {
    unsigned* rd = oz.rd();
    NNB_CUDA(cudaMemsetAsync(rd, 0, sizeof(unsigned) * 4, sh.s));
    if (!oz.fcombined) {
      NNB_TRY(oz_col_combine(oz.stats.as<double>(), G, oz.stride, n, oz.fexps(), rd + 1, sh.s));
      oz.fcombined = true;
    }
    if (need_left)
      for (int g : sh.local)
        NNB_TRY(oz_row_stats(left(g), ldl, sh.rows[g], n, lexps + sh.row0[g], rd, sh.s));
    double r[4];
    if (sh.comm && G > 1) {  // every rank's 4 slots (16 B), then the slot-wise max
      unsigned* slots = oz.slots.as<unsigned>();
      NNB_CUDA(cudaMemcpyAsync(slots + 4 * sh.comm->rank, rd, sizeof(unsigned) * 4, cudaMemcpyDeviceToDevice, sh.s));
      NNB_TRY(gather_records(sh, oz.slots.as<double>(), 2));
      max_slots_kernel<<<1, 32, 0, sh.s>>>(slots, G, oz.rdf());
      count_launch();
      NNB_TRY(oz_read_ratios(oz.rdf(), r, sh.s));
    } else {
      NNB_TRY(oz_read_ratios(rd, r, sh.s));
    }
    if (!oz.fknown) {
      oz.fb1 = r[1];
      oz.fb2 = r[3];
      oz.fknown = true;
    }
    if (need_left) {
      a1 = r[0];
      a2 = r[2];
      if (pinned) {
        oz.aa1 = a1;
        oz.aa2 = a2;
        oz.aknown = true;
      }
    }
  }
  const int s = oz_moduli(a1, a2, oz.fb1, oz.fb2, n);
  // ---- 3. F's residues: own block(s) split, then the ring (again only if s grew)
  if (oz.fplanes < s) {
    if (oz.fcap < s) {
      NNB_TRY(oz.fres.alloc((size_t)G * s * n * oz.kpb, sh.s));
      oz.fcap = s;
    }
    for (int g : sh.local)
      NNB_TRY(oz_split_right(oz.fsrc + sh.row0[g] * sh.ld, sh.ld, sh.rows[g], n, oz.fexps(), s,
                             oz.fres.as<int8_t>() + (size_t)g * s * n * oz.kpb, oz.kpb, sh.s));
    NNB_TRY(oz_ring(sh, oz, s));
    oz.fplanes = s;
  }
  const int fs = oz.fplanes;  // F's planes (a prefix of them serves s)
  // ---- 4. per local rank: left residues, the G block GEMMs, the reconstruction
  for (size_t li = 0; li < sh.local.size(); ++li) {
    const int g = sh.local[li];
    const int64_t rows = sh.rows[g];
    if (rows == 0) continue;
    DevBuf* lbuf = &oz.lres;
    if (pinned) {
      lbuf = oz.ares[li].get();
      if (oz.aplanes[li] < s) {
        NNB_TRY(lbuf->alloc((size_t)s * rows * oz.kp, sh.s));
        NNB_TRY(oz_split_left(left(g), ldl, rows, n, lexps + sh.row0[g], s, lbuf->as<int8_t>(), oz.kp, sh.s));
        oz.aplanes[li] = s;
      }
    } else {
      if (oz.lcap < (int64_t)s * rows) {
        NNB_TRY(oz.lres.alloc((size_t)s * rows * oz.kp, sh.s));
        oz.lcap = (int64_t)s * rows;
      }
      NNB_TRY(oz_split_left(left(g), ldl, rows, n, lexps + sh.row0[g], s, lbuf->as<int8_t>(), oz.kp, sh.s));
    }
    if (oz.ocap < (int64_t)s * rows) {
      NNB_TRY(oz.out.alloc((size_t)s * rows * oz.kp, sh.s));
      oz.ocap = (int64_t)s * rows;
    }
    // residue arrays are plane-major, so an array split for more planes than s serves s as
    // its first s planes; only F's block offsets depend on the planes it was split with (fs)
    // the K blocks in ring order (own block first), grouped 1, 2, then the rest: one launch
    // per group, each waiting only for its last block's ring step, so the ring (≈2.5 ms a step
    // at G=8, N=32768) stays ahead of the GEMMs (≈7 ms a block) while 3 launches instead of G
    // re-read and re-write the residues so far
    std::vector<std::pair<int, int>> groups;  // [q0, q1) in ring steps
    for (int q0 = 0, want = 1; q0 < G; want = (want == 1 ? 2 : G)) {
      const int q1 = std::min(G, q0 + std::min<int>(want, (int)kMaxGroup));
      groups.emplace_back(q0, q1);
      q0 = q1;
    }
    bool first = true;
    for (const auto& grp : groups) {
      int64_t a_k0[kMaxGroup], b_row0[kMaxGroup];
      int nb = 0;
      for (int q = grp.first; q < grp.second; ++q) {
        const int jj = ((g - q) % G + G) % G;
        if (sh.rows[jj] == 0) continue;
        a_k0[nb] = sh.row0[jj];
        b_row0[nb] = (int64_t)jj * fs * n;
        ++nb;
      }
      if (nb == 0) continue;
      const int q_last = grp.second - 1;
      if (sh.comm && q_last > 0) NNB_CUDA(cudaStreamWaitEvent(sh.s, sh.ev[q_last], 0));
      // the int8 GEMM is persistent (one CTA per SM, never yielding): while ring steps are
      // still to come it leaves kRingSms SMs to NCCL's send/recv CTAs, which could not
      // otherwise be scheduled before the grid drains (stream priority orders only pending CTAs)
      const int reserve = (sh.comm && G > 1 && q_last < G - 1) ? kRingSms : 0;
      NNB_TRY(oz_gemm_blocks(lbuf->as<int8_t>(), rows, oz.kp, a_k0, oz.fres.as<int8_t>(), n, (int64_t)G * fs * n,
                             oz.kpb, b_row0, nb, s, oz.out.as<uint8_t>(), oz.kp, !first, sh.s, reserve));
      first = false;
    }
    NNB_TRY(oz_reconstruct(s, oz.out.as<uint8_t>(), oz.kp, rows, n, lexps + sh.row0[g], oz.fexps(), ep_of(g),
                           &sh.red, sh.s));
    NNB_TRY(after(g));
  }
  return 0;
}

int run_sharded(Shard& sh, const double* A_local, int64_t lda_rows_stride, bool a_full,
                double* XF0, double* XF1, double* RF, double* Vbase, const ChainCfg& cfg,
                double* eps_hist, ChainOut* out, OzSh* oz) {
  const int G = sh.world, p = cfg.p;
  const int64_t ld = sh.ld;
  const int slots = cfg.max_iters + 1;
  const double scale = 1.0 / std::sqrt(static_cast<double>(sh.n));
  NNB_TRY(sh.red.init(max_tiles_for(sh.n, sh.n), sh.s));
  DevBuf scal;
  const size_t nf_count = (size_t)slots * (p + 1);
  // per-rank [ss, nf] pairs, gathered pairs, eps history, nf history, temp scalars
  NNB_TRY(scal.alloc(sizeof(double) * (2 * G + 2 * G + slots + 8) + sizeof(int) * (nf_count + 8 + G),
                     sh.s));
  NNB_CUDA(cudaMemsetAsync(scal.p, 0, scal.bytes, sh.s));
  double* pairs = scal.as<double>();      // [2G] this process's per-rank pairs
  double* gathered = pairs + 2 * G;       // [2G] all ranks' pairs
  double* eps_dev = gathered + 2 * G;     // [slots]
  double* ss_tmp = eps_dev + slots;       // [8]
  int* nf_dev = reinterpret_cast<int*>(ss_tmp + 8);  // [nf_count]
  int* nf_tmp = nf_dev + nf_count;        // [8 + G]

  double* XF[2] = {XF0, XF1};
  int cur = 0;
  cudaEvent_t e0, e1;
  NNB_CUDA(cudaEventCreate(&e0));
  NNB_CUDA(cudaEventCreate(&e1));
  NNB_CUDA(cudaEventRecord(e0, sh.s));

  auto a_rows = [&](int g) -> const double* {
    return a_full ? A_local + sh.row0[g] * lda_rows_stride : A_local;
  };
  auto vbuf = [&](int g, int which) -> double* {
    // emulation: full-size V buffers sliced per rank; real: rows_g × ld buffers
    const int64_t rows_total = a_full ? sh.n : sh.rows[g];
    return Vbase + (size_t)which * rows_total * ld + (a_full ? sh.row0[g] * ld : 0);
  };

  std::vector<double> eps_h(slots, 0.0);
  std::vector<int> nf_h(nf_count, 0);
  int k = 0, products = 0, stopped = 1, recorded = 0;
  // Fixed-count mode stops at a divergent nest (proj/src/solver.cpp:151-157) as the
  // single-GPU chain does: the rank-combined non-finite flags of nest k (identical on
  // every rank, so every rank takes the same decision) go to pinned memory behind an
  // event; nest k is enqueued once nest k−2 completed finite.
  const bool watch = cfg.tol <= 0.0 && cfg.max_iters >= 3;
  constexpr int kLag = 2;
  int* nf_watch = nullptr;
  std::vector<cudaEvent_t> nest_done(slots, nullptr);
  if (watch) NNB_CUDA(cudaHostAlloc(&nf_watch, sizeof(int) * nf_count, cudaHostAllocDefault));
  struct WatchGuard {
    std::vector<cudaEvent_t>& ev;
    int* pinned;
    ~WatchGuard() {
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
      if (pinned) cudaFreeHost(pinned);
    }
  } watch_guard{nest_done, nf_watch};
  for (;; ++k) {
    const bool last = k >= cfg.max_iters;
    if (last && !cfg.final_residual) break;
    if (watch && k >= kLag && nest_done[k - kLag]) {
      NNB_CUDA(cudaEventSynchronize(nest_done[k - kLag]));
      bool bad = false;
      for (int j = 0; j <= p; ++j) bad |= nf_watch[(k - kLag) * (p + 1) + j] != 0;
      if (bad) break;  // reported below from the device flags
    }
    // ---- R_g = I_g − A_g·X (ring all-gather of X overlapped) ----
    if (oz) {
      NNB_TRY(oz_prepare_right(sh, *oz, XF[cur]));
      NNB_TRY(oz_product(
          sh, *oz, a_rows, lda_rows_stride, true,
          [&](int g) {
            GemmEpilogue ep;
            ep.C = RF + sh.row0[g] * ld;
            ep.ldc = ld;
            ep.alpha = -1.0;
            ep.gamma = 1.0;
            ep.diag_offset = sh.row0[g];
            ep.ss_out = ss_tmp;
            ep.nf_out = nf_tmp;
            return ep;
          },
          [&](int g) {
            pack_pair_kernel<<<1, 32, 0, sh.s>>>(ss_tmp, nf_tmp, pairs + 2 * g);
            count_launch();
            return 0;
          }));
    } else {
      NNB_TRY(ring_allgather(sh, XF[cur]));
      for (int g : sh.local) {
        NNB_TRY(ksplit_product(sh, g, a_rows(g), lda_rows_stride, XF[cur], -1.0, nullptr, 0.0, 1.0,
                               RF + sh.row0[g] * ld, ld, true, ss_tmp, nf_tmp));
        pack_pair_kernel<<<1, 32, 0, sh.s>>>(ss_tmp, nf_tmp, pairs + 2 * g);
        count_launch();
      }
    }
    // ---- eps: per-rank pairs gathered, summed in rank order ----
    NNB_TRY(gather_pairs(sh, pairs, gathered));
    combine_ranks_kernel<<<1, 32, 0, sh.s>>>(gathered, G, eps_dev + k, nf_dev + k * (p + 1), scale);
    count_launch();
    ++products;
    recorded = k + 1;
    if (cfg.tol > 0.0) {
      NNB_CUDA(cudaMemcpyAsync(eps_h.data(), eps_dev, sizeof(double) * slots,
                               cudaMemcpyDeviceToHost, sh.s));
      NNB_CUDA(cudaMemcpyAsync(nf_h.data(), nf_dev, sizeof(int) * nf_count,
                               cudaMemcpyDeviceToHost, sh.s));
      NNB_CUDA(cudaStreamSynchronize(sh.s));
      bool bad = false;
      for (int q = 0; q <= k * (p + 1); ++q) bad |= nf_h[q] != 0;
      if (bad) break;
      if (eps_h[k] < cfg.tol) {
        stopped = 0;
        break;
      }
    }
    if (last) break;
    if (p == 0) continue;
    // ---- Horner: V_g = X_g + V_g·R (ring all-gather of R overlapped with the first) ----
    const int nxt = cur ^ 1;
    if (oz) {
      NNB_TRY(oz_prepare_right(sh, *oz, RF));
      for (int j = 1; j <= p; ++j) {
        // V_g = X_g + V_g·R, the first V_g being X_g; the last lands in XF[nxt]
        NNB_TRY(oz_product(
            sh, *oz,
            [&](int g) -> const double* {
              return j == 1 ? XF[cur] + sh.row0[g] * ld : vbuf(g, (j - 2) & 1);
            },
            ld, false,
            [&](int g) {
              GemmEpilogue ep;
              ep.C = (j == p) ? XF[nxt] + sh.row0[g] * ld : vbuf(g, (j - 1) & 1);
              ep.ldc = ld;
              ep.D = XF[cur] + sh.row0[g] * ld;
              ep.ldd = ld;
              ep.beta = 1.0;
              ep.ss_out = ss_tmp + 1;
              ep.nf_out = nf_tmp + 8 + g;
              return ep;
            },
            [](int) { return 0; }));
      }
    } else {
    NNB_TRY(ring_allgather(sh, RF));
    for (int g : sh.local) {
      const double* xg = XF[cur] + sh.row0[g] * ld;
      const double* v = xg;
      for (int j = 1; j <= p; ++j) {
        double* dst = (j == p) ? XF[nxt] + sh.row0[g] * ld : vbuf(g, (j - 1) & 1);
        // the nf of a Horner product on rank g is folded into slot j via nf_tmp[g]
        NNB_TRY(ksplit_product(sh, g, v, ld, RF, 1.0, xg, 1.0, 0.0, dst, ld, j == 1, ss_tmp + 1,
                               nf_tmp + 8 + g));
        v = dst;
      }
    }
    }
    products += p;  // global N^3-equivalent products (each rank did its row share)
    // fold this nest's Horner non-finite flags (all local ranks; gathered over ranks below)
    for (int g : sh.local) {
      pack_pair_kernel<<<1, 32, 0, sh.s>>>(ss_tmp + 1, nf_tmp + 8 + g, pairs + 2 * g);
      count_launch();
    }
    NNB_TRY(gather_pairs(sh, pairs, gathered));
    combine_ranks_kernel<<<1, 32, 0, sh.s>>>(gathered, G, ss_tmp + 2, nf_dev + k * (p + 1) + p,
                                             scale);
    count_launch();
    cur = nxt;
    if (watch) {
      NNB_CUDA(cudaMemcpyAsync(nf_watch + k * (p + 1), nf_dev + k * (p + 1), sizeof(int) * (p + 1),
                               cudaMemcpyDeviceToHost, sh.s));
      NNB_CUDA(cudaEventCreateWithFlags(&nest_done[k], cudaEventDisableTiming));
      NNB_CUDA(cudaEventRecord(nest_done[k], sh.s));
    }
  }
  NNB_CUDA(cudaEventRecord(e1, sh.s));
  NNB_CUDA(cudaMemcpyAsync(eps_h.data(), eps_dev, sizeof(double) * slots, cudaMemcpyDeviceToHost,
                           sh.s));
  NNB_CUDA(cudaMemcpyAsync(nf_h.data(), nf_dev, sizeof(int) * nf_count, cudaMemcpyDeviceToHost,
                           sh.s));
  NNB_CUDA(cudaStreamSynchronize(sh.s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (eps_hist)
    for (int q = 0; q < recorded; ++q) eps_hist[q] = eps_h[q];
  out->iters = std::min(k, cfg.max_iters);
  out->products = products;
  out->stopped = stopped;
  out->last_eps = recorded ? eps_h[recorded - 1] : 0.0;
  out->device_ms = ms;
  out->fail_iter = 0;
  // the final iterate lives in XF[cur]; the caller copies it out
  out->x_index = cur;
  for (int kk = 0; kk <= out->iters && kk < slots; ++kk)
    for (int j = 0; j <= p; ++j) {
      if (!nf_h[kk * (p + 1) + j]) continue;
      if (j == 0) return fail(NNB_ERR_DOMAIN, "sharded chain: residual product went non-finite at nest " + std::to_string(kk));
      out->fail_iter = kk + 1;
      return fail(NNB_ERR_DIVERGENCE, "sharded chain: non-finite iterate at nest " + std::to_string(kk + 1));
    }
  return 0;
}

}  // namespace
}  // namespace nnb

using namespace nnb;

extern "C" {

void nnb_partition_rows(int64_t n, int32_t world, int32_t rank, int64_t* row0, int64_t* rows) {
  std::vector<int64_t> r0, rs;
  partition(n, world < 1 ? 1 : world, r0, rs);
  const int g = rank < 0 ? 0 : (rank >= world ? world - 1 : rank);
  if (row0) *row0 = r0[g];
  if (rows) *rows = rs[g];
}

int nnb_comm_unique_id(void* id_out) {
  auto& api = nccl();
  if (!api.ok) return fail(NNB_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NNB_NCCL(api.getUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == NNB_UNIQUE_ID_BYTES, "unique id size");
  std::memcpy(id_out, &id, sizeof(id));
  return 0;
}

int nnb_comm_init(const void* id, int32_t world, int32_t rank, nnb_comm_t* comm_out) {
  NNB_TRY(require_device());
  auto& api = nccl();
  if (!api.ok) return fail(NNB_ERR_NCCL, "libnccl.so.2 could not be loaded");
  if (world < 1 || rank < 0 || rank >= world) return fail(NNB_ERR_DOMAIN, "comm: bad rank/world");
  auto* c = new nnb_comm();
  c->world = world;
  c->rank = rank;
  cudaGetDevice(&c->device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclResult_t r = api.commInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(NNB_ERR_NCCL, std::string("ncclCommInitRank: ") + api.errorString(r));
  }
  // The ring's send/recv kernels must not queue behind a 1-CTA-per-SM GEMM grid:
  // the block scheduler dispatches pending CTAs of the highest-priority stream first
  // as SMs free up, so the communication stream gets the greatest priority.
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  if (cudaStreamCreateWithPriority(&c->cs, cudaStreamNonBlocking, greatest) != cudaSuccess) {
    api.commDestroy(c->comm);
    delete c;
    return fail(NNB_ERR_CUDA, "comm: communication stream");
  }
  *comm_out = c;
  return 0;
}

int nnb_comm_destroy(nnb_comm_t comm) {
  if (!comm) return 0;
  if (comm->comm) nccl().commDestroy(comm->comm);
  if (comm->cs) cudaStreamDestroy(comm->cs);
  delete comm;
  return 0;
}

// the sharded products take the int8 emulation exactly where the single-GPU chain's
// products of the whole matrices would (engine.cu gemm())
static bool use_ozaki(int64_t n) {
  return n <= 131071 && (arith() == 2 || (arith() == 0 && ozaki_pays(n, n, n)));
}

static int chain_cfg_sharded(const nnb_chain_config* cfg, ChainCfg* c) {
  if (!cfg) return fail(NNB_ERR_DOMAIN, "sharded chain: config is NULL");
  if (cfg->depth_p < 0 || cfg->max_iters < 0) return fail(NNB_ERR_DOMAIN, "sharded chain: bad depth/budget");
  c->p = cfg->depth_p;
  c->max_iters = cfg->max_iters;
  c->tol = cfg->tol;
  c->order = cfg->order;
  c->final_residual = cfg->final_residual;
  return 0;
}

static void fill(nnb_chain_result* r, const ChainOut& o) {
  if (!r) return;
  r->iters = o.iters;
  r->fail_iter = o.fail_iter;
  r->stopped = o.stopped;
  r->products = o.products;
  r->last_eps = o.last_eps;
  r->device_ms = o.device_ms;
}

int nnb_nn_chain_sharded_d(nnb_comm_t comm, const double* A_rows, int64_t n, const double* X0_rows,
                           const nnb_chain_config* cfg, double* X_rows_out, double* eps_hist,
                           nnb_chain_result* result, void* stream) {
  NNB_TRY(require_device());
  if (!comm) return fail(NNB_ERR_DOMAIN, "sharded chain: comm is NULL");
  if (n < 1) return fail(NNB_ERR_SHAPE, "sharded chain: n must be >= 1");
  ChainCfg c;
  NNB_TRY(chain_cfg_sharded(cfg, &c));
  if (cfg->order != NNB_ORDER_NORTHSTAR)
    return fail(NNB_ERR_DOMAIN, "sharded chain: only the row-sharded NORTHSTAR order is supported");
  Shard sh;
  sh.n = n;
  sh.ld = pad8(n);
  sh.world = comm->world;
  sh.comm = comm;
  sh.local = {comm->rank};
  sh.s = resolve(stream);
  partition(n, sh.world, sh.row0, sh.rows);
  const int me = comm->rank;
  const int64_t ld = sh.ld, rows = sh.rows[me], row0 = sh.row0[me];
  sh.ev.resize(sh.world);
  for (auto& e : sh.ev) NNB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  NNB_CUDA(cudaEventCreateWithFlags(&sh.ready, cudaEventDisableTiming));

  DevBuf big;  // A_g | XF0 | XF1 | RF | V0 | V1
  const size_t full = (size_t)n * ld, blk = (size_t)std::max<int64_t>(rows, 1) * ld;
  NNB_TRY(big.alloc(sizeof(double) * (3 * full + 3 * blk), sh.s));
  double* Ag = big.as<double>();
  double* XF0 = Ag + blk;
  double* XF1 = XF0 + full;
  double* RF = XF1 + full;
  double* V = RF + full;
  if (rows)
    NNB_CUDA(cudaMemcpy2DAsync(Ag, ld * 8, A_rows, n * 8, n * 8, rows, cudaMemcpyDefault, sh.s));
  double* Xg = XF0 + row0 * ld;
  switch (cfg->x0_kind) {
    case NNB_X0_GIVEN:
      if (!X0_rows) return fail(NNB_ERR_DOMAIN, "sharded chain: X0 required");
      if (rows)
        NNB_CUDA(cudaMemcpy2DAsync(Xg, ld * 8, X0_rows, n * 8, n * 8, rows, cudaMemcpyDefault, sh.s));
      break;
    case NNB_X0_SCALED_IDENTITY:
      NNB_TRY(axpby(0.0, Xg, ld, 0.0, nullptr, 0, cfg->x0_scale, row0, Xg, ld, rows, n, sh.s));
      break;
    case NNB_X0_JACOBI:
      jacobi_rows_kernel<<<1184, 256, 0, sh.s>>>(Ag, ld, rows, row0, n, Xg, ld);
      count_launch();
      break;
    case NNB_X0_TRANSPOSE_NORM: {
      // gather A into RF (free before the first nest), build the full X0 in XF1, keep our rows
      NNB_TRY(copy2d(Ag, ld, RF + row0 * ld, ld, rows, n, sh.s));
      NNB_TRY(ring_allgather(sh, RF));
      if (sh.world > 1) NNB_CUDA(cudaStreamWaitEvent(sh.s, sh.ev[sh.world - 1], 0));
      NNB_TRY(x0_build(RF, ld, n, NNB_X0_TRANSPOSE_NORM, 1.0, XF1, ld, sh.s));
      NNB_TRY(copy2d(XF1 + row0 * ld, ld, Xg, ld, rows, n, sh.s));
      break;
    }
    default:
      return fail(NNB_ERR_DOMAIN, "sharded chain: unknown X0 kind");
  }
  OzSh ozs;
  OzSh* oz = nullptr;
  if (use_ozaki(n)) {
    NNB_TRY(oz_init(sh, ozs));
    oz = &ozs;
  }
  ChainOut o;
  const int st = run_sharded(sh, Ag, ld, false, XF0, XF1, RF, V, c, eps_hist, &o, oz);
  fill(result, o);
  for (auto& e : sh.ev) cudaEventDestroy(e);
  cudaEventDestroy(sh.ready);
  if (st != 0 && st != NNB_ERR_DIVERGENCE && st != NNB_ERR_DOMAIN) return st;
  double* xf = o.x_index ? XF1 : XF0;
  if (rows)
    NNB_CUDA(cudaMemcpy2DAsync(X_rows_out, n * 8, xf + row0 * ld, ld * 8, n * 8, rows,
                               cudaMemcpyDefault, sh.s));
  NNB_CUDA(cudaStreamSynchronize(sh.s));
  return st;
}

int nnb_nn_chain_sharded_emulated_d(const double* A, int64_t n, int32_t world, const double* X0,
                                    const nnb_chain_config* cfg, double* X_out, double* eps_hist,
                                    nnb_chain_result* result, void* stream) {
  NNB_TRY(require_device());
  if (n < 1 || world < 1) return fail(NNB_ERR_SHAPE, "sharded emulation: bad n/world");
  ChainCfg c;
  NNB_TRY(chain_cfg_sharded(cfg, &c));
  if (cfg->order != NNB_ORDER_NORTHSTAR)
    return fail(NNB_ERR_DOMAIN, "sharded chain: only the row-sharded NORTHSTAR order is supported");
  Shard sh;
  sh.n = n;
  sh.ld = pad8(n);
  sh.world = world;
  sh.s = resolve(stream);
  partition(n, world, sh.row0, sh.rows);
  for (int g = 0; g < world; ++g) sh.local.push_back(g);
  sh.ev.resize(world);
  const int64_t ld = sh.ld;
  const size_t full = (size_t)n * ld;
  DevBuf big;  // A | XF0 | XF1 | RF | V0 | V1 (full-size, sliced per virtual rank)
  NNB_TRY(big.alloc(sizeof(double) * 6 * full, sh.s));
  double* Af = big.as<double>();
  double* XF0 = Af + full;
  double* XF1 = XF0 + full;
  double* RF = XF1 + full;
  double* V = RF + full;
  NNB_CUDA(cudaMemcpy2DAsync(Af, ld * 8, A, n * 8, n * 8, n, cudaMemcpyDefault, sh.s));
  if (cfg->x0_kind == NNB_X0_GIVEN) {
    if (!X0) return fail(NNB_ERR_DOMAIN, "sharded emulation: X0 required");
    NNB_CUDA(cudaMemcpy2DAsync(XF0, ld * 8, X0, n * 8, n * 8, n, cudaMemcpyDefault, sh.s));
  } else {
    NNB_TRY(x0_build(Af, ld, n, cfg->x0_kind, cfg->x0_scale, XF0, ld, sh.s));
  }
  OzSh ozs;
  OzSh* oz = nullptr;
  if (use_ozaki(n)) {
    NNB_TRY(oz_init(sh, ozs));
    oz = &ozs;
  }
  ChainOut o;
  const int st = run_sharded(sh, Af, ld, true, XF0, XF1, RF, V, c, eps_hist, &o, oz);
  fill(result, o);
  if (st != 0 && st != NNB_ERR_DIVERGENCE && st != NNB_ERR_DOMAIN) return st;
  NNB_CUDA(cudaMemcpy2DAsync(X_out, n * 8, o.x_index ? XF1 : XF0, ld * 8, n * 8, n,
                             cudaMemcpyDefault, sh.s));
  NNB_CUDA(cudaStreamSynchronize(sh.s));
  return st;
}

}  // extern "C"
