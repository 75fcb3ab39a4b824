// Shared pieces of the single-GPU and row-sharded sparse factorized solves.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace nnb {

enum SpmvMode { kInner = 0, kFactorEnd = 1, kFinal = 2 };

// One application t_out = t_in − θ·W·t_in (+ factor update / final scale by mode).
template <typename Idx>
struct SpmvOp {
  const Idx* rp;        // row offsets of the rows this call owns (local, from 0)
  const int32_t* col;   // column indices into t_ext
  const double* val;
  int64_t k;            // right-hand sides
  const double* t_ext;  // gather base (own rows, plus halo rows around them when sharded)
  const double* t_own;  // t_in indexed by owned row
  double* out;          // indexed by owned row
  const double* zold;   // indexed by owned row (factor end / final)
  double theta;
  int* flag;            // non-finite flag of this factor
};

template <typename Idx>
void spmv_apply(const SpmvOp<Idx>& op, int mode, int64_t r_begin, int64_t r_end, cudaStream_t s);

int narrow_offsets(const int64_t* in, int32_t* out, int64_t count, int64_t base, cudaStream_t s);

}  // namespace nnb
