// ORACLE — test infrastructure only.  Never linked into the product library.
//
// A thin extern "C" harness over the UNMODIFIED reference sources compiled in
// place from /root/reference/proj/src (see oracle/Makefile).  It lets the
// pytest parity suite, the golden-fixture generator and bench.py's
// cpu_baseline / --impl reference legs drive the reference's own C++ API
// through ctypes.  Every entry point calls the reference function it names;
// the only logic here is marshalling (interleaved complex128 <-> nn::DenseMatrix)
// and the driver loop of SURVEY.md §8(c), which mirrors
// /root/reference/proj/src/solver.cpp:138-159 for an explicit X0.
#include <algorithm>
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "nn/errors.hpp"
#include "nn/factorized.hpp"
#include "nn/kernels.hpp"
#include "nn/normalization.hpp"
#include "nn/rng.hpp"
#include "nn/solver.hpp"
#include "nn/sparse_csr.hpp"

using nn::DenseMatrix;
using nn::Scalar;

namespace {

thread_local std::string g_err;

enum Status {
  kOk = 0, kShape = 1, kDomain = 2, kDivergence = 3, kContraction = 4,
  kPlan = 5, kBudget = 6, kOther = 99
};

DenseMatrix load(const double* p, std::size_t r, std::size_t c) {
  std::vector<Scalar> v(r * c);
  std::memcpy(v.data(), p, sizeof(Scalar) * r * c);
  return DenseMatrix(r, c, std::move(v));
}

void store(const DenseMatrix& m, double* out) {
  std::memcpy(out, m.data().data(), sizeof(Scalar) * m.size());
}

template <class Fn>
int guarded(Fn&& fn, int* fail_index = nullptr) {
  try {
    fn();
    return kOk;
  } catch (const nn::DivergenceError& e) {
    g_err = e.what();
    if (fail_index) *fail_index = static_cast<int>(e.nest_index);
    return kDivergence;
  } catch (const nn::ContractionError& e) {
    g_err = e.what(); return kContraction;
  } catch (const nn::PlanError& e) {
    g_err = e.what(); return kPlan;
  } catch (const nn::BudgetError& e) {
    g_err = e.what(); return kBudget;
  } catch (const nn::ShapeError& e) {
    g_err = e.what(); return kShape;
  } catch (const nn::DomainError& e) {
    g_err = e.what(); return kDomain;
  } catch (const std::exception& e) {
    g_err = e.what(); return kOther;
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// SURVEY §8(c) driver: eps = residual_epsilon(X, A); record; stop on tol or
// count; X = nn_step(X, A, p) — the body of nn_invert
// (/root/reference/proj/src/solver.cpp:138-159) with an explicit X0, theta=1.
int chain(const DenseMatrix& a, DenseMatrix& x, int p, int max_iters, double tol,
          double* eps_hist, int* iters_out, int* fail_iter) {
  int it = 0;
  while (true) {
    const double eps = nn::residual_epsilon(x, a);
    if (eps_hist) eps_hist[it] = eps;
    if (tol > 0.0 && eps < tol) break;
    if (it >= max_iters) break;
    try {
      x = nn::nn_step(x, a, static_cast<std::size_t>(p));
    } catch (const nn::DomainError&) {
      throw nn::DivergenceError("chain: non-finite iterate at nest " + std::to_string(it + 1),
                                static_cast<std::size_t>(it + 1));
    }
    ++it;
  }
  if (iters_out) *iters_out = it;
  return kOk;
}

}  // namespace

extern "C" {

const char* nnref_last_error() { return g_err.c_str(); }

unsigned nnref_worker_count() { return nn::worker_count(); }

// nn::GaussianStream (proj/include/nn/rng.hpp:15-52): n draws from seed.
void nnref_gaussian(uint64_t seed, int64_t n, double* out) {
  nn::GaussianStream g(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = g.next();
}

// nn::random_spd (proj/src/kernels.cpp:352-381); complex128 interleaved out.
int nnref_random_spd(int64_t n, double cond, uint64_t seed, double* out) {
  return guarded([&] { store(nn::random_spd(static_cast<std::size_t>(n), cond, seed), out); });
}

// nn::direct_inverse_oracle (proj/src/kernels.cpp:317-350); pivot index on SingularMatrixError (status 11).
int nnref_direct_inverse_z(const double* m, int64_t n, double* out, int* pivot) {
  try {
    store(nn::direct_inverse_oracle(load(m, n, n)), out);
    return kOk;
  } catch (const nn::SingularMatrixError& e) {
    g_err = e.what();
    *pivot = static_cast<int>(e.pivot_index);
    return 11;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kOther;
  }
}

// nn::random_conditioned_complex (proj/src/kernels.cpp:383-407).
int nnref_random_conditioned_complex(int64_t n, double cond, uint64_t seed, double* out) {
  return guarded([&] { store(nn::random_conditioned_complex(static_cast<std::size_t>(n), cond, seed), out); });
}

// nn::random_sparse_spd (proj/src/kernels.cpp:409-432) as CSR arrays; nnz_out
// first (call with row_ptr == nullptr to size the buffers).
int nnref_random_sparse_spd(int64_t n, double density, uint64_t seed, int64_t* nnz_out, int64_t* row_ptr,
                            int64_t* col, double* val) {
  return guarded([&] {
    const nn::SparseMatrixCsr m = nn::random_sparse_spd(static_cast<std::size_t>(n), density, seed);
    *nnz_out = static_cast<int64_t>(m.nnz());
    if (!row_ptr) return;
    for (std::size_t i = 0; i <= m.rows(); ++i) row_ptr[i] = static_cast<int64_t>(m.row_ptr()[i]);
    for (std::size_t k = 0; k < m.nnz(); ++k) {
      col[k] = static_cast<int64_t>(m.col_idx()[k]);
      val[k] = m.values()[k].real();
    }
  });
}

// nn::matmul (proj/src/kernels.cpp:137-162).
int nnref_matmul_z(const double* a, const double* b, int64_t m, int64_t k, int64_t n,
                   double* c, double* n3) {
  return guarded([&] {
    nn::OpCounter cnt;
    store(nn::matmul(load(a, m, k), load(b, k, n), &cnt), c);
    if (n3) *n3 = cnt.n3_multiplies();
  });
}

// nn::residual_epsilon (proj/src/solver.cpp:72-75).
int nnref_residual_eps_z(const double* x, const double* a, int64_t n, double* eps) {
  return guarded([&] { *eps = nn::residual_epsilon(load(x, n, n), load(a, n, n)); });
}

// nn::frobenius_norm (proj/src/kernels.cpp:238-242) and nn::trace (:231-236).
int nnref_frobenius_z(const double* m, int64_t r, int64_t c, double* out) {
  return guarded([&] { *out = nn::frobenius_norm(load(m, r, c)); });
}
int nnref_trace_z(const double* m, int64_t n, double* out2) {
  return guarded([&] {
    const Scalar t = nn::trace(load(m, n, n));
    out2[0] = t.real(); out2[1] = t.imag();
  });
}

// Elementwise kernels (proj/src/kernels.cpp:175-221); op: 0 add, 1 sub,
// 2 scale(by s), 3 identity_minus, 4 plus_identity.
int nnref_elementwise_z(int op, const double* a, const double* b, int64_t r, int64_t c,
                        double sre, double sim, double* out, int64_t* n2) {
  return guarded([&] {
    nn::OpCounter cnt;
    const DenseMatrix ma = load(a, r, c);
    DenseMatrix o;
    switch (op) {
      case 0: o = nn::add(ma, load(b, r, c), &cnt); break;
      case 1: o = nn::sub(ma, load(b, r, c), &cnt); break;
      case 2: o = nn::scale(ma, Scalar{sre, sim}, &cnt); break;
      case 3: o = nn::identity_minus(ma, &cnt); break;
      default: o = nn::plus_identity(ma, &cnt); break;
    }
    store(o, out);
    if (n2) *n2 = cnt.n2_ops();
  });
}

// nn::nn_step (proj/src/solver.cpp:93-103) / newton_step (:105-111) /
// chebyshev_step (:113-121); which: 0 nn_step(L), 1 newton, 2 chebyshev.
int nnref_step_z(int which, const double* x, const double* a, int64_t n, int64_t depth_l,
                 double* out, double* n3) {
  return guarded([&] {
    nn::OpCounter cnt;
    const DenseMatrix mx = load(x, n, n), ma = load(a, n, n);
    DenseMatrix o = which == 1 ? nn::newton_step(mx, ma, &cnt)
                  : which == 2 ? nn::chebyshev_step(mx, ma, &cnt)
                               : nn::nn_step(mx, ma, static_cast<std::size_t>(depth_l), &cnt);
    store(o, out);
    if (n3) *n3 = cnt.n3_multiplies();
  });
}

// nn::ns_sum (proj/src/solver.cpp:77-91).
int nnref_ns_sum_z(const double* x0, const double* a, int64_t n, int64_t order, double* out,
                   double* n3) {
  return guarded([&] {
    nn::OpCounter cnt;
    store(nn::ns_sum(load(x0, n, n), load(a, n, n), static_cast<std::size_t>(order), &cnt), out);
    if (n3) *n3 = cnt.n3_multiplies();
  });
}

// SURVEY §8(c) explicit-X0 chain over the reference's nn_step/residual_epsilon.
// eps_hist needs max_iters+1 slots.  seconds = solver loop only.
int nnref_chain_z(const double* a, int64_t n, const double* x0, int p, int max_iters,
                  double tol, double* x_out, double* eps_hist, int* iters_out,
                  int* fail_iter, double* seconds) {
  return guarded([&] {
    const DenseMatrix ma = load(a, n, n);
    DenseMatrix x = load(x0, n, n);
    const double t0 = now_s();
    chain(ma, x, p, max_iters, tol, eps_hist, iters_out, fail_iter);
    if (seconds) *seconds = now_s() - t0;
    store(x, x_out);
  }, fail_iter);
}

// nn::solve_normal_equations (proj/src/factorized.cpp:63-99) on a dense n×n A
// and n×k B.  Returns 20 (with the report's history and counts filled) when
// the reference raises NonConvergenceError.
int nnref_solve_normal_z(const double* a, int64_t n, const double* b, int64_t k, int64_t depth_l,
                         int64_t max_nests, double tol, double* x_out, double* hist, int64_t* hist_len,
                         double* counts, int* stop_reason, double* backward, int* fail_iter) {
  int nonconv = 0;
  const int st = guarded([&] {
    nn::SolverConfig cfg;
    cfg.depth_L = static_cast<std::size_t>(depth_l);
    cfg.max_nests = static_cast<std::size_t>(max_nests);
    cfg.tol = tol;
    nn::OpCounter cnt;
    auto report_out = [&](const nn::ConvergenceReport& rep) {
      for (std::size_t i = 0; i < rep.history.size(); ++i) hist[i] = rep.history[i].second;
      *hist_len = static_cast<int64_t>(rep.history.size());
      *stop_reason = rep.stopped_reason == nn::StopReason::Tolerance ? 0 : 1;
    };
    try {
      nn::LinearSystem sys{load(a, n, n), load(b, n, k), false};
      auto res = nn::solve_normal_equations(sys, cfg, &cnt);
      store(res.x, x_out);
      report_out(res.report);
      *backward = res.backward_error;
    } catch (const nn::NonConvergenceError& e) {
      report_out(e.report);
      nonconv = 1;
    }
    counts[0] = cnt.n3_multiplies();
    counts[1] = static_cast<double>(cnt.n2_ops());
  }, fail_iter);
  return st == kOk && nonconv ? 20 : st;
}

// nn::nn_invert (proj/src/solver.cpp:123-174) with an explicit Normalization.
// hist gets (eps) per recorded nest; counts[0]=n3, counts[1]=n2.
int nnref_nn_invert_z(const double* w, int64_t n, double theta, int valid, int64_t depth_l,
                      int64_t max_nests, double tol, double* x_out, double* hist,
                      int64_t* hist_len, double* counts, int* stop_reason,
                      double* alpha, int* fail_iter) {
  return guarded([&] {
    nn::Normalization norm;
    norm.theta = theta;
    norm.valid = valid != 0;
    nn::SolverConfig cfg;
    cfg.depth_L = static_cast<std::size_t>(depth_l);
    cfg.max_nests = static_cast<std::size_t>(max_nests);
    cfg.tol = tol;
    nn::OpCounter cnt;
    auto [x, rep] = nn::nn_invert(load(w, n, n), norm, cfg, &cnt);
    store(x, x_out);
    for (std::size_t i = 0; i < rep.history.size(); ++i) hist[i] = rep.history[i].second;
    *hist_len = static_cast<int64_t>(rep.history.size());
    counts[0] = rep.n3_multiplies;
    counts[1] = static_cast<double>(rep.n2_ops);
    *stop_reason = rep.stopped_reason == nn::StopReason::Tolerance ? 0 : 1;
    *alpha = rep.alpha_estimate ? *rep.alpha_estimate : -1.0;
  }, fail_iter);
}

// nn::theta_trace (proj/src/normalization.cpp:35-41).
int nnref_theta_trace_z(const double* w, int64_t n, double* theta, double* contraction,
                        int* valid) {
  return guarded([&] {
    const nn::Normalization nm = nn::theta_trace(load(w, n, n));
    *theta = nm.theta; *contraction = nm.contraction_norm; *valid = nm.valid ? 1 : 0;
  });
}

// Batched C2 leg: per-system §8(c) chain (Jacobi X0 = diag(A)^-1) or the
// ns_sum baseline, systems split across `threads` std::threads (the
// reference functions are re-entrant).  mode 0: NN chain with
// `iters` nests of depth p; mode 1: ns_sum of order `iters` from the same X0.
// eps_last: residual after the final nest (mode 0 only).
int nnref_batched_z(int mode, const double* a, int64_t batch, int64_t n, int p, int iters,
                    double* x_out, double* eps_last, int threads, double* seconds) {
  return guarded([&] {
    const int nt = std::max(1, threads);
    std::vector<std::thread> pool;
    std::vector<std::string> errs(nt);
    const double t0 = now_s();
    for (int t = 0; t < nt; ++t) {
      pool.emplace_back([&, t] {
        try {
          for (int64_t s = t; s < batch; s += nt) {
            const DenseMatrix ma = load(a + 2 * s * n * n, n, n);
            std::vector<Scalar> d(n);
            for (int64_t i = 0; i < n; ++i) d[i] = Scalar{1.0, 0.0} / ma(i, i);
            DenseMatrix x = DenseMatrix::diagonal(d);
            if (mode == 0) {
              std::vector<double> hist(iters + 1);
              chain(ma, x, p, iters, 0.0, hist.data(), nullptr, nullptr);
              if (eps_last) eps_last[s] = hist[iters];
            } else {
              x = nn::ns_sum(x, ma, static_cast<std::size_t>(iters));
            }
            store(x, x_out + 2 * s * n * n);
          }
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    if (seconds) *seconds = now_s() - t0;
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// CSR helpers: the reference CSR is built only through SparseMatrixCsr::build
// (proj/src/sparse_csr.cpp:7-40); values are real here (C5 is real).
static nn::SparseMatrixCsr csr_from(const int64_t* row_ptr, const int32_t* col,
                                    const double* val, int64_t n) {
  std::vector<nn::SparseMatrixCsr::Triplet> t;
  t.reserve(static_cast<std::size_t>(row_ptr[n]));
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k)
      t.push_back({static_cast<std::size_t>(r), static_cast<std::size_t>(col[k]),
                   Scalar{val[k], 0.0}});
  return nn::SparseMatrixCsr::build(static_cast<std::size_t>(n), static_cast<std::size_t>(n),
                                    std::move(t));
}

// nn::spmv_block (proj/src/kernels.cpp:454-471); x, out complex n×k.
int nnref_spmv_block(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                     const double* x, int64_t k, double* out) {
  return guarded([&] {
    store(nn::spmv_block(csr_from(row_ptr, col, val, n), load(x, n, k)), out);
  });
}

// nn::solve_sparse_factorized (proj/src/factorized.cpp:101-140) with an
// explicit valid Normalization{theta}; b/x complex n×k.  counts[0] = spmv_count.
int nnref_sparse_factorized(const int64_t* row_ptr, const int32_t* col, const double* val,
                            int64_t n, const double* b, int64_t k, int64_t gamma, double theta,
                            double* x_out, double* counts, double* seconds, int* fail_index) {
  return guarded([&] {
    nn::LinearSystem sys{csr_from(row_ptr, col, val, n), load(b, n, k), false};
    nn::Normalization norm;
    norm.theta = theta;
    norm.valid = true;
    nn::OpCounter cnt;
    const double t0 = now_s();
    const DenseMatrix x = nn::solve_sparse_factorized(sys, nn::BigInt(gamma), norm, &cnt);
    if (seconds) *seconds = now_s() - t0;
    store(x, x_out);
    if (counts) counts[0] = static_cast<double>(cnt.spmv_count());
  }, fail_index);
}

// nn::ns_factorized (proj/src/factorized.cpp:42-61), nn::power_ladder
// (proj/src/kernels.cpp:434-452), nn::nn_explicit (proj/src/solver.cpp:176-199).
int nnref_ns_factorized_z(const double* phi0, const double* w, int64_t n, int64_t gamma, double* out,
                          double* n3) {
  return guarded([&] {
    nn::OpCounter cnt;
    const auto plan = nn::FactorizedPlan::for_order(nn::BigInt(gamma), nn::FactorizedMode::DenseStored);
    store(nn::ns_factorized(load(phi0, n, n), load(w, n, n), plan, &cnt), out);
    if (n3) *n3 = cnt.n3_multiplies();
  });
}
int nnref_power_ladder_z(const double* p, int64_t n, uint64_t e, double* out, double* n3) {
  return guarded([&] {
    nn::OpCounter cnt;
    store(nn::power_ladder(load(p, n, n), e, &cnt), out);
    if (n3) *n3 = cnt.n3_multiplies();
  });
}
int nnref_nn_explicit_z(const double* phi0, const double* w, int64_t n, int64_t nests, int64_t depth,
                        double* out, double* n3) {
  return guarded([&] {
    nn::OpCounter cnt;
    store(nn::nn_explicit(load(phi0, n, n), load(w, n, n), static_cast<std::size_t>(nests),
                          static_cast<std::size_t>(depth), &cnt),
          out);
    if (n3) *n3 = cnt.n3_multiplies();
  });
}

// nn::equivalent_ns_order (proj/src/solver.cpp:201-205), saturating.
uint64_t nnref_equivalent_ns_order(int64_t nests, int64_t depth) {
  const auto v = nn::equivalent_ns_order(static_cast<std::size_t>(nests),
                                         static_cast<std::size_t>(depth));
  return static_cast<unsigned long long>(v);
}

}  // extern "C"
