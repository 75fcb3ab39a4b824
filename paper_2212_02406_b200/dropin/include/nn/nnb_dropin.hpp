// B200 drop-in for the reference's hot-path C++ API (namespace nn).
//
// Source-compatible with /root/reference/proj/include/nn/*.hpp for the
// functions on the Nested Neumann hot path: the same
// types, signatures, default arguments, exception classes and OpCounter
// tallies, with every matrix operation executed by libnnb.so on the GPU
// (include/nnb.h).  Host code here only marshals DenseMatrix/CSR objects,
// synthesises the reference's operation counts and keeps the host-side
// bookkeeping (reports, nest estimates, order fits).
//
// Out of scope (not declared; link the reference's nncore for it): the exact
// rational cost model (analytic only).
#pragma once

#include <atomic>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <optional>
#include <random>
#include <stdexcept>
#include <type_traits>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#if __has_include(<boost/multiprecision/cpp_int.hpp>)
#include <boost/multiprecision/cpp_int.hpp>
#define NN_DROPIN_HAVE_BOOST 1
#endif

namespace nn {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define NN_DROPIN_PLAIN_ERROR(Name) \
  struct Name : Error {             \
    using Error::Error;             \
  }
NN_DROPIN_PLAIN_ERROR(ShapeError);
NN_DROPIN_PLAIN_ERROR(DomainError);
NN_DROPIN_PLAIN_ERROR(NotPsdError);
NN_DROPIN_PLAIN_ERROR(DegenerateProbeError);
NN_DROPIN_PLAIN_ERROR(ContractionError);
NN_DROPIN_PLAIN_ERROR(PlanError);
NN_DROPIN_PLAIN_ERROR(BudgetError);
NN_DROPIN_PLAIN_ERROR(EstimationError);
NN_DROPIN_PLAIN_ERROR(IoError);
#undef NN_DROPIN_PLAIN_ERROR

struct SingularMatrixError : Error {
  SingularMatrixError(const std::string& what, std::size_t pivot) : Error(what), pivot_index(pivot) {}
  std::size_t pivot_index;
};

struct DivergenceError : Error {
  DivergenceError(const std::string& what, std::size_t nest) : Error(what), nest_index(nest) {}
  std::size_t nest_index;
};

// ------------------------------------------------------------------ scalars / BigInt
using Scalar = std::complex<double>;

#ifdef NN_DROPIN_HAVE_BOOST
using BigInt = boost::multiprecision::cpp_int;
#else
// Exact unsigned 128-bit stand-in when Boost.Multiprecision is not installed:
// covers every order the hot path can apply (gamma <= 2^30, nests such that
// (L+1)^(i+1) < 2^128); arithmetic saturates instead of overflowing.
class BigInt {
 public:
  using rep = unsigned __int128;
  BigInt() = default;
  template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
  BigInt(I v) : v_(v < I{} ? rep(0) : rep(v)) {}
  static BigInt raw(rep v) { BigInt b; b.v_ = v; return b; }
  rep value() const { return v_; }
  explicit operator std::size_t() const { return static_cast<std::size_t>(v_); }
  explicit operator unsigned long long() const { return static_cast<unsigned long long>(v_); }
  std::string str() const;
  friend BigInt operator+(BigInt a, BigInt b) { return raw(a.v_ > ~rep(0) - b.v_ ? ~rep(0) : a.v_ + b.v_); }
  friend BigInt operator-(BigInt a, BigInt b) { return raw(a.v_ < b.v_ ? 0 : a.v_ - b.v_); }
  friend BigInt operator*(BigInt a, BigInt b) {
    return raw(a.v_ && b.v_ > ~rep(0) / a.v_ ? ~rep(0) : a.v_ * b.v_);
  }
  friend BigInt operator&(BigInt a, BigInt b) { return raw(a.v_ & b.v_); }
  friend BigInt operator<<(BigInt a, int s) { return raw(s >= 128 ? 0 : a.v_ << s); }
  friend bool operator==(BigInt a, BigInt b) { return a.v_ == b.v_; }
  friend bool operator!=(BigInt a, BigInt b) { return a.v_ != b.v_; }
  friend bool operator<(BigInt a, BigInt b) { return a.v_ < b.v_; }
  friend bool operator>(BigInt a, BigInt b) { return a.v_ > b.v_; }
  friend bool operator<=(BigInt a, BigInt b) { return a.v_ <= b.v_; }
  friend bool operator>=(BigInt a, BigInt b) { return a.v_ >= b.v_; }

 private:
  rep v_ = 0;
};
#endif

// ------------------------------------------------------------------ DenseMatrix
/// Row-major complex<double> matrix held on the host; purely real data is
/// carried with zero imaginary parts and routed to the real device kernels.
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(std::size_t rows, std::size_t cols) : r_(rows), c_(cols), v_(rows * cols) {}
  DenseMatrix(std::size_t rows, std::size_t cols, std::vector<Scalar> data);
  DenseMatrix(std::initializer_list<std::initializer_list<Scalar>> rows);

  static DenseMatrix identity(std::size_t n);
  static DenseMatrix diagonal(const std::vector<Scalar>& d);

  std::size_t rows() const { return r_; }
  std::size_t cols() const { return c_; }
  std::size_t size() const { return v_.size(); }
  bool square() const { return r_ == c_; }
  Scalar& operator()(std::size_t i, std::size_t j) { return v_[i * c_ + j]; }
  const Scalar& operator()(std::size_t i, std::size_t j) const { return v_[i * c_ + j]; }
  const std::vector<Scalar>& data() const { return v_; }
  std::vector<Scalar>& data() { return v_; }
  bool all_finite() const;
  bool is_identity() const;
  bool operator==(const DenseMatrix& o) const { return r_ == o.r_ && c_ == o.c_ && v_ == o.v_; }

 private:
  std::size_t r_ = 0, c_ = 0;
  std::vector<Scalar> v_;
};

// ------------------------------------------------------------------ OpCounter
/// Heavy-operation tally (n3 products, n2 passes, sparse applications);
/// atomic, shareable.  The device path fuses passes but reports the
/// reference's counts.
class OpCounter {
 public:
  OpCounter() = default;
  OpCounter(const OpCounter&) = delete;
  OpCounter& operator=(const OpCounter&) = delete;
  void add_n3(double units) { n3_.fetch_add(units, std::memory_order_relaxed); }
  void add_n2(std::int64_t k = 1) { n2_.fetch_add(k, std::memory_order_relaxed); }
  void add_spmv(std::int64_t k) { spmv_.fetch_add(k, std::memory_order_relaxed); }
  double n3_multiplies() const { return n3_.load(std::memory_order_relaxed); }
  std::int64_t n2_ops() const { return n2_.load(std::memory_order_relaxed); }
  std::int64_t spmv_count() const { return spmv_.load(std::memory_order_relaxed); }
  void reset() {
    n3_.store(0.0, std::memory_order_relaxed);
    n2_.store(0, std::memory_order_relaxed);
    spmv_.store(0, std::memory_order_relaxed);
  }

 private:
  std::atomic<double> n3_{0.0};
  std::atomic<std::int64_t> n2_{0};
  std::atomic<std::int64_t> spmv_{0};
};

// ------------------------------------------------------------------ GaussianStream
/// Seeded standard normals: mt19937_64, 53-bit uniforms, Box–Muller pairs
/// (cosine first, sine kept as the spare) — the reference's stream, so seeded
/// inputs are identical on both sides of the drop-in.
class GaussianStream {
 public:
  explicit GaussianStream(std::uint64_t seed) : eng_(seed) {}
  double next();
  std::vector<double> take(std::size_t n) {
    std::vector<double> out(n);
    for (auto& x : out) x = next();
    return out;
  }

 private:
  std::mt19937_64 eng_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

// ------------------------------------------------------------------ CSR
class SparseMatrixCsr {
 public:
  struct Triplet {
    std::size_t row;
    std::size_t col;
    Scalar value;
  };
  SparseMatrixCsr() = default;
  static SparseMatrixCsr build(std::size_t rows, std::size_t cols, std::vector<Triplet> triplets);
  static SparseMatrixCsr identity(std::size_t n);
  DenseMatrix densify() const;
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::size_t nnz() const { return val_.size(); }
  bool square() const { return rows_ == cols_; }
  const std::vector<std::size_t>& row_ptr() const { return ptr_; }
  const std::vector<std::size_t>& col_idx() const { return idx_; }
  const std::vector<Scalar>& values() const { return val_; }
  Scalar trace() const;

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<std::size_t> ptr_{0};
  std::vector<std::size_t> idx_;
  std::vector<Scalar> val_;
};

// ------------------------------------------------------------------ kernels
/// Number of CUDA devices visible (the device path has no CPU workers).
unsigned worker_count();
DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b, OpCounter* counter = nullptr);
DenseMatrix add(const DenseMatrix& a, const DenseMatrix& b, OpCounter* counter = nullptr);
DenseMatrix sub(const DenseMatrix& a, const DenseMatrix& b, OpCounter* counter = nullptr);
DenseMatrix scale(const DenseMatrix& m, Scalar factor, OpCounter* counter = nullptr);
DenseMatrix identity_minus(const DenseMatrix& m, OpCounter* counter = nullptr);
DenseMatrix plus_identity(const DenseMatrix& m, OpCounter* counter = nullptr);
DenseMatrix conjugate_transpose(const DenseMatrix& m, OpCounter* counter = nullptr);
/// Gauss–Jordan inverse with partial pivoting on the device (kernels.cpp:317-350):
/// the small-scale ground truth, bit-identical for real input; SingularMatrixError
/// with the pivot index when a pivot is <= 1e-13·||m||_F.
DenseMatrix direct_inverse_oracle(const DenseMatrix& m);
/// m·x on the device (kernels.cpp:164-173); untallied.
std::vector<Scalar> matvec(const DenseMatrix& m, const std::vector<Scalar>& x);
Scalar trace(const DenseMatrix& m);
double frobenius_norm(const DenseMatrix& m);

struct SpectralEstimate {
  double value = 0.0;
  bool converged = false;
  int iterations = 0;
};
SpectralEstimate spectral_norm_estimate(const DenseMatrix& m, double tol = 1e-12,
                                        int max_iters = 2000,
                                        std::uint64_t seed = 0x5eed5eedULL);
SpectralEstimate spectral_norm_estimate_shifted(const SparseMatrixCsr& w, Scalar theta,
                                                double tol = 1e-12, int max_iters = 2000,
                                                std::uint64_t seed = 0x5eed5eedULL);
/// Seeded test matrices of proj/include/nn/kernels.hpp:69-82.  random_spd and
/// random_conditioned_complex run the Householder QR and the products on the
/// GPU (random_spd bit-identical to the reference); random_sparse_spd is the
/// reference's sequential pattern/value stream on the host.
DenseMatrix random_spd(std::size_t n, double cond, std::uint64_t seed);
DenseMatrix random_conditioned_complex(std::size_t n, double cond, std::uint64_t seed);
SparseMatrixCsr random_sparse_spd(std::size_t n, double density, std::uint64_t seed);
DenseMatrix spmv_block(const SparseMatrixCsr& p, const DenseMatrix& x,
                       OpCounter* counter = nullptr);
/// p^exponent by square-and-multiply; floor(log2 e) + popcount(e) − 1 products.
DenseMatrix power_ladder(const DenseMatrix& p, std::uint64_t exponent, OpCounter* counter = nullptr);

// ------------------------------------------------------------------ normalization
enum class ThetaKind { TraceTheta1, PowerTheta2 };
struct Normalization {
  double theta = 0.0;
  ThetaKind kind = ThetaKind::TraceTheta1;
  std::size_t k_order = 0;
  double contraction_norm = 0.0;
  bool valid = false;
};
Normalization theta_trace(const DenseMatrix& w);
Normalization theta_trace(const SparseMatrixCsr& w);
/// theta = k / ((k+1)·r²), r the growth of k+1 normalised applications of W to a
/// GaussianStream probe (proj/src/normalization.cpp:51-92), every product on the GPU.
Normalization theta_power(const DenseMatrix& w, std::size_t k, std::uint64_t seed);
/// Measured ||I − phi·w_tilde||_2 (normalization.cpp:101-104); untallied.
double contraction_check(const DenseMatrix& phi, const DenseMatrix& w_tilde);
DenseMatrix normalize(const DenseMatrix& w, const Normalization& norm);

// ------------------------------------------------------------------ solver
struct SolverConfig {
  std::size_t depth_L = 2;
  std::size_t max_nests = 64;
  double tol = 1e-10;
  bool record_history = true;
};
struct NestState {
  DenseMatrix phi;
  std::size_t nest_index = 0;
  double epsilon = 0.0;
  std::optional<double> contraction;
};
enum class StopReason { Tolerance, MaxNests };
struct ConvergenceReport {
  SolverConfig config;
  std::vector<std::pair<std::size_t, double>> history;
  double n3_multiplies = 0.0;
  std::int64_t n2_ops = 0;
  std::int64_t spmv_count = 0;
  StopReason stopped_reason = StopReason::MaxNests;
  std::optional<double> alpha_estimate;
  std::optional<double> kappa_used;
};

std::string stop_reason_name(StopReason r);
std::string report_to_json(const ConvergenceReport& report);
double residual_epsilon(const DenseMatrix& phi, const DenseMatrix& w_tilde);
DenseMatrix ns_sum(const DenseMatrix& phi0, const DenseMatrix& w_tilde, std::size_t order,
                   OpCounter* counter = nullptr);
DenseMatrix nn_step(const DenseMatrix& phi, const DenseMatrix& w_tilde, std::size_t depth_L,
                    OpCounter* counter = nullptr);
DenseMatrix newton_step(const DenseMatrix& z, const DenseMatrix& w_tilde,
                        OpCounter* counter = nullptr);
DenseMatrix chebyshev_step(const DenseMatrix& z, const DenseMatrix& w_tilde,
                           OpCounter* counter = nullptr);
std::pair<DenseMatrix, ConvergenceReport> nn_invert(const DenseMatrix& w, const Normalization& norm,
                                                    const SolverConfig& config,
                                                    OpCounter* counter = nullptr);
DenseMatrix nn_explicit(const DenseMatrix& phi0, const DenseMatrix& w_tilde, std::size_t nests_i,
                        std::size_t depth_L, OpCounter* counter = nullptr);
BigInt equivalent_ns_order(std::size_t nests_i, std::size_t depth_L);
std::size_t estimate_nests(double kappa, std::size_t depth_L);
double convergence_order_estimate(const ConvergenceReport& report);

// ------------------------------------------------------------------ factorized (sparse path)
enum class FactorizedMode { DenseStored, SparseMatrixFree };
struct FactorizedPlan {
  BigInt gamma;
  std::size_t num_factors = 0;
  FactorizedMode mode = FactorizedMode::DenseStored;
  static FactorizedPlan for_order(const BigInt& gamma, FactorizedMode mode);
};
struct LinearSystem {
  std::variant<DenseMatrix, SparseMatrixCsr> a;
  DenseMatrix b;
  bool hermitian_normal = false;
};
struct CnsConfig {
  std::size_t ci_steps = 1;
  std::size_t ns_terms = 1;
  bool factorize_outer = false;
};
struct NonConvergenceError : Error {
  NonConvergenceError(const std::string& what, ConvergenceReport rep)
      : Error(what), report(std::move(rep)) {}
  ConvergenceReport report;
};
DenseMatrix ns_factorized(const DenseMatrix& phi, const DenseMatrix& w_tilde, const FactorizedPlan& plan,
                          OpCounter* counter = nullptr);
DenseMatrix solve_sparse_factorized(const LinearSystem& sys, const BigInt& gamma,
                                    const Normalization& norm, OpCounter* counter = nullptr);

/// Chebyshev–Neumann hybrid (proj/src/factorized.cpp:142-158): ci_steps
/// Chebyshev steps from I build the preconditioner, then an outer series of
/// ns_terms terms (product form when factorize_outer and ns_terms + 1 = 2^s).
/// Effective series order 3^ci_steps·(ns_terms + 1) − 1; every product on the GPU.
DenseMatrix cns_invert(const DenseMatrix& w_tilde, const CnsConfig& cns, OpCounter* counter = nullptr);

struct NormalSolveResult {
  DenseMatrix x;
  ConvergenceReport report;
  double backward_error = 0.0;  // ||W x - rhs||_F / ||rhs||_F on the normal equations
};
/// A x = B through W = A^H A (Hermitian PSD), theta_trace(W), nn_invert(W)
/// and x = W^-1 A^H B, every product on the GPU.
NormalSolveResult solve_normal_equations(const LinearSystem& sys, const SolverConfig& config,
                                         OpCounter* counter = nullptr);

}  // namespace nn
