// Implementation of the nn:: drop-in (nnb_dropin.hpp) over the libnnb C-ABI.
//
// Every matrix computation is a libnnb call (GPU); this file marshals
// DenseMatrix / SparseMatrixCsr objects, maps status codes to the
// reference's exception classes, and reproduces the reference's OpCounter
// tallies and report fields.  Each function names the reference routine it
// stands in for.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <functional>
#include <sstream>

#include "nn/nnb_dropin.hpp"
#include "nnb.h"

namespace nn {
namespace {

[[noreturn]] void raise(int st, const std::string& who, std::size_t index = 0) {
  const std::string msg = who + ": " + nnb_last_error();
  switch (st) {
    case NNB_ERR_SHAPE: throw ShapeError(msg);
    case NNB_ERR_DOMAIN: throw DomainError(msg);
    case NNB_ERR_DIVERGENCE: throw DivergenceError(msg, index);
    case NNB_ERR_CONTRACTION: throw ContractionError(msg);
    case NNB_ERR_PLAN: throw PlanError(msg);
    case NNB_ERR_BUDGET: throw BudgetError(msg);
    default: throw Error(msg);
  }
}

void check(int st, const std::string& who, std::size_t index = 0) {
  if (st != NNB_OK) raise(st, who, index);
}

bool real_valued(const DenseMatrix& m) {
  return std::all_of(m.data().begin(), m.data().end(), [](const Scalar& v) { return v.imag() == 0.0; });
}

std::vector<double> real_part(const DenseMatrix& m) {
  std::vector<double> out(m.size());
  std::transform(m.data().begin(), m.data().end(), out.begin(), [](const Scalar& v) { return v.real(); });
  return out;
}

DenseMatrix from_real(std::size_t r, std::size_t c, const std::vector<double>& v) {
  DenseMatrix m(r, c);
  for (std::size_t i = 0; i < v.size(); ++i) m.data()[i] = Scalar{v[i], 0.0};
  return m;
}

const double* zp(const DenseMatrix& m) { return reinterpret_cast<const double*>(m.data().data()); }
double* zp(DenseMatrix& m) { return reinterpret_cast<double*>(m.data().data()); }

// The reference tallies one n3 unit per product as it runs; replaying the
// fused device schedule's count the same way keeps the atomic double sum
// bit-identical when fractional (non-square) products are mixed in.
void add_products(OpCounter* counter, double count) {
  if (!counter) return;
  for (double i = 0.0; i < count; i += 1.0) counter->add_n3(1.0);
}

void require_finite(const DenseMatrix& m, const char* op) {
  if (!m.all_finite()) throw DomainError(std::string(op) + ": produced a non-finite entry");
}

// out = alpha*A + beta*B + gamma*I on the device, rounding like std::complex.
DenseMatrix axpby(Scalar alpha, const DenseMatrix& a, Scalar beta, const DenseMatrix* b, Scalar gamma,
                  const char* who) {
  DenseMatrix out(a.rows(), a.cols());
  if (a.size() == 0) return out;
  const double al[2] = {alpha.real(), alpha.imag()}, be[2] = {beta.real(), beta.imag()},
               ga[2] = {gamma.real(), gamma.imag()};
  check(nnb_axpby_z(al, zp(a), be, b ? zp(*b) : nullptr, ga, zp(out), (int64_t)a.rows(),
                    (int64_t)a.cols(), nullptr),
        who);
  require_finite(out, who);
  return out;
}

// The device CSR view: int64 row offsets, int32 columns, real values.
struct DeviceCsr {
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> val;
};

DeviceCsr device_csr(const SparseMatrixCsr& w, const char* who) {
  DeviceCsr d;
  d.rp.assign(w.row_ptr().begin(), w.row_ptr().end());
  d.ci.resize(w.nnz());
  d.val.resize(w.nnz());
  for (std::size_t k = 0; k < w.nnz(); ++k) {
    if (w.values()[k].imag() != 0.0)
      throw DomainError(std::string(who) + ": complex CSR values are not supported by the device path");
    if (w.col_idx()[k] > static_cast<std::size_t>(INT32_MAX))
      throw ShapeError(std::string(who) + ": column index exceeds int32");
    d.ci[k] = static_cast<int32_t>(w.col_idx()[k]);
    d.val[k] = w.values()[k].real();
  }
  return d;
}

std::vector<Scalar> gaussian_probe(std::size_t n, std::uint64_t seed) {
  // proj/src/kernels.cpp:49-62: complex Gaussian entries, normalised
  GaussianStream g(seed);
  std::vector<Scalar> v(n);
  double s = 0.0;
  for (auto& x : v) {
    const double re = g.next();
    const double im = g.next();
    x = Scalar{re, im};
    s += std::norm(x);
  }
  const double nrm = std::sqrt(s);
  if (nrm > 0.0)
    for (auto& x : v) x /= nrm;
  return v;
}

void conform_square(const DenseMatrix& phi, const DenseMatrix& w, const char* who) {
  if (!w.square() || phi.rows() != w.rows() || phi.cols() != w.rows())
    throw ShapeError(std::string(who) + ": shapes do not conform");
}

// One reference-order nest on the device (nnb_nn_step_*).
DenseMatrix device_nest(const DenseMatrix& phi, const DenseMatrix& w, std::size_t depth, const char* who) {
  const std::size_t n = w.rows();
  if (real_valued(phi) && real_valued(w)) {
    const auto pr = real_part(phi), wr = real_part(w);
    std::vector<double> out(n * n);
    check(nnb_nn_step_d(pr.data(), wr.data(), (int64_t)n, (int32_t)depth, out.data(), nullptr), who);
    return from_real(n, n, out);
  }
  DenseMatrix out(n, n);
  check(nnb_nn_step_z(zp(phi), zp(w), (int64_t)n, (int32_t)depth, zp(out), nullptr), who);
  return out;
}

// Product-form schedules through the C-ABI (real data → _d, complex → _z).
DenseMatrix run_schedule(const DenseMatrix& a, const DenseMatrix* b, int64_t x, int64_t y,
                         const std::function<int(const double*, const double*, double*, double*, bool)>& call,
                         double* products, const char* who) {
  const std::size_t n = a.rows();
  DenseMatrix out(n, n);
  if (real_valued(a) && (!b || real_valued(*b))) {
    const auto ar = real_part(a);
    std::vector<double> br = b ? real_part(*b) : std::vector<double>();
    std::vector<double> o(n * n);
    check(call(ar.data(), b ? br.data() : nullptr, o.data(), products, false), who);
    return from_real(n, n, o);
  }
  check(call(zp(a), b ? zp(*b) : nullptr, zp(out), products, true), who);
  return out;
}

}  // namespace

// ====================================================================== types
DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols, std::vector<Scalar> data)
    : r_(rows), c_(cols), v_(std::move(data)) {
  if (v_.size() != r_ * c_) throw ShapeError("DenseMatrix: data length does not match rows*cols");
  if (!all_finite()) throw DomainError("DenseMatrix: non-finite entry on construction");
}

DenseMatrix::DenseMatrix(std::initializer_list<std::initializer_list<Scalar>> rows)
    : r_(rows.size()), c_(rows.size() ? rows.begin()->size() : 0) {
  v_.reserve(r_ * c_);
  for (const auto& row : rows) {
    if (row.size() != c_) throw ShapeError("DenseMatrix: ragged initializer");
    v_.insert(v_.end(), row.begin(), row.end());
  }
}

DenseMatrix DenseMatrix::identity(std::size_t n) {
  DenseMatrix m(n, n);
  for (std::size_t i = 0; i < n; ++i) m.v_[i * n + i] = Scalar{1.0, 0.0};
  return m;
}

DenseMatrix DenseMatrix::diagonal(const std::vector<Scalar>& d) {
  DenseMatrix m(d.size(), d.size());
  for (std::size_t i = 0; i < d.size(); ++i) m.v_[i * d.size() + i] = d[i];
  return m;
}

bool DenseMatrix::all_finite() const {
  return std::all_of(v_.begin(), v_.end(), [](const Scalar& s) {
    return std::isfinite(s.real()) && std::isfinite(s.imag());
  });
}

bool DenseMatrix::is_identity() const {
  if (r_ != c_) return false;
  for (std::size_t i = 0; i < r_; ++i)
    for (std::size_t j = 0; j < c_; ++j)
      if (v_[i * c_ + j] != (i == j ? Scalar{1.0, 0.0} : Scalar{0.0, 0.0})) return false;
  return true;
}

double GaussianStream::next() {
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  auto unit = [this] { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; };
  double u1 = unit();
  while (u1 <= 0.0) u1 = unit();  // (0, 1]
  const double u2 = unit();
  const double rad = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * 3.14159265358979323846 * u2;
  spare_ = rad * std::sin(ang);
  have_spare_ = true;
  return rad * std::cos(ang);
}

SparseMatrixCsr SparseMatrixCsr::build(std::size_t rows, std::size_t cols, std::vector<Triplet> t) {
  // canonical form of proj/src/sparse_csr.cpp:7-40: sorted, duplicates summed, zeros dropped
  for (const auto& e : t)
    if (e.row >= rows || e.col >= cols) throw ShapeError("SparseMatrixCsr: triplet index out of bounds");
  std::sort(t.begin(), t.end(), [](const Triplet& x, const Triplet& y) {
    return x.row != y.row ? x.row < y.row : x.col < y.col;
  });
  SparseMatrixCsr m;
  m.rows_ = rows;
  m.cols_ = cols;
  m.ptr_.assign(rows + 1, 0);
  std::size_t i = 0;
  while (i < t.size()) {
    Scalar sum = t[i].value;
    std::size_t j = i + 1;
    while (j < t.size() && t[j].row == t[i].row && t[j].col == t[i].col) sum += t[j++].value;
    if (sum != Scalar{0.0, 0.0}) {
      m.idx_.push_back(t[i].col);
      m.val_.push_back(sum);
      ++m.ptr_[t[i].row + 1];
    }
    i = j;
  }
  std::partial_sum(m.ptr_.begin(), m.ptr_.end(), m.ptr_.begin());
  return m;
}

SparseMatrixCsr SparseMatrixCsr::identity(std::size_t n) {
  std::vector<Triplet> t(n);
  for (std::size_t i = 0; i < n; ++i) t[i] = {i, i, Scalar{1.0, 0.0}};
  return build(n, n, std::move(t));
}

DenseMatrix SparseMatrixCsr::densify() const {
  DenseMatrix d(rows_, cols_);
  for (std::size_t r = 0; r < rows_; ++r)
    for (std::size_t k = ptr_[r]; k < ptr_[r + 1]; ++k) d(r, idx_[k]) = val_[k];
  return d;
}

Scalar SparseMatrixCsr::trace() const {
  Scalar t{0.0, 0.0};
  for (std::size_t r = 0; r < std::min(rows_, cols_); ++r)
    for (std::size_t k = ptr_[r]; k < ptr_[r + 1]; ++k)
      if (idx_[k] == r) t += val_[k];
  return t;
}

#ifndef NN_DROPIN_HAVE_BOOST
std::string BigInt::str() const {
  if (v_ == 0) return "0";
  std::string s;
  for (rep v = v_; v; v /= 10) s.push_back(static_cast<char>('0' + static_cast<int>(v % 10)));
  return std::string(s.rbegin(), s.rend());
}
static std::size_t msb_of(const BigInt& v) {
  std::size_t b = 0;
  for (auto x = v.value(); x > 1; x >>= 1) ++b;
  return b;
}
static BigInt pow_big(BigInt base, unsigned e) {
  BigInt r(1);
  while (e--) r = r * base;
  return r;
}
#else
static std::size_t msb_of(const BigInt& v) { return boost::multiprecision::msb(v); }
static BigInt pow_big(BigInt base, unsigned e) { return boost::multiprecision::pow(base, e); }
#endif

// ====================================================================== kernels
unsigned worker_count() { return static_cast<unsigned>(std::max(1, nnb_device_count())); }

DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b, OpCounter* counter) {
  // nn::matmul, proj/src/kernels.cpp:137-162
  if (a.cols() != b.rows())
    throw ShapeError("matmul: inner dimensions disagree (" + std::to_string(a.cols()) + " vs " +
                     std::to_string(b.rows()) + ")");
  const std::size_t m = a.rows(), k = a.cols(), n = b.cols();
  DenseMatrix out(m, n);
  if (m && n) {
    if (real_valued(a) && real_valued(b)) {
      const auto ar = real_part(a), br = real_part(b);
      std::vector<double> c(m * n);
      check(nnb_gemm_d(ar.data(), (int64_t)k, br.data(), (int64_t)n, c.data(), (int64_t)n, (int64_t)m,
                       (int64_t)k, (int64_t)n, nullptr),
            "matmul");
      out = from_real(m, n, c);
    } else {
      check(nnb_gemm_z(zp(a), zp(b), zp(out), (int64_t)m, (int64_t)k, (int64_t)n, nullptr), "matmul");
    }
  }
  if (counter) {
    if (m == k && k == n) {
      counter->add_n3(1.0);
    } else {
      const double big = static_cast<double>(std::max({m, k, n}));
      counter->add_n3(static_cast<double>(m) * k * n / (big * big * big));
    }
  }
  return out;
}

DenseMatrix add(const DenseMatrix& a, const DenseMatrix& b, OpCounter* counter) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw ShapeError("add: shape mismatch");
  auto out = axpby(1.0, a, 1.0, &b, 0.0, "add");
  if (counter) counter->add_n2();
  return out;
}

DenseMatrix sub(const DenseMatrix& a, const DenseMatrix& b, OpCounter* counter) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw ShapeError("sub: shape mismatch");
  auto out = axpby(1.0, a, -1.0, &b, 0.0, "sub");
  if (counter) counter->add_n2();
  return out;
}

DenseMatrix scale(const DenseMatrix& m, Scalar factor, OpCounter* counter) {
  auto out = axpby(factor, m, 0.0, nullptr, 0.0, "scale");
  if (counter) counter->add_n2();
  return out;
}

DenseMatrix identity_minus(const DenseMatrix& m, OpCounter* counter) {
  if (!m.square()) throw ShapeError("identity_minus: matrix must be square");
  auto out = axpby(-1.0, m, 0.0, nullptr, 1.0, "identity_minus");
  if (counter) counter->add_n2();
  return out;
}

DenseMatrix plus_identity(const DenseMatrix& m, OpCounter* counter) {
  if (!m.square()) throw ShapeError("plus_identity: matrix must be square");
  auto out = axpby(1.0, m, 0.0, nullptr, 1.0, "plus_identity");
  if (counter) counter->add_n2();
  return out;
}

DenseMatrix conjugate_transpose(const DenseMatrix& m, OpCounter* counter) {
  DenseMatrix out(m.cols(), m.rows());
  if (m.size())
    check(nnb_conj_transpose_z(zp(m), (int64_t)m.rows(), (int64_t)m.cols(), zp(out), nullptr),
          "conjugate_transpose");
  if (counter) counter->add_n2();  // one O(n^2) pass, as kernels.cpp:223-229 tallies it
  return out;
}

Scalar trace(const DenseMatrix& m) {
  if (!m.square()) throw ShapeError("trace: matrix must be square");
  double t[2] = {0.0, 0.0};
  if (m.size()) check(nnb_trace_z(zp(m), (int64_t)m.rows(), t, nullptr), "trace");
  return Scalar{t[0], t[1]};
}

double frobenius_norm(const DenseMatrix& m) {
  double v = 0.0;
  if (m.size()) check(nnb_frobenius_z(zp(m), (int64_t)m.size(), &v, nullptr), "frobenius_norm");
  return v;
}

SpectralEstimate spectral_norm_estimate(const DenseMatrix& m, double tol, int max_iters,
                                        std::uint64_t seed) {
  // proj/src/kernels.cpp:244-269 on the device
  if (!m.square()) throw ShapeError("spectral_norm_estimate: matrix must be square");
  if (tol <= 0.0) throw DomainError("spectral_norm_estimate: tol must be positive");
  if (m.rows() == 0) return {0.0, true, 0};
  const auto v0 = gaussian_probe(m.rows(), seed);
  double value = 0.0;
  int32_t conv = 0, its = 0;
  check(nnb_spectral_norm_z(zp(m), (int64_t)m.rows(), reinterpret_cast<const double*>(v0.data()), tol,
                            max_iters, &value, &conv, &its, nullptr),
        "spectral_norm_estimate");
  return {value, conv != 0, its};
}

SpectralEstimate spectral_norm_estimate_shifted(const SparseMatrixCsr& w, Scalar theta, double tol,
                                                int max_iters, std::uint64_t seed) {
  // proj/src/kernels.cpp:271-305 on the device
  if (!w.square()) throw ShapeError("spectral_norm_estimate_shifted: matrix must be square");
  if (w.rows() == 0) return {0.0, true, 0};
  if (theta.imag() != 0.0) throw DomainError("spectral_norm_estimate_shifted: theta must be real");
  const auto d = device_csr(w, "spectral_norm_estimate_shifted");
  const auto v0 = gaussian_probe(w.rows(), seed);
  double value = 0.0;
  int32_t conv = 0, its = 0;
  check(nnb_spectral_norm_shifted_csr(d.rp.data(), d.ci.data(), d.val.data(), (int64_t)w.rows(),
                                      (int64_t)w.nnz(), theta.real(),
                                      reinterpret_cast<const double*>(v0.data()), tol, max_iters, &value,
                                      &conv, &its, nullptr),
        "spectral_norm_estimate_shifted");
  return {value, conv != 0, its};
}

DenseMatrix spmv_block(const SparseMatrixCsr& p, const DenseMatrix& x, OpCounter* counter) {
  // proj/src/kernels.cpp:454-471: complex n×k block = real n×2k block for real W
  if (p.cols() != x.rows()) throw ShapeError("spmv_block: inner dimensions disagree");
  if (!p.square()) throw DomainError("spmv_block: the device path needs a square CSR operator");
  DenseMatrix out(p.rows(), x.cols());
  if (p.rows() && x.cols()) {
    const auto d = device_csr(p, "spmv_block");
    check(nnb_spmv_block_d(d.rp.data(), d.ci.data(), d.val.data(), (int64_t)p.rows(), (int64_t)p.nnz(), zp(x),
                           (int64_t)(2 * x.cols()), zp(out), nullptr),
          "spmv_block");
  }
  if (counter) counter->add_spmv(static_cast<std::int64_t>(x.cols()));
  require_finite(out, "spmv_block");
  return out;
}

DenseMatrix power_ladder(const DenseMatrix& p, std::uint64_t exponent, OpCounter* counter) {
  // proj/src/kernels.cpp:434-452 on the device
  if (!p.square()) throw ShapeError("power_ladder: matrix must be square");
  if (exponent == 0) return DenseMatrix::identity(p.rows());
  double prods = 0;
  const int64_t n = (int64_t)p.rows();
  DenseMatrix out = run_schedule(
      p, nullptr, 0, 0,
      [&](const double* a, const double*, double* o, double* pr, bool z) {
        return z ? nnb_power_ladder_z(a, n, exponent, o, pr, nullptr) : nnb_power_ladder_d(a, n, exponent, o, pr, nullptr);
      },
      &prods, "power_ladder");
  add_products(counter, prods);
  return out;
}

// ====================================================================== normalization
static double positive_real_trace(Scalar t, const char* who) {
  // proj/src/normalization.cpp:25-33
  const double mag = std::abs(t);
  if (mag > 0.0 && std::abs(t.imag()) > 1e-12 * mag)
    throw NotPsdError(std::string(who) + ": trace has a non-real part");
  if (t.real() <= 0.0) throw NotPsdError(std::string(who) + ": trace is not strictly positive");
  return t.real();
}

static Normalization measured(double theta, double contraction, ThetaKind kind = ThetaKind::TraceTheta1,
                              std::size_t k = 0) {
  Normalization n;
  n.theta = theta;
  n.kind = kind;
  n.k_order = k;
  n.contraction_norm = contraction;
  n.valid = contraction < 1.0;
  return n;
}

Normalization theta_power(const DenseMatrix& w, std::size_t k, std::uint64_t seed) {
  if (!w.square()) throw ShapeError("theta_power: matrix must be square");
  if (k < 1) throw DomainError("theta_power: k must be >= 1");
  const std::size_t n = w.rows();
  // k+1 normalised applications; the last growth factor r = ||W^{k+1}v|| / ||W^k v||
  auto growth_of = [&](std::uint64_t s) -> std::optional<double> {
    const std::vector<Scalar> probe = gaussian_probe(n, s);  // unit complex Gaussian, as the reference draws it
    if (probe.empty() || std::all_of(probe.begin(), probe.end(), [](const Scalar& x) { return x == Scalar{}; }))
      return std::nullopt;
    DenseMatrix v(n, 1, probe);
    double r = 0.0;
    for (std::size_t j = 0; j <= k; ++j) {
      v = matmul(w, v);
      r = frobenius_norm(v);
      if (r == 0.0) return std::nullopt;
      v = scale(v, Scalar{1.0 / r, 0.0});
    }
    return r;
  };
  std::optional<double> r = growth_of(seed);
  if (!r) r = growth_of(seed + 1);
  if (!r) throw DegenerateProbeError("theta_power: probe vector annihilated twice");
  const double kd = static_cast<double>(k);
  const double theta = kd / ((kd + 1.0) * (*r) * (*r));
  const DenseMatrix shifted = identity_minus(scale(w, Scalar{theta, 0.0}));
  return measured(theta, spectral_norm_estimate(shifted).value, ThetaKind::PowerTheta2, k);
}

double contraction_check(const DenseMatrix& phi, const DenseMatrix& w_tilde) {
  return spectral_norm_estimate(identity_minus(matmul(phi, w_tilde))).value;
}

DenseMatrix direct_inverse_oracle(const DenseMatrix& m) {
  if (!m.square()) throw ShapeError("direct_inverse_oracle: matrix must be square");
  const std::size_t n = m.rows();
  if (real_valued(m)) {
    const auto r = real_part(m);
    std::vector<double> out(n * n);
    int32_t piv = -1;
    const int st = nnb_direct_inverse_d(r.data(), (int64_t)n, out.data(), &piv, nullptr);
    if (st == NNB_ERR_SINGULAR) throw SingularMatrixError(nnb_last_error(), static_cast<std::size_t>(piv));
    check(st, "direct_inverse_oracle");
    return from_real(n, n, out);
  }
  DenseMatrix out(n, n);
  int32_t piv = -1;
  const int st = nnb_direct_inverse_z(zp(m), (int64_t)n, zp(out), &piv, nullptr);
  if (st == NNB_ERR_SINGULAR) throw SingularMatrixError(nnb_last_error(), static_cast<std::size_t>(piv));
  check(st, "direct_inverse_oracle");
  return out;
}

std::vector<Scalar> matvec(const DenseMatrix& m, const std::vector<Scalar>& x) {
  if (m.cols() != x.size()) throw ShapeError("matvec: dimension mismatch");
  return matmul(m, DenseMatrix(x.size(), 1, x)).data();
}

Normalization theta_trace(const DenseMatrix& w) {
  const double theta = 1.0 / positive_real_trace(trace(w), "theta_trace");
  const DenseMatrix shifted = identity_minus(scale(w, Scalar{theta, 0.0}));
  return measured(theta, spectral_norm_estimate(shifted).value);
}

Normalization theta_trace(const SparseMatrixCsr& w) {
  if (!w.square()) throw ShapeError("theta_trace: matrix must be square");
  const double theta = 1.0 / positive_real_trace(w.trace(), "theta_trace");
  return measured(theta, spectral_norm_estimate_shifted(w, Scalar{theta, 0.0}).value);
}

DenseMatrix normalize(const DenseMatrix& w, const Normalization& norm) {
  if (!norm.valid)
    throw ContractionError("normalize: normalization does not satisfy the contraction condition");
  return scale(w, Scalar{norm.theta, 0.0});
}

// ====================================================================== solver
std::string stop_reason_name(StopReason r) { return r == StopReason::Tolerance ? "tolerance" : "max_nests"; }

static std::string num(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

std::string report_to_json(const ConvergenceReport& rep) {
  // the stable document of proj/src/solver.cpp:51-70 (same keys and nesting)
  std::ostringstream o;
  o << "{\n  \"alpha_estimate\": " << (rep.alpha_estimate ? num(*rep.alpha_estimate) : "null")
    << ",\n  \"config\": {\n    \"depth_L\": " << rep.config.depth_L
    << ",\n    \"max_nests\": " << rep.config.max_nests << ",\n    \"record_history\": "
    << (rep.config.record_history ? "true" : "false") << ",\n    \"tol\": " << num(rep.config.tol)
    << "\n  },\n  \"counts\": {\n    \"n2_ops\": " << rep.n2_ops << ",\n    \"n3_multiplies\": "
    << num(rep.n3_multiplies) << ",\n    \"spmv_count\": " << rep.spmv_count << "\n  },\n  \"history\": [";
  for (std::size_t i = 0; i < rep.history.size(); ++i)
    o << (i ? "," : "") << "\n    [\n      " << rep.history[i].first << ",\n      " << num(rep.history[i].second)
      << "\n    ]";
  o << (rep.history.empty() ? "]" : "\n  ]") << ",\n  \"kappa_used\": "
    << (rep.kappa_used ? num(*rep.kappa_used) : "null") << ",\n  \"stopped_reason\": \""
    << stop_reason_name(rep.stopped_reason) << "\"\n}";
  return o.str();
}

double residual_epsilon(const DenseMatrix& phi, const DenseMatrix& w_tilde) {
  // proj/src/solver.cpp:72-75, untallied
  if (phi.cols() != w_tilde.rows()) throw ShapeError("matmul: inner dimensions disagree");
  if (phi.rows() != w_tilde.cols()) throw ShapeError("identity_minus: matrix must be square");
  const std::size_t n = w_tilde.rows();
  double eps = 0.0;
  if (real_valued(phi) && real_valued(w_tilde)) {
    const auto pr = real_part(phi), wr = real_part(w_tilde);
    check(nnb_residual_eps_d(pr.data(), wr.data(), (int64_t)n, &eps, nullptr), "residual_epsilon");
  } else {
    check(nnb_residual_eps_z(zp(phi), zp(w_tilde), (int64_t)n, &eps, nullptr), "residual_epsilon");
  }
  return eps;
}

DenseMatrix ns_sum(const DenseMatrix& phi0, const DenseMatrix& w_tilde, std::size_t order, OpCounter* counter) {
  // proj/src/solver.cpp:77-91
  conform_square(phi0, w_tilde, "ns_sum");
  if (order == 0) return phi0;
  const std::size_t n = w_tilde.rows();
  double products = 0.0;
  DenseMatrix out(n, n);
  if (real_valued(phi0) && real_valued(w_tilde)) {
    const auto pr = real_part(phi0), wr = real_part(w_tilde);
    std::vector<double> o(n * n);
    check(nnb_ns_sum_d(pr.data(), wr.data(), (int64_t)n, (int64_t)order, o.data(), &products, nullptr), "ns_sum");
    out = from_real(n, n, o);
  } else {
    check(nnb_ns_sum_z(zp(phi0), zp(w_tilde), (int64_t)n, (int64_t)order, zp(out), &products, nullptr), "ns_sum");
  }
  if (counter) {
    add_products(counter, products);  // order-1 chain products (+2 when phi0 != I)
    counter->add_n2(static_cast<std::int64_t>(order) + 1);  // identity_minus + order plus_identity
  }
  return out;
}

DenseMatrix nn_step(const DenseMatrix& phi, const DenseMatrix& w_tilde, std::size_t depth_L, OpCounter* counter) {
  // proj/src/solver.cpp:93-103: exactly L+1 products (and L+1 n2 passes)
  conform_square(phi, w_tilde, "nn_step");
  if (depth_L == 0) return phi;
  DenseMatrix out = device_nest(phi, w_tilde, depth_L, "nn_step");
  if (counter) {
    add_products(counter, static_cast<double>(depth_L + 1));
    counter->add_n2(static_cast<std::int64_t>(depth_L + 1));
  }
  return out;
}

DenseMatrix newton_step(const DenseMatrix& z, const DenseMatrix& w_tilde, OpCounter* counter) {
  // Z(2I − W~Z) (proj/src/solver.cpp:105-111) ≡ the depth-1 nest (2 products, 1 n2 pass)
  conform_square(z, w_tilde, "newton_step");
  DenseMatrix out = device_nest(z, w_tilde, 1, "newton_step");
  if (counter) {
    add_products(counter, 2.0);
    counter->add_n2(1);
  }
  return out;
}

DenseMatrix chebyshev_step(const DenseMatrix& z, const DenseMatrix& w_tilde, OpCounter* counter) {
  // Z[3I − W~Z(3I − W~Z)] (proj/src/solver.cpp:113-121) ≡ the depth-2 nest (3 products, 2 passes)
  conform_square(z, w_tilde, "chebyshev_step");
  DenseMatrix out = device_nest(z, w_tilde, 2, "chebyshev_step");
  if (counter) {
    add_products(counter, 3.0);
    counter->add_n2(2);
  }
  return out;
}

std::pair<DenseMatrix, ConvergenceReport> nn_invert(const DenseMatrix& w, const Normalization& norm,
                                                    const SolverConfig& config, OpCounter* counter) {
  // proj/src/solver.cpp:123-174: phi0 = I on W~ = theta W, the whole nest loop on the device
  if (!w.square()) throw ShapeError("nn_invert: matrix must be square");
  if (config.tol < 1e-15) throw DomainError("SolverConfig: tol below double precision (minimum 1e-15)");
  if (config.max_nests < 1) throw DomainError("SolverConfig: max_nests must be >= 1");
  const DenseMatrix w_tilde = normalize(w, norm);
  const std::size_t n = w.rows();
  nnb_chain_config cfg{static_cast<int32_t>(config.depth_L), static_cast<int32_t>(config.max_nests), config.tol,
                       NNB_ORDER_REFERENCE, NNB_X0_SCALED_IDENTITY, 1.0, 1};
  nnb_chain_result res{};
  std::vector<double> hist(config.max_nests + 1, 0.0);
  DenseMatrix phi(n, n);
  int st;
  if (real_valued(w_tilde)) {
    const auto wr = real_part(w_tilde);
    std::vector<double> x(n * n);
    st = nnb_nn_chain_d(wr.data(), (int64_t)n, nullptr, &cfg, x.data(), hist.data(), &res, nullptr);
    if (st == NNB_OK) phi = from_real(n, n, x);
  } else {
    st = nnb_nn_chain_z(zp(w_tilde), (int64_t)n, nullptr, &cfg, zp(phi), hist.data(), &res, nullptr);
  }
  if (st == NNB_ERR_DIVERGENCE)
    throw DivergenceError("nn_invert: non-finite iterate at nest " + std::to_string(res.fail_iter),
                          static_cast<std::size_t>(res.fail_iter));
  check(st, "nn_invert");

  ConvergenceReport report;
  report.config = config;
  const std::size_t nests = static_cast<std::size_t>(res.iters);
  if (config.record_history)
    for (std::size_t k = 0; k <= nests; ++k) report.history.emplace_back(k, hist[k]);
  report.stopped_reason = res.stopped == 0 ? StopReason::Tolerance : StopReason::MaxNests;
  // nn_step with depth_L = 0 returns phi untouched: no products, no elementwise ops
  // (proj/src/solver.cpp:97)
  const std::size_t per_nest = config.depth_L > 0 ? config.depth_L + 1 : 0;
  const double n3 = static_cast<double>(nests * per_nest);
  const std::int64_t n2 = static_cast<std::int64_t>(nests * per_nest);
  if (counter) {
    add_products(counter, n3);
    counter->add_n2(n2);
    report.n3_multiplies = n3;
    report.n2_ops = n2;
  }
  if (config.record_history) {
    try {
      report.alpha_estimate = convergence_order_estimate(report);
    } catch (const EstimationError&) {
      report.alpha_estimate.reset();
    }
  }
  return {scale(phi, Scalar{norm.theta, 0.0}, counter), report};
}

DenseMatrix nn_explicit(const DenseMatrix& phi0, const DenseMatrix& w_tilde, std::size_t nests_i,
                        std::size_t depth_L, OpCounter* counter) {
  // proj/src/solver.cpp:176-199 on the device (BudgetError as the reference)
  conform_square(phi0, w_tilde, "nn_explicit");
  if (pow_big(BigInt(depth_L + 1), static_cast<unsigned>(nests_i)) > (BigInt(1) << 62))
    throw BudgetError("nn_explicit: inner power (L+1)^i is not representable");
  double prods = 0;
  const int64_t n = (int64_t)w_tilde.rows();
  DenseMatrix out = run_schedule(
      phi0, &w_tilde, 0, 0,
      [&](const double* a, const double* b, double* o, double* pr, bool z) {
        return z ? nnb_nn_explicit_z(a, b, n, (int64_t)nests_i, (int64_t)depth_L, o, pr, nullptr)
                 : nnb_nn_explicit_d(a, b, n, (int64_t)nests_i, (int64_t)depth_L, o, pr, nullptr);
      },
      &prods, "nn_explicit");
  if (counter) {
    add_products(counter, prods);
    counter->add_n2(1 + static_cast<std::int64_t>((nests_i + 1) * depth_L));  // identity_minus + plus_identity's
  }
  return out;
}

BigInt equivalent_ns_order(std::size_t nests_i, std::size_t depth_L) {
  return pow_big(BigInt(depth_L + 1), static_cast<unsigned>(nests_i + 1)) - 1;
}

std::size_t estimate_nests(double kappa, std::size_t depth_L) {
  // proj/src/solver.cpp:207-217: ceil(log_{L+1}(2 kappa^{2 ln 2}) − 1), at least 1
  if (kappa < 1.0) throw DomainError("estimate_nests: kappa must be >= 1");
  if (depth_L < 1) throw DomainError("estimate_nests: depth must be >= 1");
  const double ln2 = std::log(2.0);
  const double v = std::ceil((ln2 + 2.0 * ln2 * std::log(kappa)) / std::log(depth_L + 1.0) - 1.0);
  return v < 1.0 ? 1 : static_cast<std::size_t>(v);
}

double convergence_order_estimate(const ConvergenceReport& report) {
  // proj/src/solver.cpp:219-257: LSQ slope of log eps_{k+1} vs log eps_k inside (1e-12, 0.5)
  auto inside = [](double e) { return e > 1e-12 && e < 0.5; };
  const auto usable = std::count_if(report.history.begin(), report.history.end(),
                                    [&](const auto& h) { return inside(h.second); });
  if (usable < 4)
    throw EstimationError("convergence_order_estimate: need at least 4 history entries inside the (1e-12, 0.5) window, have " +
                          std::to_string(usable));
  std::vector<std::pair<double, double>> pts;
  for (std::size_t k = 0; k + 1 < report.history.size(); ++k) {
    const auto& a = report.history[k];
    const auto& b = report.history[k + 1];
    if (inside(a.second) && inside(b.second) && b.first == a.first + 1)
      pts.emplace_back(std::log(a.second), std::log(b.second));
  }
  if (pts.size() < 2) throw EstimationError("convergence_order_estimate: too few usable pairs");
  double mx = 0.0, my = 0.0;
  for (const auto& [x, y] : pts) {
    mx += x;
    my += y;
  }
  mx /= static_cast<double>(pts.size());
  my /= static_cast<double>(pts.size());
  double sxy = 0.0, sxx = 0.0;
  for (const auto& [x, y] : pts) {
    sxy += (x - mx) * (y - my);
    sxx += (x - mx) * (x - mx);
  }
  if (sxx == 0.0) throw EstimationError("convergence_order_estimate: degenerate abscissae");
  return sxy / sxx;
}

// ====================================================================== factorized
FactorizedPlan FactorizedPlan::for_order(const BigInt& gamma, FactorizedMode mode) {
  if (gamma < BigInt(1)) throw PlanError("FactorizedPlan: order must be >= 1");
  if (((gamma + BigInt(1)) & gamma) != BigInt(0)) throw PlanError("FactorizedPlan: order + 1 must be a power of two");
  FactorizedPlan plan;
  plan.gamma = gamma;
  plan.num_factors = msb_of(gamma + BigInt(1));
  plan.mode = mode;
  return plan;
}

DenseMatrix ns_factorized(const DenseMatrix& phi, const DenseMatrix& w_tilde, const FactorizedPlan& plan,
                          OpCounter* counter) {
  // proj/src/factorized.cpp:42-61 on the device: 2s−1 products from the identity, 2s+1 otherwise
  if (plan.mode != FactorizedMode::DenseStored) throw PlanError("ns_factorized: plan must be in dense mode");
  conform_square(phi, w_tilde, "ns_factorized");
  double prods = 0;
  const int64_t n = (int64_t)w_tilde.rows();
  const int64_t gamma = static_cast<int64_t>(static_cast<unsigned long long>(plan.gamma));
  DenseMatrix out = run_schedule(
      phi, &w_tilde, 0, 0,
      [&](const double* a, const double* b, double* o, double* pr, bool z) {
        return z ? nnb_ns_factorized_z(a, b, n, gamma, o, pr, nullptr) : nnb_ns_factorized_d(a, b, n, gamma, o, pr, nullptr);
      },
      &prods, "ns_factorized");
  if (counter) {
    add_products(counter, prods);
    counter->add_n2(static_cast<std::int64_t>(plan.num_factors) + 1);  // identity_minus + s plus_identity
  }
  return out;
}

// ==================================================================== generators
namespace {
std::vector<double> log_uniform_spectrum(std::size_t n, double cond) {
  std::vector<double> lam(n, 1.0);  // kernels.cpp:116-124: cond^-t, t from 1 down to 0
  if (n > 1)
    for (std::size_t j = 0; j < n; ++j)
      lam[j] = std::pow(cond, -(static_cast<double>(n - 1 - j) / static_cast<double>(n - 1)));
  return lam;
}
}  // namespace

DenseMatrix random_spd(std::size_t n, double cond, std::uint64_t seed) {
  if (n < 1) throw DomainError("random_spd: n must be >= 1");
  if (cond < 1.0) throw DomainError("random_spd: cond must be >= 1");
  GaussianStream g(seed);
  const std::vector<double> gauss = g.take(n * n);  // row-major, as the reference fills it
  const std::vector<double> lam = log_uniform_spectrum(n, cond);
  std::vector<double> w(n * n);
  check(nnb_random_spd_d(gauss.data(), lam.data(), (int64_t)n, w.data(), nullptr), "random_spd");
  return from_real(n, n, w);
}

DenseMatrix random_conditioned_complex(std::size_t n, double cond, std::uint64_t seed) {
  if (n < 1) throw DomainError("random_conditioned_complex: n must be >= 1");
  if (cond < 1.0) throw DomainError("random_conditioned_complex: cond must be >= 1");
  GaussianStream g(seed);
  const std::vector<double> gu = g.take(2 * n * n), gv = g.take(2 * n * n);  // (re, im) pairs, U's draw first
  const std::vector<double> sigma = log_uniform_spectrum(n, cond);
  DenseMatrix out(n, n);
  check(nnb_random_conditioned_z(gu.data(), gv.data(), sigma.data(), (int64_t)n, zp(out), nullptr),
        "random_conditioned_complex");
  return out;
}

SparseMatrixCsr random_sparse_spd(std::size_t n, double density, std::uint64_t seed) {
  if (n < 1) throw DomainError("random_sparse_spd: n must be >= 1");
  if (density < 0.0 || density > 1.0) throw DomainError("random_sparse_spd: density must be in [0,1]");
  // kernels.cpp:409-432: an upper-triangle pattern stream and a value stream,
  // mirrored, with a diagonal 1 + Σ|off-diagonal| for strict dominance
  std::mt19937_64 pattern(seed);
  GaussianStream values(seed ^ 0x9e3779b97f4a7c15ULL);
  std::vector<SparseMatrixCsr::Triplet> t;
  std::vector<double> offsum(n, 0.0);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = i + 1; j < n; ++j) {
      if (static_cast<double>(pattern() >> 11) * 0x1.0p-53 >= density) continue;
      const double x = values.next();
      t.push_back({i, j, Scalar{x, 0.0}});
      t.push_back({j, i, Scalar{x, 0.0}});
      offsum[i] += std::fabs(x);
      offsum[j] += std::fabs(x);
    }
  for (std::size_t i = 0; i < n; ++i) t.push_back({i, i, Scalar{1.0 + offsum[i], 0.0}});
  return SparseMatrixCsr::build(n, n, std::move(t));
}

DenseMatrix cns_invert(const DenseMatrix& w_tilde, const CnsConfig& cns, OpCounter* counter) {
  if (!w_tilde.square()) throw ShapeError("cns_invert: matrix must be square");
  if (cns.ns_terms < 1) throw DomainError("cns_invert: ns_terms must be >= 1");
  DenseMatrix pre = DenseMatrix::identity(w_tilde.rows());  // order 3^ci_steps − 1 after the steps
  for (std::size_t i = 0; i < cns.ci_steps; ++i) pre = chebyshev_step(pre, w_tilde, counter);
  const std::size_t t = cns.ns_terms;
  if (cns.factorize_outer && ((t + 1) & t) == 0)  // t + 1 a power of two: the product form applies
    return ns_factorized(pre, w_tilde, FactorizedPlan::for_order(BigInt(t), FactorizedMode::DenseStored), counter);
  return ns_sum(pre, w_tilde, t, counter);
}

// proj/src/factorized.cpp:63-99: W = A^H A and rhs = A^H B (unless the caller
// already formed them), theta from theta_trace(W), W^-1 from nn_invert, then
// x = W^-1 rhs.  The backward error on the normal equations is diagnostic and
// untallied; NonConvergenceError when the nest budget ran out above tol.
NormalSolveResult solve_normal_equations(const LinearSystem& sys, const SolverConfig& config, OpCounter* counter) {
  const DenseMatrix a = std::holds_alternative<DenseMatrix>(sys.a) ? std::get<DenseMatrix>(sys.a)
                                                                    : std::get<SparseMatrixCsr>(sys.a).densify();
  if (!a.square()) throw ShapeError("solve_normal_equations: A must be square");
  if (sys.b.rows() != a.rows()) throw ShapeError("solve_normal_equations: B row count does not match A");
  DenseMatrix w = a, rhs = sys.b;
  if (!sys.hermitian_normal) {
    const DenseMatrix ah = conjugate_transpose(a, counter);
    w = matmul(ah, a, counter);
    rhs = matmul(ah, sys.b, counter);
  }
  auto [w_inv, report] = nn_invert(w, theta_trace(w), config, counter);
  NormalSolveResult res{matmul(w_inv, rhs, counter), std::move(report), 0.0};
  const double rn = frobenius_norm(rhs), en = frobenius_norm(sub(matmul(w, res.x), rhs));
  res.backward_error = rn > 0.0 ? en / rn : en;
  if (res.report.stopped_reason == StopReason::MaxNests && res.backward_error > config.tol)
    throw NonConvergenceError("solve_normal_equations: nest budget exhausted with backward error " +
                                  std::to_string(res.backward_error),
                              res.report);
  return res;
}

DenseMatrix solve_sparse_factorized(const LinearSystem& sys, const BigInt& gamma, const Normalization& norm,
                                    OpCounter* counter) {
  // proj/src/factorized.cpp:101-140 on the device; checks in the reference's order
  if (!std::holds_alternative<SparseMatrixCsr>(sys.a))
    throw ShapeError("solve_sparse_factorized: system matrix must be CSR");
  const SparseMatrixCsr& w = std::get<SparseMatrixCsr>(sys.a);
  if (!w.square()) throw ShapeError("solve_sparse_factorized: W must be square");
  if (sys.b.rows() != w.rows()) throw ShapeError("solve_sparse_factorized: B row count does not match W");
  if (!norm.valid) throw ContractionError("solve_sparse_factorized: invalid normalization");
  const std::size_t s = FactorizedPlan::for_order(gamma, FactorizedMode::SparseMatrixFree).num_factors;
  if (gamma > (BigInt(1) << 30)) throw BudgetError("solve_sparse_factorized: order too large to apply");
  const auto d = device_csr(w, "solve_sparse_factorized");
  const std::size_t n = w.rows(), k = sys.b.cols();
  DenseMatrix x(n, k);
  int64_t applied = 0;
  int32_t fail_factor = -1;
  // complex n×k block = real n×2k block (W is real): one device solve for all columns
  const int st = nnb_sparse_factorized_d(d.rp.data(), d.ci.data(), d.val.data(), (int64_t)n, (int64_t)w.nnz(),
                                         zp(sys.b), (int64_t)(2 * k), static_cast<int64_t>(static_cast<unsigned long long>(gamma)),
                                         norm.theta, zp(x), &applied, &fail_factor, nullptr);
  if (st == NNB_ERR_DIVERGENCE)
    throw DivergenceError("solve_sparse_factorized: non-finite block at factor " + std::to_string(fail_factor),
                          static_cast<std::size_t>(fail_factor));
  check(st, "solve_sparse_factorized");
  if (counter) {
    const auto g = static_cast<std::int64_t>(static_cast<unsigned long long>(gamma));
    counter->add_spmv(g * static_cast<std::int64_t>(k));
    counter->add_n2(g + static_cast<std::int64_t>(s) + 1);  // fused_axpy_sub per application, add per factor, scale
  }
  return x;
}

}  // namespace nn
