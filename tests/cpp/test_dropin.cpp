// Drop-in API tests: the reference's hot-path unit tests (proj/tests/test_solver.cpp,
// test_matrix_core.cpp, test_factorized.cpp, test_preconditioning.cpp) restated
// against the nn:: drop-in (every matrix op on the GPU through libnnb).
//   ./test_dropin            all tests (needs a GPU)
//   ./test_dropin --host     host-only checks (GaussianStream, CSR build, BigInt, formulas)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <filesystem>
#include <sstream>

#include "nn/factorized.hpp"
#include "nn/matrix_market.hpp"
#include "nn/kernels.hpp"
#include "nn/normalization.hpp"
#include "nn/rng.hpp"
#include "nn/solver.hpp"

using namespace nn;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(c)) {                                                               \
      ++g_fail;                                                               \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);              \
    }                                                                         \
  } while (0)
#define CHECK_THROWS(expr, Type)                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    bool ok_ = false;                                                         \
    try { (void)(expr); } catch (const Type&) { ok_ = true; } catch (...) {}  \
    if (!ok_) { ++g_fail; std::printf("  FAIL %s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #Type); } \
  } while (0)

static double rel(const DenseMatrix& a, const DenseMatrix& b) {
  double d = 0, n = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    d += std::norm(a.data()[i] - b.data()[i]);
    n += std::norm(b.data()[i]);
  }
  return n > 0 ? std::sqrt(d / n) : std::sqrt(d);
}

static DenseMatrix gauss(std::size_t r, std::size_t c, std::uint64_t seed, bool cplx = false) {
  GaussianStream g(seed);
  DenseMatrix m(r, c);
  for (auto& v : m.data()) {
    const double re = g.next();
    v = Scalar{re, cplx ? g.next() : 0.0};
  }
  return m;
}

// SPD test matrix B·B^T/n + shift·I (the reference's random_spd is out of scope)
static DenseMatrix spd(std::size_t n, double shift, std::uint64_t seed) {
  DenseMatrix b = gauss(n, n, seed);
  DenseMatrix bt(n, n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) bt(j, i) = b(i, j);
  DenseMatrix a = scale(matmul(b, bt), Scalar{1.0 / n, 0});
  for (std::size_t i = 0; i < n; ++i) a(i, i) += shift;
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = i + 1; j < n; ++j) a(j, i) = a(i, j);
  return a;
}

static DenseMatrix normalized(std::size_t n, double shift, std::uint64_t seed) {
  const DenseMatrix w = spd(n, shift, seed);
  return normalize(w, theta_trace(w));
}

static DenseMatrix s1(double v) { return DenseMatrix::diagonal({Scalar{v, 0}}); }

// Matrix Market I/O (proj/tests/test_matrix_market.cpp restated; host only)
static void mm_tests() {
  GaussianStream g(7);
  DenseMatrix m(5, 3);
  for (auto& v : m.data()) v = Scalar{g.next() * 1e-7, g.next() * 1e9};
  std::stringstream ss;
  mm::write_dense(ss, m);
  CHECK(mm::read_dense(ss) == m);  // 17 significant digits: bit-exact round trip

  DenseMatrix r(2, 2);
  r(0, 0) = Scalar{1.5, 0};
  std::stringstream sr;
  mm::write_dense(sr, r);
  CHECK(sr.str().find("array real general") != std::string::npos);
  CHECK(mm::read_dense(sr) == r);

  std::istringstream colmajor("%%MatrixMarket matrix array real general\n% a comment line\n2 3\n1\n2\n3\n4\n5\n6\n");
  const DenseMatrix cm = mm::read_dense(colmajor);
  CHECK(cm(0, 0) == (Scalar{1, 0}) && cm(1, 0) == (Scalar{2, 0}) && cm(0, 1) == (Scalar{3, 0}) &&
        cm(1, 2) == (Scalar{6, 0}));

  const SparseMatrixCsr sp = random_sparse_spd(24, 0.15, 3);
  std::stringstream ssp;
  mm::write_sparse(ssp, sp);
  const SparseMatrixCsr back = mm::read_sparse(ssp);
  CHECK(back.row_ptr() == sp.row_ptr() && back.col_idx() == sp.col_idx() && back.values() == sp.values());

  std::istringstream sym("%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 5.0\n3 3 1.0\n");
  const SparseMatrixCsr s3 = mm::read_sparse(sym);
  CHECK(s3.nnz() == 3 && s3.densify()(1, 0) == (Scalar{5, 0}) && s3.densify()(0, 1) == (Scalar{5, 0}));
  std::istringstream her("%%MatrixMarket matrix coordinate complex hermitian\n2 2 1\n2 1 1.0 2.0\n");
  const DenseMatrix h = mm::read_sparse(her).densify();
  CHECK(h(1, 0) == (Scalar{1, 2}) && h(0, 1) == (Scalar{1, -2}));
  std::istringstream icoord("%%MatrixMarket matrix coordinate integer general\n2 2 1\n1 2 7\n");
  const DenseMatrix dc = mm::read_dense(icoord);
  CHECK(dc(0, 1) == (Scalar{7, 0}) && dc(1, 0) == (Scalar{0, 0}));
  std::istringstream symarr("%%MATRIXMARKET matrix ARRAY real Symmetric\n2 2\n1\n2\n3\n");
  CHECK_THROWS(mm::read_dense(symarr), IoError);  // the tag itself is case-sensitive
  std::istringstream symarr2("%%MatrixMarket matrix ARRAY real Symmetric\n2 2\n1\n2\n3\n");
  const DenseMatrix sa = mm::read_dense(symarr2);
  CHECK(sa(1, 0) == (Scalar{2, 0}) && sa(0, 1) == (Scalar{2, 0}) && sa(1, 1) == (Scalar{3, 0}));

  std::istringstream bad_banner("%%NotMatrixMarket\n1 1\n1\n");
  CHECK_THROWS(mm::read_dense(bad_banner), IoError);
  std::istringstream truncated("%%MatrixMarket matrix array real general\n3 3\n1\n2\n");
  CHECK_THROWS(mm::read_dense(truncated), IoError);
  std::istringstream out_of_range("%%MatrixMarket matrix coordinate real general\n2 2 1\n5 1 1.0\n");
  CHECK_THROWS(mm::read_sparse(out_of_range), IoError);
  std::istringstream array_as_sparse("%%MatrixMarket matrix array real general\n1 1\n1\n");
  CHECK_THROWS(mm::read_sparse(array_as_sparse), IoError);
  std::istringstream missing_im("%%MatrixMarket matrix array complex general\n1 1\n1.0\n");
  CHECK_THROWS(mm::read_dense(missing_im), IoError);

  namespace fs = std::filesystem;
  const fs::path dir = fs::temp_directory_path() / "nnb_mm_test";
  fs::create_directories(dir);
  const std::string path = (dir / "w.mtx").string(), spath = (dir / "s.mtx").string();
  mm::write_dense_file(path, m);
  CHECK(mm::read_dense_file(path) == m);
  CHECK(!fs::exists(path + ".tmp"));
  CHECK(!mm::file_is_coordinate(path));
  mm::write_sparse_file(spath, random_sparse_spd(6, 0.3, 6));
  CHECK(mm::file_is_coordinate(spath));
  CHECK_THROWS(mm::read_dense_file((dir / "missing.mtx").string()), IoError);
  fs::remove_all(dir);
}

static void host_tests() {
  // GaussianStream: mt19937_64 + Box-Muller (values printed for the pytest cross-check)
  GaussianStream g(42);
  std::printf("gaussian42:");
  for (int i = 0; i < 6; ++i) std::printf(" %.17g", g.next());
  std::printf("\n");
  // CSR canonicalisation (proj/tests/test_matrix_core.cpp:275-290)
  const SparseMatrixCsr m = SparseMatrixCsr::build(
      2, 3, {{1, 2, Scalar{5, 0}}, {0, 1, Scalar{2, 0}}, {0, 1, Scalar{-2, 0}}, {1, 0, Scalar{1, 0}}, {1, 2, Scalar{3, 0}}});
  CHECK(m.nnz() == 2);
  CHECK((m.row_ptr() == std::vector<std::size_t>{0, 0, 2}));
  CHECK((m.col_idx() == std::vector<std::size_t>{0, 2}));
  CHECK(m.values()[1] == (Scalar{8, 0}));
  CHECK_THROWS(SparseMatrixCsr::build(2, 2, {{2, 0, Scalar{1, 0}}}), ShapeError);
  // order formulas (proj/tests/test_solver.cpp:297-320)
  CHECK(equivalent_ns_order(1, 2) == BigInt(8));
  CHECK(equivalent_ns_order(3, 2) == BigInt(80));
  CHECK(equivalent_ns_order(50, 2).str() == "2153693963075557766310746");
  CHECK(equivalent_ns_order(37, 2).str() == "1350851717672992088");
  CHECK(estimate_nests(1e6, 2) == 18);
  CHECK(estimate_nests(1e4, 2) == 12);
  CHECK(estimate_nests(1.0, 1) == 1);
  CHECK_THROWS(estimate_nests(0.5, 2), DomainError);
  CHECK(FactorizedPlan::for_order(15, FactorizedMode::DenseStored).num_factors == 4);
  CHECK_THROWS(FactorizedPlan::for_order(6, FactorizedMode::DenseStored), PlanError);
  CHECK_THROWS(FactorizedPlan::for_order(0, FactorizedMode::DenseStored), PlanError);
  CHECK_THROWS(DenseMatrix(1, 1, {Scalar{INFINITY, 0}}), DomainError);
  CHECK_THROWS((DenseMatrix{{Scalar{1, 0}}, {Scalar{1, 0}, Scalar{2, 0}}}), ShapeError);
  mm_tests();
}

static void device_tests() {
  // ---- matrix core
  {
    const DenseMatrix m = gauss(3, 3, 11);
    CHECK(rel(matmul(DenseMatrix::identity(3), m), m) == 0.0);
    const DenseMatrix p = matmul(DenseMatrix::diagonal({Scalar{2, 0}, Scalar{3, 0}}),
                                 DenseMatrix::diagonal({Scalar{5, 0}, Scalar{7, 0}}));
    CHECK(p(0, 0) == (Scalar{10, 0}) && p(1, 1) == (Scalar{21, 0}) && p(0, 1) == (Scalar{0, 0}));
    const DenseMatrix a = gauss(4, 4, 21, true), b = gauss(4, 4, 22, true);
    DenseMatrix naive(4, 4);
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 4; ++k)
        for (int i = 0; i < 4; ++i) naive(i, j) += a(i, k) * b(k, j);
    CHECK(rel(matmul(a, b), naive) < 1e-15);
    CHECK_THROWS(matmul(gauss(2, 3, 1), gauss(2, 2, 2)), ShapeError);
    OpCounter c;
    matmul(gauss(8, 8, 3), gauss(8, 8, 4), &c);
    CHECK(c.n3_multiplies() == 1.0);
    matmul(gauss(8, 2, 5), gauss(2, 8, 6), &c);
    CHECK(std::fabs(c.n3_multiplies() - 1.25) < 1e-15);
    CHECK(trace(DenseMatrix::identity(3)) == (Scalar{3, 0}));
    CHECK(std::fabs(frobenius_norm(DenseMatrix::identity(4)) - 2.0) < 1e-15);
    CHECK(frobenius_norm(DenseMatrix(4, 4)) == 0.0);
    // associativity at kernel scale (complex)
    const DenseMatrix x = gauss(32, 32, 1, true), y = gauss(32, 32, 101, true), z = gauss(32, 32, 201, true);
    CHECK(rel(matmul(matmul(x, y), z), matmul(x, matmul(y, z))) < 1e-12);
  }
  // ---- preconditioning (proj/tests/test_preconditioning.cpp:13-27)
  {
    const DenseMatrix w = DenseMatrix::diagonal({Scalar{1, 0}, Scalar{3, 0}});
    const Normalization n = theta_trace(w);
    CHECK(std::fabs(n.theta - 0.25) < 1e-15);
    CHECK(std::fabs(n.contraction_norm - 0.75) < 1e-9);
    CHECK(n.valid);
    CHECK(std::fabs(trace(normalize(w, n)).real() - 1.0) < 1e-14);
    Normalization bad = n;
    bad.valid = false;
    CHECK_THROWS(normalize(w, bad), ContractionError);
  }
  // ---- ns_sum (proj/tests/test_solver.cpp:30-71)
  {
    const DenseMatrix wt = normalized(4, 1.0, 1), phi0 = spd(4, 2.0, 2);
    CHECK(ns_sum(phi0, wt, 0) == phi0);
    const DenseMatrix s = ns_sum(DenseMatrix::identity(2), DenseMatrix::diagonal({Scalar{0.25, 0}, Scalar{0.75, 0}}), 3);
    CHECK(std::fabs(s(0, 0).real() - (1 + 0.75 + 0.75 * 0.75 + 0.75 * 0.75 * 0.75)) < 1e-15);
    CHECK(std::fabs(s(1, 1).real() - (1 + 0.25 + 0.25 * 0.25 + 0.25 * 0.25 * 0.25)) < 1e-15);
    const DenseMatrix w6 = normalized(6, 0.5, 4);
    const DenseMatrix p0 = scale(DenseMatrix::identity(6), Scalar{1.5, 0});
    for (std::size_t order : {1, 2, 5, 17}) {  // vs explicit power accumulation
      const DenseMatrix P = identity_minus(matmul(p0, w6));
      DenseMatrix acc = DenseMatrix::identity(6), pw = DenseMatrix::identity(6);
      for (std::size_t k = 1; k <= order; ++k) {
        pw = matmul(pw, P);
        acc = add(acc, pw);
      }
      CHECK(rel(ns_sum(p0, w6, order), matmul(acc, p0)) < 1e-13);
    }
    OpCounter c;
    ns_sum(DenseMatrix::identity(6), w6, 7, &c);
    CHECK(c.n3_multiplies() == 6.0);
    c.reset();
    ns_sum(scale(DenseMatrix::identity(6), Scalar{0.9, 0}), w6, 7, &c);
    CHECK(c.n3_multiplies() == 8.0);
  }
  // ---- nn_step / newton / chebyshev (proj/tests/test_solver.cpp:73-132)
  {
    for (std::uint64_t seed : {1ULL, 9ULL}) {
      const DenseMatrix wt = normalized(16, 0.3, seed);
      DenseMatrix z = DenseMatrix::identity(16);
      const DenseMatrix I = DenseMatrix::identity(16);
      for (int step = 0; step < 4; ++step) {
        // the closed forms, composed from separate device ops
        const DenseMatrix y = matmul(wt, z);
        const DenseMatrix newton = matmul(z, sub(scale(I, Scalar{2, 0}), y));
        const DenseMatrix inner = matmul(y, sub(scale(I, Scalar{3, 0}), y));
        const DenseMatrix cheby = matmul(z, sub(scale(I, Scalar{3, 0}), inner));
        CHECK(rel(nn_step(z, wt, 1), newton) < 1e-13);
        CHECK(rel(nn_step(z, wt, 2), cheby) < 1e-13);
        CHECK(rel(newton_step(z, wt), newton) < 1e-13);
        CHECK(rel(chebyshev_step(z, wt), cheby) < 1e-13);
        z = newton;
      }
    }
    const DenseMatrix wt = normalized(8, 0.5, 7);
    DenseMatrix phi = DenseMatrix::identity(8);
    for (std::size_t depth : {1, 2, 3, 5}) {
      OpCounter c;
      phi = nn_step(phi, wt, depth, &c);
      CHECK(c.n3_multiplies() == static_cast<double>(depth + 1));
    }
    CHECK(nn_step(phi, wt, 0) == phi);
    OpCounter c;
    DenseMatrix zz = newton_step(s1(1.0), s1(0.5), &c);
    CHECK(std::fabs(zz(0, 0).real() - 1.5) < 1e-15);
    zz = newton_step(zz, s1(0.5), &c);
    CHECK(std::fabs(zz(0, 0).real() - 1.875) < 1e-15);
    CHECK(c.n3_multiplies() == 4.0);
    OpCounter c2;
    CHECK(std::fabs(chebyshev_step(s1(1.0), s1(0.5), &c2)(0, 0).real() - 1.75) < 1e-15);
    CHECK(c2.n3_multiplies() == 3.0);
    CHECK_THROWS(nn_step(DenseMatrix::identity(3), DenseMatrix::identity(4), 1), ShapeError);
  }
  // ---- equivalence chain: recursive NN == plain series (proj/tests/test_solver.cpp:278-295)
  {
    const DenseMatrix wt = normalized(8, 0.5, 20), id = DenseMatrix::identity(8);
    for (std::size_t depth = 1; depth <= 5; ++depth)
      for (std::size_t nests = 0;; ++nests) {
        const BigInt order = equivalent_ns_order(nests, depth);
        if (order > BigInt(200)) break;
        DenseMatrix rec = id;
        for (std::size_t j = 0; j <= nests; ++j) rec = nn_step(rec, wt, depth);
        CHECK(rel(rec, ns_sum(id, wt, static_cast<std::size_t>(order))) < 1e-11);
      }
  }
  // ---- nn_invert (proj/tests/test_solver.cpp:134-228, 378-386)
  {
    const DenseMatrix w = DenseMatrix::identity(12);
    SolverConfig cfg;
    cfg.depth_L = 2;
    cfg.tol = 1e-12;
    cfg.max_nests = 40;
    const auto [inv, rep] = nn_invert(w, theta_trace(w), cfg);
    CHECK(rep.stopped_reason == StopReason::Tolerance);
    CHECK(rel(inv, w) < 1e-12);

    const DenseMatrix w16 = spd(16, 0.01, 13);
    const Normalization nm = theta_trace(w16);
    for (std::size_t depth = 1; depth <= 3; ++depth)
      for (std::size_t nests = 1; nests <= 4; ++nests) {
        SolverConfig c;
        c.depth_L = depth;
        c.max_nests = nests;
        c.tol = 1e-15;
        OpCounter cnt;
        const auto [x, r] = nn_invert(w16, nm, c, &cnt);
        CHECK(r.stopped_reason == StopReason::MaxNests);
        CHECK(r.n3_multiplies == static_cast<double>(nests * (depth + 1)));
        CHECK(cnt.n3_multiplies() == static_cast<double>(nests * (depth + 1)));
        CHECK(r.history.size() == nests + 1);
      }
    {  // depth_L = 0: nn_step is the identity (proj/src/solver.cpp:97), so no products are tallied
      SolverConfig c0;
      c0.depth_L = 0;
      c0.max_nests = 3;
      c0.tol = 1e-15;
      OpCounter cnt;
      const auto [x0, r0] = nn_invert(w16, nm, c0, &cnt);
      CHECK(r0.n3_multiplies == 0.0 && r0.n2_ops == 0);
      CHECK(cnt.n3_multiplies() == 0.0);
      CHECK(r0.history.size() == 4);
    }
    // deeper nests converge in fewer iterations; history strictly decreasing above 1e-12
    SolverConfig c;
    c.tol = 1e-10;
    c.max_nests = 64;
    c.depth_L = 1;
    const auto r1 = nn_invert(w16, nm, c).second;
    c.depth_L = 2;
    const auto r2 = nn_invert(w16, nm, c).second;
    CHECK(r1.stopped_reason == StopReason::Tolerance && r2.stopped_reason == StopReason::Tolerance);
    CHECK(r1.history.back().first > r2.history.back().first);
    for (std::size_t k = 0; k + 1 < r2.history.size(); ++k)
      if (r2.history[k].second > 1e-12) CHECK(r2.history[k + 1].second < r2.history[k].second);
    // inverse quality
    c.tol = 1e-12;
    const auto [inv16, rep16] = nn_invert(w16, nm, c);
    const DenseMatrix resid = sub(matmul(w16, inv16), DenseMatrix::identity(16));
    CHECK(frobenius_norm(resid) / 4.0 < 1e-10);
    // json report keys
    const std::string js = report_to_json(rep16);
    CHECK(js.find("\"stopped_reason\": \"tolerance\"") != std::string::npos);
    CHECK(js.find("\"history\"") != std::string::npos && js.find("\"n3_multiplies\"") != std::string::npos);
    // errors
    Normalization bad = nm;
    bad.valid = false;
    CHECK_THROWS(nn_invert(w16, bad, c), ContractionError);
    Normalization absurd = nm;
    absurd.theta = 1e160;
    try {
      nn_invert(w16, absurd, SolverConfig{});
      CHECK(false);
    } catch (const DivergenceError& e) {
      CHECK(e.nest_index >= 1);
    }
    SolverConfig v;
    v.tol = 1e-16;
    CHECK_THROWS(nn_invert(w16, nm, v), DomainError);
    v.tol = 1e-10;
    v.max_nests = 0;
    CHECK_THROWS(nn_invert(w16, nm, v), DomainError);
  }
  // ---- sparse path (proj/tests/test_matrix_core.cpp:242-273, test_factorized.cpp:150-207)
  {
    const DenseMatrix b = gauss(6, 3, 81, true);
    CHECK(spmv_block(SparseMatrixCsr::identity(6), b) == b);
    std::vector<SparseMatrixCsr::Triplet> t;
    const std::size_t n = 64;
    for (std::size_t i = 0; i < n; ++i) {
      t.push_back({i, i, Scalar{4.5, 0}});
      if (i + 1 < n) {
        t.push_back({i, i + 1, Scalar{-1, 0}});
        t.push_back({i + 1, i, Scalar{-1, 0}});
      }
      if (i + 8 < n) {
        t.push_back({i, i + 8, Scalar{-1, 0}});
        t.push_back({i + 8, i, Scalar{-1, 0}});
      }
    }
    const SparseMatrixCsr w = SparseMatrixCsr::build(n, n, t);
    const DenseMatrix x = gauss(n, 4, 92, true);
    OpCounter c;
    CHECK(rel(spmv_block(w, x, &c), matmul(w.densify(), x)) < 1e-15);
    CHECK(c.spmv_count() == 4);
    const Normalization nm = theta_trace(w);
    CHECK(nm.valid);
    DenseMatrix rhs(n, 2);
    for (std::size_t i = 0; i < rhs.size(); ++i) rhs.data()[i] = Scalar{std::cos(double(i)), 0};
    OpCounter cs;
    const DenseMatrix xs = solve_sparse_factorized({w, rhs, false}, 15, nm, &cs);
    CHECK(cs.spmv_count() == 15 * 2);
    // dense factorized series theta * prod_{f<4} (I + P^{2^f}) B, composed from device products
    const DenseMatrix P = identity_minus(scale(w.densify(), Scalar{nm.theta, 0}));
    DenseMatrix acc = DenseMatrix::identity(n), pw = P;
    for (int f = 0; f < 4; ++f) {
      acc = matmul(acc, plus_identity(pw));
      pw = matmul(pw, pw);
    }
    CHECK(rel(xs, scale(matmul(acc, rhs), Scalar{nm.theta, 0})) < 1e-11);
    // the same through the dense factorized series (proj/tests/test_factorized.cpp:170-186)
    const auto plan15 = FactorizedPlan::for_order(15, FactorizedMode::DenseStored);
    const DenseMatrix wt_dense = scale(w.densify(), Scalar{nm.theta, 0});
    CHECK(rel(xs, scale(matmul(ns_factorized(DenseMatrix::identity(n), wt_dense, plan15), rhs),
                        Scalar{nm.theta, 0})) < 1e-11);
    // identity system: theta = 1/8, x = (1 - (7/8)^16) B
    const SparseMatrixCsr I8 = SparseMatrixCsr::identity(8);
    const DenseMatrix b8 = gauss(8, 8, 10);
    const DenseMatrix x8 = solve_sparse_factorized({I8, b8, false}, 15, theta_trace(I8));
    CHECK(rel(x8, scale(b8, Scalar{1 - std::pow(7.0 / 8.0, 16.0), 0})) < 1e-12);
    // rejections
    CHECK_THROWS(solve_sparse_factorized({w, rhs, false}, 6, nm), PlanError);
    CHECK_THROWS(solve_sparse_factorized({w, DenseMatrix(5, 1), false}, 7, nm), ShapeError);
    CHECK_THROWS(solve_sparse_factorized({rhs, rhs, false}, 7, nm), ShapeError);
    Normalization inv = nm;
    inv.valid = false;
    CHECK_THROWS(solve_sparse_factorized({w, rhs, false}, 7, inv), ContractionError);
    Normalization absurd = nm;
    absurd.theta = 1e150;
    CHECK_THROWS(solve_sparse_factorized({w, rhs, false}, 32767, absurd), DivergenceError);
  }
}

// ns_factorized / power_ladder / nn_explicit (proj/tests/test_factorized.cpp:33-72,
// test_matrix_core.cpp:220-240, test_solver.cpp:257-300)
static void schedule_tests() {
  const DenseMatrix wt = normalized(16, 0.5, 2), id = DenseMatrix::identity(16);
  CHECK(rel(ns_factorized(DenseMatrix::identity(6), normalized(6, 0.5, 1),
                          FactorizedPlan::for_order(1, FactorizedMode::DenseStored)),
            ns_sum(DenseMatrix::identity(6), normalized(6, 0.5, 1), 1)) < 1e-15);
  const DenseMatrix out = ns_factorized(s1(1.0), s1(0.5), FactorizedPlan::for_order(7, FactorizedMode::DenseStored));
  CHECK(std::fabs(out(0, 0).real() - 1.9921875) < 1e-15);
  for (long g : {1L, 3L, 7L, 15L, 31L, 63L}) {
    const auto plan = FactorizedPlan::for_order(g, FactorizedMode::DenseStored);
    CHECK(rel(ns_factorized(id, wt, plan), ns_sum(id, wt, static_cast<std::size_t>(g))) < 1e-12);
    const double s = static_cast<double>(plan.num_factors);
    OpCounter ci, cg;
    ns_factorized(id, wt, plan, &ci);
    ns_factorized(scale(id, Scalar{0.5, 0}), wt, plan, &cg);
    CHECK(ci.n3_multiplies() == 2 * s - 1);
    CHECK(cg.n3_multiplies() == 2 * s + 1);
  }
  CHECK_THROWS(ns_factorized(id, wt, FactorizedPlan::for_order(3, FactorizedMode::SparseMatrixFree)), PlanError);
  OpCounter c;
  const DenseMatrix p14 = power_ladder(DenseMatrix::diagonal({Scalar{2, 0}}), 14, &c);
  CHECK(p14(0, 0) == (Scalar{16384, 0}));
  CHECK(c.n3_multiplies() == 5.0);
  const DenseMatrix m = gauss(4, 4, 61);
  OpCounter c1;
  CHECK(power_ladder(m, 1, &c1) == m && c1.n3_multiplies() == 0.0);
  CHECK(power_ladder(m, 0) == DenseMatrix::identity(4));
  const DenseMatrix base = scale(gauss(8, 8, 71, true), Scalar{0.3, 0});
  DenseMatrix seq = base;
  for (std::uint64_t e = 2; e <= 37; ++e) {
    seq = matmul(seq, base);
    if (e == 2 || e == 14 || e == 37) CHECK(rel(power_ladder(base, e), seq) < 1e-12);
  }
  for (std::size_t depth : {1, 2, 4}) CHECK(rel(nn_explicit(id, wt, 0, depth), ns_sum(id, wt, depth)) < 1e-13);
  CHECK(std::fabs(nn_explicit(s1(1.0), s1(0.5), 1, 1)(0, 0).real() - 1.875) < 1e-15);
  CHECK(rel(nn_explicit(id, wt, 2, 2), ns_sum(id, wt, 26)) < 1e-11);
  CHECK_THROWS(nn_explicit(DenseMatrix::identity(2), normalized(2, 0.5, 21), 40, 2), BudgetError);
}

// theta_power / contraction_check / matvec (proj/tests/test_preconditioning.cpp:49-123 restated)
static void power_normalization_tests() {
  for (std::size_t k : {1, 2, 8}) {
    const auto nm = theta_power(DenseMatrix::identity(6), k, 3);
    CHECK(std::fabs(nm.theta - static_cast<double>(k) / (k + 1.0)) < 1e-12);
    CHECK(std::fabs(nm.contraction_norm - 1.0 / (k + 1.0)) < 1e-9);
    CHECK(nm.valid && nm.kind == ThetaKind::PowerTheta2 && nm.k_order == k);
  }
  const auto d13 = theta_power(DenseMatrix::diagonal({Scalar{1, 0}, Scalar{3, 0}}), 8, 7);
  CHECK(std::fabs(d13.theta - 8.0 / 81.0) < 1e-5 * (8.0 / 81.0));
  CHECK(std::fabs(d13.contraction_norm - (1.0 - d13.theta)) < 1e-6 && d13.valid);
  // test_preconditioning.cpp:70 expects contraction 1/5 here, but theta = 4/(5·0.1²) = 80 gives
  // ||I − 80·0.1·I|| = 7 (SURVEY.md Appendix A lists it as failing in the reference): pin that
  const auto sc = theta_power(scale(DenseMatrix::identity(4), Scalar{0.1, 0}), 4, 5);
  CHECK(std::fabs(sc.theta - 80.0) < 1e-10 * 80.0 && std::fabs(sc.contraction_norm - 7.0) < 1e-9 && !sc.valid);
  DenseMatrix nilpotent(2, 2);
  nilpotent(0, 1) = Scalar{1, 0};
  CHECK_THROWS(theta_power(nilpotent, 1, 11), DegenerateProbeError);
  CHECK_THROWS(theta_power(DenseMatrix::identity(3), 0, 1), DomainError);

  const DenseMatrix wt = DenseMatrix::diagonal({Scalar{0.25, 0}, Scalar{0.75, 0}});
  const DenseMatrix inv = direct_inverse_oracle(wt);
  CHECK(inv(0, 0) == (Scalar{4.0, 0}) && std::fabs(inv(1, 1).real() - 4.0 / 3.0) < 1e-15);
  CHECK(contraction_check(inv, wt) < 1e-9);
  DenseMatrix sing(3, 3);
  sing(0, 0) = Scalar{1, 0};
  bool threw = false;
  try {
    direct_inverse_oracle(sing);
  } catch (const SingularMatrixError& e) {
    threw = e.pivot_index == 1;
  }
  CHECK(threw);
  CHECK(std::fabs(contraction_check(DenseMatrix::identity(2), wt) - 0.75) < 1e-9);
  CHECK(std::fabs(contraction_check(DenseMatrix(2, 2), wt) - 1.0) < 1e-9);

  const DenseMatrix m = gauss(5, 3, 81, true);
  const std::vector<Scalar> x = {Scalar{1, 2}, Scalar{-0.5, 0}, Scalar{0, 3}};
  const std::vector<Scalar> y = matvec(m, x);
  double err = 0.0;
  for (std::size_t i = 0; i < 5; ++i) {
    Scalar s{0, 0};
    for (std::size_t k = 0; k < 3; ++k) s += m(i, k) * x[k];
    err = std::max(err, std::abs(y[i] - s));
  }
  CHECK(y.size() == 5 && err < 1e-14);
  CHECK_THROWS(matvec(m, std::vector<Scalar>(2)), ShapeError);
}

// cns_invert (proj/tests/test_factorized.cpp:209-250 restated)
static void cns_tests() {
  const DenseMatrix wt = normalized(8, 0.5, 14), id = DenseMatrix::identity(8);
  CnsConfig plain;
  plain.ci_steps = 0;
  plain.ns_terms = 5;
  CHECK(rel(cns_invert(wt, plain), ns_sum(id, wt, 5)) < 1e-14);
  CnsConfig two;
  two.ci_steps = 2;
  two.ns_terms = 1;
  double expect = 0.0;  // Σ_{n=0}^{17} 0.5^n
  for (int k = 17; k >= 0; --k) expect += std::pow(0.5, k);
  CHECK(std::fabs(cns_invert(s1(0.5), two)(0, 0).real() - expect) < 1e-14 * expect);
  CHECK(std::fabs(chebyshev_step(chebyshev_step(s1(1.0), s1(0.5)), s1(0.5))(0, 0).real() - 1.99609375) < 1e-15);
  CnsConfig eff;
  eff.ci_steps = 2;
  eff.ns_terms = 2;  // effective order 3^2·3 − 1 = 26
  CHECK(rel(cns_invert(wt, eff), ns_sum(id, wt, 26)) < 1e-11);
  CnsConfig p3;
  p3.ci_steps = 1;
  p3.ns_terms = 3;
  CnsConfig f3 = p3;
  f3.factorize_outer = true;
  CHECK(rel(cns_invert(wt, f3), cns_invert(wt, p3)) < 1e-12);
  CnsConfig bad;
  bad.ns_terms = 0;
  CHECK_THROWS(cns_invert(wt, bad), DomainError);
}

// conjugate_transpose and solve_normal_equations (proj/tests/test_factorized.cpp:80-148,
// test_matrix_core.cpp conjugate_transpose cases), inputs from this file's generators.
static void normal_equation_tests() {
  const DenseMatrix z = gauss(5, 3, 91, true);
  const DenseMatrix zh = conjugate_transpose(z);
  CHECK(zh.rows() == 3 && zh.cols() == 5);
  bool conj_ok = true;
  for (std::size_t i = 0; i < 5; ++i)
    for (std::size_t j = 0; j < 3; ++j) conj_ok &= zh(j, i) == std::conj(z(i, j));
  CHECK(conj_ok);
  CHECK(conjugate_transpose(zh) == z);
  OpCounter ct;
  conjugate_transpose(z, &ct);
  CHECK(ct.n2_ops() == 1 && ct.n3_multiplies() == 0.0);

  SolverConfig cfg;
  cfg.depth_L = 2;
  cfg.tol = 1e-12;
  cfg.max_nests = 40;
  const DenseMatrix b6 = spd(6, 3.0, 5);
  CHECK(rel(solve_normal_equations({DenseMatrix::identity(6), b6, false}, cfg).x, b6) < 1e-12);

  const DenseMatrix d = DenseMatrix::diagonal({Scalar{1, 0}, Scalar{2, 0}, Scalar{4, 0}});
  DenseMatrix ones(3, 1);
  ones(0, 0) = ones(1, 0) = ones(2, 0) = Scalar{1, 0};
  cfg.tol = 1e-13;
  cfg.max_nests = 60;
  const auto rd = solve_normal_equations({d, ones, false}, cfg);
  CHECK(std::fabs(rd.x(0, 0).real() - 1.0) < 1e-10 && std::fabs(rd.x(1, 0).real() - 0.5) < 1e-10 &&
        std::fabs(rd.x(2, 0).real() - 0.25) < 1e-10);
  CHECK(rd.backward_error < 1e-12);

  // W = A^H A is Hermitian to rounding
  DenseMatrix a = gauss(12, 12, 93, true);
  for (std::size_t i = 0; i < 12; ++i) a(i, i) += Scalar{4.0, 0};
  const DenseMatrix w = matmul(conjugate_transpose(a), a);
  CHECK(rel(conjugate_transpose(w), w) < 1e-12);

  // a complex system: x solves A x = B, tallies as the reference counts them
  const DenseMatrix bb = gauss(12, 2, 95, true);
  cfg.depth_L = 2;
  cfg.tol = 1e-11;
  cfg.max_nests = 40;
  OpCounter cs;
  const auto rs = solve_normal_equations({a, bb, false}, cfg, &cs);
  CHECK(rel(matmul(a, rs.x), bb) < 1e-9);
  CHECK(rs.report.stopped_reason == StopReason::Tolerance);
  const double nests = static_cast<double>(rs.report.history.size() - 1);
  CHECK(std::fabs(cs.n3_multiplies() - (1.0 + 2.0 * (2.0 / 12.0) + 3.0 * nests)) < 1e-12);
  CHECK(cs.n2_ops() == static_cast<std::int64_t>(1 + 3 * nests + 1));

  // the pre-formed normal equations take the same path minus the W/rhs products
  const DenseMatrix ah = conjugate_transpose(a);
  const auto rh = solve_normal_equations({matmul(ah, a), matmul(ah, bb), true}, cfg);
  CHECK(rel(rh.x, rs.x) < 1e-12);

  // the nest budget runs out: NonConvergenceError carries the report
  cfg.depth_L = 1;
  cfg.tol = 1e-12;
  cfg.max_nests = 2;
  DenseMatrix e0(12, 1);
  e0(0, 0) = Scalar{1, 0};
  bool threw = false;
  try {
    solve_normal_equations({gauss(12, 12, 97, true), e0, false}, cfg);
  } catch (const NonConvergenceError& e) {
    threw = e.report.stopped_reason == StopReason::MaxNests && e.report.history.size() == 3;
  }
  CHECK(threw);
  CHECK_THROWS(solve_normal_equations({gauss(3, 4, 1), ones, false}, cfg), ShapeError);
  CHECK_THROWS(solve_normal_equations({d, DenseMatrix(4, 1), false}, cfg), ShapeError);
}

// --normal IN OUT: solve_normal_equations on a system from a binary file
//   IN:  int64 n, k, depth_L, max_nests; double tol; complex A (n×n); complex B (n×k)
//   OUT: int64 status (0 ok, 20 NonConvergenceError), history length h; double history[h],
//        n3, n2, backward; complex x (n×k)
static int normal_cli(const char* in_path, const char* out_path) {
  std::FILE* f = std::fopen(in_path, "rb");
  if (!f) return 2;
  std::int64_t hdr[4];
  double tol = 0.0;
  bool ok = std::fread(hdr, sizeof(hdr), 1, f) == 1 && std::fread(&tol, sizeof(tol), 1, f) == 1;
  const std::size_t n = static_cast<std::size_t>(hdr[0]), k = static_cast<std::size_t>(hdr[1]);
  DenseMatrix a(n, n), b(n, k);
  ok = ok && std::fread(a.data().data(), sizeof(Scalar), n * n, f) == n * n &&
       std::fread(b.data().data(), sizeof(Scalar), n * k, f) == n * k;
  std::fclose(f);
  if (!ok) return 2;
  SolverConfig cfg;
  cfg.depth_L = static_cast<std::size_t>(hdr[2]);
  cfg.max_nests = static_cast<std::size_t>(hdr[3]);
  cfg.tol = tol;
  OpCounter cnt;
  std::int64_t status = 0;
  NormalSolveResult res;
  try {
    res = solve_normal_equations({a, b, false}, cfg, &cnt);
  } catch (const NonConvergenceError& e) {
    status = 20;
    res.report = e.report;
    res.x = DenseMatrix(n, k);
  }
  std::FILE* o = std::fopen(out_path, "wb");
  if (!o) return 2;
  const std::int64_t h = static_cast<std::int64_t>(res.report.history.size());
  std::fwrite(&status, sizeof(status), 1, o);
  std::fwrite(&h, sizeof(h), 1, o);
  for (const auto& e : res.report.history) std::fwrite(&e.second, sizeof(double), 1, o);
  const double tail[3] = {cnt.n3_multiplies(), static_cast<double>(cnt.n2_ops()), res.backward_error};
  std::fwrite(tail, sizeof(tail), 1, o);
  std::fwrite(res.x.data().data(), sizeof(Scalar), n * k, o);
  std::fclose(o);
  return 0;
}

int main(int argc, char** argv) {
  if (argc == 4 && std::strcmp(argv[1], "--normal") == 0) return normal_cli(argv[2], argv[3]);
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host") == 0;
  host_tests();
  if (!host_only) {
    device_tests();
    schedule_tests();
    normal_equation_tests();
    power_normalization_tests();
    cns_tests();
  }
  std::printf("%s: %d checks, %d failures\n", host_only ? "host" : "all", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
