// nnbench on the B200 drop-in: the reference CLI's
// subcommands, options, stdout lines, JSON reports, CSV schema and exit codes
// (/root/reference/proj/tools/nnbench.cpp), with every matrix operation on
// the GPU through libnn_b200 → libnnb.
//
//   nnbench gen-matrix --N n --out f.mtx [--cond c] [--seed s] [--kind spd|complex|sparse-spd] [--density d]
//   nnbench invert IN.mtx [--method nn|newton|chebyshev|ns|nn-explicit|factorized-ns|cns] [--depth|-L L]
//                  [--nests|-i k] [--order|--gamma g] [--tol t] [--theta trace|power:k] [--seed s] [--out X.mtx]
//                  [--report r.json] [--estimate-kappa]
//   nnbench solve --matrix|-A A.mtx --rhs|-b B.mtx [--method nn|sparse-factorized] [--depth|-L L]
//                 [--nests|-i k] [--order|--gamma g] [--tol t] [--out x.mtx] [--report r.json]
//   nnbench bench --methods m1,m2 [--N n1,n2] [--cond c1,c2] [--depths L1,L2] [--nests|-i k] [--tol t]
//                 [--seed s] [--out grid.csv]
//
// Exit codes: 0 success / tolerance reached, 2 nest budget exhausted, 1 input
// or validation error.  Not provided: analyze-cost (the exact-rational cost
// model is out of scope).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "nn/factorized.hpp"
#include "nn/kernels.hpp"
#include "nn/matrix_market.hpp"
#include "nn/normalization.hpp"
#include "nn/solver.hpp"

using namespace nn;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string g17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

// ---- options: "--name value", "--name=value", short aliases, flags ----------
class Options {
 public:
  Options(int argc, char** argv, const std::map<std::string, std::string>& aliases,
          const std::vector<std::string>& flags) {
    for (int k = 2; k < argc; ++k) {
      std::string a = argv[k];
      if (a.size() < 2 || a[0] != '-') {
        positional_.push_back(a);
        continue;
      }
      std::string value;
      bool has_value = false;
      if (const auto eq = a.find('='); eq != std::string::npos) {
        value = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_value = true;
      }
      if (auto it = aliases.find(a); it != aliases.end()) a = it->second;
      bool is_flag = false;
      for (const auto& f : flags) is_flag |= f == a;
      if (is_flag) {
        values_[a] = "1";
        continue;
      }
      if (!has_value) {
        if (k + 1 >= argc) throw UsageError("option " + a + " needs a value");
        value = argv[++k];
      }
      values_[a] = value;
    }
  }
  bool has(const std::string& k) const { return values_.count(k) != 0; }
  std::string str(const std::string& k, const std::string& d = "") const {
    auto it = values_.find(k);
    return it == values_.end() ? d : it->second;
  }
  double num(const std::string& k, double d) const { return has(k) ? parse_double(str(k)) : d; }
  long long integer(const std::string& k, long long d) const { return has(k) ? parse_int(str(k)) : d; }
  std::string require(const std::string& k) const {
    if (!has(k)) throw UsageError(k + " is required");
    return str(k);
  }
  const std::vector<std::string>& positional() const { return positional_; }
  template <class T, class F>
  std::vector<T> list(const std::string& k, std::vector<T> d, F parse) const {
    if (!has(k)) return d;
    std::vector<T> out;
    std::stringstream ss(str(k));
    std::string item;
    while (std::getline(ss, item, ','))
      if (!item.empty()) out.push_back(parse(item));
    return out;
  }
  static double parse_double(const std::string& s) {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || *end) throw UsageError("not a number: '" + s + "'");
    return v;
  }
  static long long parse_int(const std::string& s) {
    char* end = nullptr;
    const long long v = std::strtoll(s.c_str(), &end, 10);
    if (end == s.c_str() || *end) throw UsageError("not an integer: '" + s + "'");
    return v;
  }

 private:
  std::map<std::string, std::string> values_;
  std::vector<std::string> positional_;
};

Normalization normalization(const DenseMatrix& w, const std::string& theta, std::uint64_t seed) {
  if (theta == "trace") return theta_trace(w);
  if (theta.rfind("power:", 0) == 0) {
    const long k = std::strtol(theta.c_str() + 6, nullptr, 10);
    if (k < 1) throw DomainError("--theta power:k requires k >= 1");
    const Normalization power = theta_power(w, static_cast<std::size_t>(k), seed);
    if (power.valid) return power;
    std::cerr << "note: power normalization not contractive (measured " << power.contraction_norm
              << "), falling back to trace\n";
    return theta_trace(w);
  }
  throw DomainError("--theta must be 'trace' or 'power:k'");
}

// ‖I − X·W‖_F / √N
double inverse_quality(const DenseMatrix& w, const DenseMatrix& x) {
  return frobenius_norm(identity_minus(matmul(x, w))) / std::sqrt(static_cast<double>(w.rows()));
}

BigInt next_factorized_order(const BigInt& at_least) {  // smallest 2^s − 1 >= at_least
  BigInt p(2);
  while (p - 1 < at_least) p = p << 1;
  return p - 1;
}

// ---------------------------------------------------------------- gen-matrix
int gen_matrix(const Options& o) {
  const std::size_t n = static_cast<std::size_t>(o.integer("--N", -1));
  if (!o.has("--N")) throw UsageError("--N is required");
  const std::string out = o.require("--out"), kind = o.str("--kind", "spd");
  const double cond = o.num("--cond", 1e2);
  const std::uint64_t seed = static_cast<std::uint64_t>(o.integer("--seed", 1));
  if (kind == "spd") mm::write_dense_file(out, random_spd(n, cond, seed));
  else if (kind == "complex") mm::write_dense_file(out, random_conditioned_complex(n, cond, seed));
  else if (kind == "sparse-spd") mm::write_sparse_file(out, random_sparse_spd(n, o.num("--density", 0.05), seed));
  else throw DomainError("--kind must be spd, complex or sparse-spd");
  std::cout << "wrote " << out << "\n";
  return 0;
}

// ---------------------------------------------------------------- invert
int invert(const Options& o) {
  if (o.positional().size() != 1) throw UsageError("invert takes exactly one input matrix");
  const DenseMatrix w = mm::read_dense_file(o.positional()[0]);
  if (!w.square()) throw ShapeError("invert: input matrix must be square");
  std::optional<double> kappa;
  if (o.has("--estimate-kappa")) {  // ||W||_2 · ||W^-1||_2 with the Gauss–Jordan oracle, as the reference
    if (w.rows() > 128) throw DomainError("--estimate-kappa is limited to N <= 128");
    kappa = spectral_norm_estimate(w).value * spectral_norm_estimate(direct_inverse_oracle(w)).value;
  }
  const std::string method = o.str("--method", "nn");
  const Normalization norm =
      normalization(w, o.str("--theta", "trace"), static_cast<std::uint64_t>(o.integer("--seed", 1)));
  SolverConfig config;
  config.depth_L = static_cast<std::size_t>(o.integer("--depth", 2));
  config.tol = o.num("--tol", 1e-10);
  const long long nests = o.integer("--nests", 0), order = o.integer("--order", -1);
  config.max_nests = nests > 0 ? static_cast<std::size_t>(nests)
                     : kappa   ? estimate_nests(*kappa, std::max<std::size_t>(config.depth_L, 1))
                               : 64;

  OpCounter counter;
  DenseMatrix inverse;
  ConvergenceReport report;
  report.config = config;
  if (method == "nn" || method == "newton" || method == "chebyshev") {
    if (method == "newton") config.depth_L = 1;
    if (method == "chebyshev") config.depth_L = 2;
    std::tie(inverse, report) = nn_invert(w, norm, config, &counter);
  } else {
    const DenseMatrix wt = normalize(w, norm), id = DenseMatrix::identity(w.rows());
    DenseMatrix phi;
    if (method == "ns") {
      if (order < 0) throw DomainError("--order is required for --method ns");
      phi = ns_sum(id, wt, static_cast<std::size_t>(order), &counter);
    } else if (method == "nn-explicit") {
      phi = nn_explicit(id, wt, config.max_nests, config.depth_L, &counter);
    } else if (method == "factorized-ns") {
      if (order < 0) throw DomainError("--order is required for --method factorized-ns");
      phi = ns_factorized(id, wt, FactorizedPlan::for_order(BigInt(order), FactorizedMode::DenseStored), &counter);
    } else if (method == "cns") {
      CnsConfig cns;
      cns.ci_steps = nests > 0 ? static_cast<std::size_t>(nests) : 1;
      cns.ns_terms = order >= 1 ? static_cast<std::size_t>(order) : 1;
      phi = cns_invert(wt, cns, &counter);
    } else {
      throw DomainError("unknown --method '" + method + "'");
    }
    const double eps = residual_epsilon(phi, wt);
    inverse = scale(phi, Scalar{norm.theta, 0.0}, &counter);
    report.history.emplace_back(0, eps);
    report.stopped_reason = eps < config.tol ? StopReason::Tolerance : StopReason::MaxNests;
    report.n3_multiplies = counter.n3_multiplies();
    report.n2_ops = counter.n2_ops();
  }
  report.kappa_used = kappa;
  if (o.has("--out")) mm::write_dense_file(o.str("--out"), inverse);
  if (o.has("--report")) mm::write_file_atomic(o.str("--report"), report_to_json(report));
  const double final_eps = report.history.empty() ? inverse_quality(w, inverse) : report.history.back().second;
  std::cout << "method=" << method << " N=" << w.rows() << " eps=" << g17(final_eps)
            << " n3=" << g17(counter.n3_multiplies()) << " stopped=" << stop_reason_name(report.stopped_reason)
            << "\n";
  return report.stopped_reason == StopReason::Tolerance ? 0 : 2;
}

// ---------------------------------------------------------------- solve
int solve(const Options& o) {
  const DenseMatrix b = mm::read_dense_file(o.require("--rhs"));
  const std::string method = o.str("--method", "nn");
  const double tol = o.num("--tol", 1e-10);
  if (method == "sparse-factorized") {
    const SparseMatrixCsr w = mm::read_sparse_file(o.require("--matrix"));
    const long long gamma = o.integer("--order", 15);
    OpCounter counter;
    const DenseMatrix x = solve_sparse_factorized({w, b, false}, BigInt(gamma), theta_trace(w), &counter);
    const double backward = frobenius_norm(sub(spmv_block(w, x), b)) / std::max(frobenius_norm(b), 1e-300);
    if (o.has("--out")) mm::write_dense_file(o.str("--out"), x);
    if (o.has("--report")) {
      std::ostringstream j;  // keys in the reference's (sorted) order
      j << "{\n  \"backward_error\": " << g17(backward) << ",\n  \"counts\": {\n    \"n2_ops\": "
        << counter.n2_ops() << ",\n    \"spmv_count\": " << counter.spmv_count() << "\n  },\n  \"gamma\": " << gamma
        << ",\n  \"method\": \"sparse-factorized\"\n}";
      mm::write_file_atomic(o.str("--report"), j.str());
    }
    std::cout << "method=sparse-factorized backward=" << g17(backward) << " spmv=" << counter.spmv_count() << "\n";
    return backward <= tol ? 0 : 2;
  }
  if (method != "nn") throw DomainError("solve supports --method nn or sparse-factorized");
  const DenseMatrix a = mm::read_dense_file(o.require("--matrix"));
  SolverConfig config;
  config.depth_L = static_cast<std::size_t>(o.integer("--depth", 2));
  config.tol = tol;
  const long long nests = o.integer("--nests", 0);
  config.max_nests = nests > 0 ? static_cast<std::size_t>(nests) : 64;
  OpCounter counter;
  try {
    const auto res = solve_normal_equations({a, b, false}, config, &counter);
    if (o.has("--out")) mm::write_dense_file(o.str("--out"), res.x);
    if (o.has("--report")) mm::write_file_atomic(o.str("--report"), report_to_json(res.report));
    std::cout << "method=nn backward=" << g17(res.backward_error) << " nests=" << res.report.history.back().first
              << "\n";
    return 0;
  } catch (const NonConvergenceError& e) {
    if (o.has("--report")) mm::write_file_atomic(o.str("--report"), report_to_json(e.report));
    std::cerr << "solve: " << e.what() << "\n";
    return 2;
  }
}

// ---------------------------------------------------------------- bench
// The reference's CSV row for one grid point; failures fill the metric
// columns with blanks and the message (commas → ';') as the status.
std::string bench_point(const std::string& method, std::size_t n, double cond, std::size_t depth,
                        std::size_t nests_opt, double tol, std::uint64_t seed, bool& failed) {
  std::ostringstream row;
  row << method << "," << n << "," << g17(cond) << ",";
  try {
    const DenseMatrix w = random_spd(n, cond, seed);
    const Normalization norm = theta_trace(w);
    const DenseMatrix wt = normalize(w, norm), id = DenseMatrix::identity(n);
    const std::size_t depth_eff = method == "newton" ? 1 : method == "chebyshev" ? 2 : depth;
    const std::size_t nests = nests_opt > 0 ? nests_opt : estimate_nests(cond, depth_eff);
    OpCounter counter;
    DenseMatrix inverse;
    std::optional<double> alpha;
    std::size_t nests_reported = nests;
    BigInt gamma = equivalent_ns_order(nests - 1, depth_eff);
    std::string predicted;  // the cost model's N^3 coefficient (cost_model.cpp:43-77)
    const auto t0 = std::chrono::steady_clock::now();
    if (method == "nn" || method == "newton" || method == "chebyshev") {
      SolverConfig config;
      config.depth_L = depth_eff;
      config.max_nests = nests;
      config.tol = tol;
      auto [inv, rep] = nn_invert(w, norm, config, &counter);
      inverse = std::move(inv);
      alpha = rep.alpha_estimate;
      nests_reported = rep.history.back().first;
      gamma = nests_reported > 0 ? equivalent_ns_order(nests_reported - 1, depth_eff) : BigInt(0);
      predicted = (BigInt(nests_reported) * BigInt(depth_eff + 1)).str();
    } else if (method == "ns") {
      if (gamma > BigInt(100000)) throw BudgetError("bench: ns order too large");
      inverse = scale(ns_sum(id, wt, static_cast<std::size_t>(gamma), &counter), Scalar{norm.theta, 0.0}, &counter);
      predicted = (gamma - 1).str();
    } else if (method == "factorized-ns") {
      gamma = next_factorized_order(gamma);
      const auto plan = FactorizedPlan::for_order(gamma, FactorizedMode::DenseStored);
      inverse = scale(ns_factorized(id, wt, plan, &counter), Scalar{norm.theta, 0.0}, &counter);
      predicted = std::to_string(2 * plan.num_factors - 1);
    } else if (method == "nn-explicit") {
      inverse = scale(nn_explicit(id, wt, nests - 1, depth_eff, &counter), Scalar{norm.theta, 0.0}, &counter);
      const unsigned long long i = nests - 1;  // (L/2)(i(i+1)(i+2)+1) + 2i(i+1)+1, in lowest terms
      const unsigned long long twice = depth_eff * (i * (i + 1) * (i + 2) + 1) + 2 * (2 * i * (i + 1) + 1);
      predicted = twice % 2 ? std::to_string(twice) + "/2" : std::to_string(twice / 2);
    } else if (method == "cns") {
      CnsConfig cns;
      cns.ci_steps = 2;
      cns.ns_terms = std::max<std::size_t>(nests, 1);
      inverse = scale(cns_invert(wt, cns, &counter), Scalar{norm.theta, 0.0}, &counter);
      gamma = BigInt(9) * BigInt(cns.ns_terms + 1) - 1;
      predicted = "0";
    } else {
      throw DomainError("unknown bench method '" + method + "'");
    }
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    row << depth_eff << "," << nests_reported << "," << gamma.str() << "," << g17(inverse_quality(w, inverse)) << ","
        << g17(counter.n3_multiplies()) << "," << counter.n2_ops() << "," << counter.spmv_count() << ","
        << (alpha ? g17(*alpha) : "") << "," << predicted << "," << g17(wall) << ",ok";
    failed = false;
  } catch (const Error& e) {
    std::string msg = e.what();
    for (char& c : msg)
      if (c == ',' || c == '\n') c = ';';
    row << ",,,,,,,,,," << msg;
    failed = true;
  }
  return row.str();
}

int bench(const Options& o) {
  const auto as_str = [](const std::string& s) { return s; };
  const auto as_size = [](const std::string& s) { return static_cast<std::size_t>(Options::parse_int(s)); };
  const auto methods = o.list<std::string>("--methods", {}, as_str);
  if (methods.empty()) throw DomainError("bench: --methods must not be empty");
  const auto sizes = o.list<std::size_t>("--N", {16}, as_size);
  const auto conds = o.list<double>("--cond", {1e2}, Options::parse_double);
  const auto depths = o.list<std::size_t>("--depths", {2}, as_size);
  const std::size_t nests = static_cast<std::size_t>(o.integer("--nests", 0));
  const double tol = o.num("--tol", 1e-10);
  const std::uint64_t seed = static_cast<std::uint64_t>(o.integer("--seed", 1));
  std::ostringstream csv;
  csv << "method,N,cond,L,i,gamma_effective,eps_final,n3_multiplies,n2_ops,spmv_count,alpha_estimate,"
         "predicted_n3,wall_seconds,status\n";
  std::size_t rows = 0, failures = 0;
  // the grid in the reference's order; points run one after another on the GPU
  for (const auto& m : methods)
    for (std::size_t in = 0; in < sizes.size(); ++in)
      for (std::size_t ic = 0; ic < conds.size(); ++ic)
        for (const std::size_t d : depths) {
          bool failed = false;
          csv << bench_point(m, sizes[in], conds[ic], d, nests, tol, seed + 1000 * in + ic, failed) << "\n";
          ++rows;
          failures += failed;
        }
  if (o.has("--out")) mm::write_file_atomic(o.str("--out"), csv.str());
  else std::cout << csv.str();
  if (failures == rows) {
    std::cerr << "bench: all " << failures << " runs failed\n";
    return 1;
  }
  return 0;
}

void usage(std::ostream& out) {
  out << "usage: nnbench <gen-matrix|invert|solve|bench> [options]   (B200 build; see the header of "
         "dropin/tools/nnbench.cpp)\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(std::cerr);
    return 1;
  }
  const std::string cmd = argv[1];
  const std::map<std::string, std::string> aliases = {{"-L", "--depth"}, {"-i", "--nests"}, {"--gamma", "--order"},
                                                      {"-A", "--matrix"}, {"-b", "--rhs"}};
  try {
    const Options o(argc, argv, aliases, {"--estimate-kappa"});
    if (cmd == "gen-matrix") return gen_matrix(o);
    if (cmd == "invert") return invert(o);
    if (cmd == "solve") return solve(o);
    if (cmd == "bench") return bench(o);
    if (cmd == "analyze-cost") throw DomainError("analyze-cost: the cost model is outside the B200 build");
    if (cmd == "-h" || cmd == "--help") {
      usage(std::cout);
      return 0;
    }
    throw UsageError("unknown subcommand '" + cmd + "'");
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    usage(std::cerr);
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
