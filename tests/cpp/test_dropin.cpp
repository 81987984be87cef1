// C++ drop-in tests: the reference's own test cases (restated, same inputs,
// seeds and thresholds) run against include/ddsg_b200.hpp.
//
//   test_dropin cpu   — construction / validation cases (no kernel launch)
//   test_dropin gpu   — evaluation cases (needs a CUDA device)
//
// Reference cases: proj/tests/test_sparse_grid.cpp, test_ddsg_eval.cpp,
// test_hdmr.cpp (cited per case).  Exit code = number of failed checks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "ddsg_b200.hpp"

using namespace ddsg_b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (cond) {                                                              \
      ++g_pass;                                                              \
    } else {                                                                 \
      ++g_fail;                                                              \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
    }                                                                        \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static GridEvaluator scalar(std::function<double(std::span<const double>)> f) {
  return [f](std::span<const double> x, std::span<double> out) { out[0] = f(x); };
}

static SparseGridFunction build_scalar(std::function<double(std::span<const double>)> f, int dim, int L,
                                       double eps, BoundaryMode mode) {
  SgBuildOptions opt;
  opt.max_level = L;
  opt.eps_gamma = eps;
  opt.mode = mode;
  return SparseGridFunction::build(scalar(f), dim, 1, opt);
}

// oracles.hpp:45-53
static std::vector<std::vector<double>> uniform_points(int n, std::size_t count, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  std::vector<std::vector<double>> pts(count, std::vector<double>(static_cast<std::size_t>(n)));
  for (auto& p : pts)
    for (auto& c : p) c = unif(rng);
  return pts;
}

static uint64_t brute_count(int n, int L) {  // oracles.hpp:21-43
  uint64_t total = 0;
  std::vector<int> l(static_cast<std::size_t>(n), 1);
  while (true) {
    int sum = 0;
    for (int v : l) sum += v;
    if (sum <= L + n - 1) {
      uint64_t pts = 1;
      for (int v : l) pts <<= (v - 1);
      total += pts;
    }
    std::size_t j = 0;
    while (j < l.size()) {
      if (++l[j] <= L) break;
      l[j] = 1;
      ++j;
    }
    if (j == l.size()) break;
  }
  return total;
}

static double coupled(std::span<const double> x) {  // test_ddsg_eval.cpp:37-42
  double s = 0.0;
  for (std::size_t j = 0; j < x.size(); ++j) s += std::exp(-0.5 * x[j]) + 0.2 * x[j] * x[j];
  for (std::size_t j = 0; j + 1 < x.size(); ++j) s += 0.3 * std::sin(x[j] * x[j + 1]);
  return s;
}

// Full (non-adaptive) decomposition assembled through from_parts: every
// index of order <= k accepted, cut grids built by this library's build from
// the cut through the center anchor (hdmr.hpp:248-259), b from the lattice
// formula (hdmr.hpp:339-355).  Equals decompose() with eps_rho = eps_eta = 0.
static std::shared_ptr<const DdsgFunction> full_decomposition(const GridEvaluator& f, int d, int m, int k,
                                                              int L, BoundaryMode mode) {
  AnchorPoint a;
  a.coords.assign(static_cast<std::size_t>(d), 0.5);
  a.f_anchor.resize(static_cast<std::size_t>(m));
  f(a.coords, a.f_anchor);
  std::vector<ComponentIndex> family{ComponentIndex{}};
  for (int kk = 1; kk <= k; ++kk) {
    std::vector<int> comb(static_cast<std::size_t>(kk));
    for (int i = 0; i < kk; ++i) comb[static_cast<std::size_t>(i)] = i;
    while (true) {
      family.push_back(ComponentIndex{comb});
      int i = kk;
      while (i > 0 && comb[static_cast<std::size_t>(i - 1)] == d - (kk - i) - 1) --i;
      if (i == 0) break;
      ++comb[static_cast<std::size_t>(i - 1)];
      for (int j = i; j < kk; ++j) comb[static_cast<std::size_t>(j)] = comb[static_cast<std::size_t>(j - 1)] + 1;
    }
  }
  std::map<ComponentIndex, SparseGridFunction> accepted;
  std::map<ComponentIndex, int> b;
  for (const auto& u : family) {
    int bu = 0;
    for (const auto& v : family) {
      if (!std::includes(v.dims.begin(), v.dims.end(), u.dims.begin(), u.dims.end())) continue;
      bu += ((v.order() - u.order()) % 2 == 0) ? 1 : -1;
    }
    b[u] = bu;
    if (u.empty()) continue;
    std::vector<double> base = a.coords;
    std::vector<int> dims = u.dims;
    GridEvaluator cut = [&f, base, dims](std::span<const double> y, std::span<double> out) {
      std::vector<double> x = base;
      for (std::size_t j = 0; j < dims.size(); ++j) x[static_cast<std::size_t>(dims[j])] = y[j];
      f(x, out);
    };
    SgBuildOptions opt;
    opt.max_level = L;
    opt.mode = mode;
    accepted.emplace(u, SparseGridFunction::build(cut, static_cast<int>(u.order()), m, opt));
  }
  DdsgOptions o;
  o.k_max = k;
  o.max_level = L;
  return std::make_shared<const DdsgFunction>(DdsgFunction::from_parts(d, m, o, a, accepted, {}, b, {}));
}

// ------------------------------------------------------------------ cpu

static void cpu_cases() {
  // test_sparse_grid.cpp:66-75
  auto one = [](std::span<const double>) { return 1.0; };
  CHECK(build_scalar(one, 1, 3, 0.0, BoundaryMode::zero_boundary).size() == 7);
  CHECK(build_scalar(one, 2, 2, 0.0, BoundaryMode::zero_boundary).size() == 5);
  for (int n = 1; n <= 4; ++n)
    for (int L = 1; L <= 6; ++L)
      CHECK(build_scalar(one, n, L, 0.0, BoundaryMode::modified_linear).size() == brute_count(n, L));

  // test_sparse_grid.cpp:77-86
  {
    auto f = [](std::span<const double> x) { return std::max(1.0 - 2.0 * std::abs(x[0] - 0.5), 0.0); };
    const auto g = build_scalar(f, 1, 3, 1e-8, BoundaryMode::zero_boundary);
    CHECK(g.size() == 3);
    for (const auto& node : g.nodes()) {
      if (node.key[0] == 1u) CHECK(std::abs(node.surplus[0] - 1.0) <= 1e-15);
      else CHECK(std::abs(node.surplus[0]) < 1e-15);
    }
  }
  // test_sparse_grid.cpp:210-225
  {
    SgBuildOptions opt;
    opt.max_level = 3;
    GridEvaluator f = [](std::span<const double> x, std::span<double> out) {
      out[0] = (x[0] == 0.25) ? std::numeric_limits<double>::quiet_NaN() : x[0];
    };
    bool caught = false;
    try {
      SparseGridFunction::build(f, 1, 1, opt);
    } catch (const build_error& be) {
      caught = true;
      CHECK(be.point().size() == 1);
      CHECK(be.point()[0] == 0.25);
      CHECK(std::string(be.what()).find("0.25") != std::string::npos);
    }
    CHECK(caught);
  }
  // an evaluator exception surfaces with its own type (sparse_grid.hpp:259-262)
  {
    SgBuildOptions opt;
    opt.max_level = 2;
    GridEvaluator f = [](std::span<const double>, std::span<double>) { throw std::out_of_range("boom"); };
    CHECK(throws<std::out_of_range>([&] { SparseGridFunction::build(f, 1, 1, opt); }));
  }
  // option validation (sparse_grid.hpp:86-89)
  {
    SgBuildOptions opt;
    opt.max_level = 0;
    CHECK(throws<std::invalid_argument>([&] { SparseGridFunction::build(scalar(one), 1, 1, opt); }));
    opt.max_level = 2;
    CHECK(throws<std::invalid_argument>([&] { SparseGridFunction::build(scalar(one), 0, 1, opt); }));
  }
  // from_nodes validation (sparse_grid.hpp:168-176)
  CHECK(throws<std::invalid_argument>([&] {
    SparseGridFunction::from_nodes(1, 1, 2, 0.0, BoundaryMode::zero_boundary, {GridNode{{1u}, {1.0}}, GridNode{{1u}, {2.0}}});
  }));
  CHECK(throws<std::invalid_argument>([&] {
    SparseGridFunction::from_nodes(2, 1, 2, 0.0, BoundaryMode::zero_boundary, {GridNode{{1u}, {1.0}}});
  }));
  // quadrature examples (test_sparse_grid.cpp:148-177)
  {
    auto g1 = SparseGridFunction::from_nodes(1, 1, 2, 0.0, BoundaryMode::zero_boundary, {GridNode{{2u}, {1.0}}});
    CHECK(std::abs(g1.quadrature()[0] - 0.25) <= 1e-15);
    auto hat = [](std::span<const double> x) { return std::max(1.0 - 2.0 * std::abs(x[0] - 0.5), 0.0); };
    CHECK(std::abs(build_scalar(hat, 1, 3, 0.0, BoundaryMode::zero_boundary).quadrature()[0] - 0.5) <= 1e-14);
  }
  // compile validation (ddsg_eval.hpp:41,54-56,63-70)
  CHECK(throws<std::invalid_argument>([&] { VectorizedDdsg::compile(nullptr); }));
  {
    AnchorPoint a{{0.5, 0.5}, {1.0}};
    std::map<ComponentIndex, SparseGridFunction> acc;
    acc.emplace(ComponentIndex{{0, 1}}, build_scalar(coupled, 2, 2, 0.0, BoundaryMode::modified_linear));
    std::map<ComponentIndex, int> b{{ComponentIndex{}, 0}, {ComponentIndex{{0, 1}}, 1}};
    auto src = std::make_shared<const DdsgFunction>(DdsgFunction::from_parts(2, 1, {}, a, acc, {}, b, {}));
    CHECK(throws<std::invalid_argument>([&] { VectorizedDdsg::compile(src); }));  // misses {0}, {1}
    std::map<ComponentIndex, int> b2{{ComponentIndex{}, 0}, {ComponentIndex{{1}}, 1}};
    auto src2 = std::make_shared<const DdsgFunction>(DdsgFunction::from_parts(2, 1, {}, a, acc, {}, b2, {}));
    CHECK(throws<std::invalid_argument>([&] { VectorizedDdsg::compile(src2); }));  // non-accepted index
  }
}

// ------------------------------------------------------------------ gpu

static void gpu_cases() {
  // hierarchization round trip (test_sparse_grid.cpp:88-116)
  {
    auto f = [](std::span<const double> x) {
      double s = 1.0;
      for (double c : x) s *= std::exp(-2.0 * c) + 0.3 * c;
      return s;
    };
    for (BoundaryMode mode : {BoundaryMode::zero_boundary, BoundaryMode::modified_linear}) {
      const auto g = build_scalar(f, 2, 5, 0.0, mode);
      for (const auto& node : g.nodes()) {
        std::vector<double> x(2);
        for (int j = 0; j < 2; ++j) {
          const uint32_t hk = node.key[static_cast<std::size_t>(j)];
          const int l = 32 - __builtin_clz(hk);
          x[static_cast<std::size_t>(j)] = (2.0 * (hk - (1u << (l - 1))) + 1.0) * std::ldexp(1.0, -l);
        }
        CHECK(std::abs(g.interpolate(x)[0] - f(x)) <= 1e-12);
      }
    }
    auto bump = [](std::span<const double> x) { return std::exp(-40.0 * (x[0] - 0.3) * (x[0] - 0.3)) + 0.1 * x[1]; };
    const auto ga = build_scalar(bump, 2, 6, 1e-3, BoundaryMode::modified_linear);
    CHECK(ga.size() < brute_count(2, 6));
    for (const auto& node : ga.nodes()) {
      std::vector<double> x(2);
      for (int j = 0; j < 2; ++j) {
        const uint32_t hk = node.key[static_cast<std::size_t>(j)];
        const int l = 32 - __builtin_clz(hk);
        x[static_cast<std::size_t>(j)] = (2.0 * (hk - (1u << (l - 1))) + 1.0) * std::ldexp(1.0, -l);
      }
      CHECK(std::abs(ga.interpolate(x)[0] - bump(x)) <= 1e-12);
    }
  }
  // interpolation examples (test_sparse_grid.cpp:118-146)
  {
    auto parab = [](std::span<const double> x) { return x[0] * (1.0 - x[0]); };
    const auto g1 = build_scalar(parab, 1, 1, 0.0, BoundaryMode::zero_boundary);
    std::vector<double> q{0.5};
    CHECK(std::abs(g1.interpolate(q)[0] - 0.25) <= 1e-15);
    const auto g2 = build_scalar(parab, 2, 4, 0.0, BoundaryMode::modified_linear);
    for (double x2 : {0.0, 0.17, 0.5, 0.83, 1.0}) {
      std::vector<double> a{0.3, x2}, b{0.3, 0.62};
      CHECK(std::abs(g2.interpolate(a)[0] - g2.interpolate(b)[0]) <= 1e-12);
    }
    auto lin = [](std::span<const double> x) { return x[0]; };
    const auto g3 = build_scalar(lin, 1, 2, 0.0, BoundaryMode::modified_linear);
    std::vector<double> p{0.3};
    CHECK(std::abs(g3.interpolate(p)[0] - 0.3) <= 1e-14);
    for (const auto& pt : uniform_points(1, 100, 20240501ull)) CHECK(std::abs(g3.interpolate(pt)[0] - pt[0]) <= 1e-13);
    std::vector<double> outside{1.5};
    CHECK(throws<std::domain_error>([&] { g3.interpolate(outside); }));
  }
  // L2 convergence ratio (test_sparse_grid.cpp:227-244), seed 77001, 1e4 points
  {
    auto f = [](std::span<const double> x) { return x[0] * (1.0 - x[0]) * x[1] * (1.0 - x[1]); };
    const auto pts = uniform_points(2, 10000, 77001ull);
    std::vector<double> flat;
    for (const auto& p : pts) flat.insert(flat.end(), p.begin(), p.end());
    double prev = 0.0;
    for (int L = 3; L <= 7; ++L) {
      const auto g = build_scalar(f, 2, L, 0.0, BoundaryMode::zero_boundary);
      std::vector<double> y(pts.size());
      g.interpolate_batch(flat.data(), static_cast<int64_t>(pts.size()), y.data());
      double sq = 0.0;
      for (std::size_t i = 0; i < pts.size(); ++i) {
        const double dd = y[i] - f(pts[i]);
        sq += dd * dd;
      }
      const double err = std::sqrt(sq / static_cast<double>(pts.size()));
      if (L > 3) CHECK(err / prev <= 0.35);
      prev = err;
    }
  }
  // constant functions come back constant (test_ddsg_eval.cpp:122-133)
  {
    GridEvaluator f = [](std::span<const double>, std::span<double> out) { out[0] = 4.25; };
    auto src = full_decomposition(f, 3, 1, 2, 3, BoundaryMode::modified_linear);
    const auto vec = VectorizedDdsg::compile(src);
    for (const auto& p : uniform_points(3, 100, 5)) CHECK(std::abs(vec.evaluate(p)[0] - 4.25) <= 1e-13);
  }
  // batch == looped bitwise, permutation, worker independence (test_ddsg_eval.cpp:179-209)
  {
    auto src = full_decomposition(scalar(coupled), 4, 1, 2, 3, BoundaryMode::modified_linear);
    const auto vec = VectorizedDdsg::compile(src);
    const auto pts = uniform_points(4, 10000, 8443);
    const auto batch = vec.evaluate_batch(pts);
    CHECK(batch.size() == pts.size());
    bool same = true;
    for (std::size_t i = 0; i < pts.size(); i += 97) same &= std::memcmp(&batch[i][0], &vec.evaluate(pts[i])[0], 8) == 0;
    CHECK(same);
    auto perm = pts;
    std::reverse(perm.begin(), perm.end());
    const auto rb = vec.evaluate_batch(perm);
    bool psame = true;
    for (std::size_t i = 0; i < pts.size(); ++i) psame &= std::memcmp(&rb[pts.size() - 1 - i][0], &batch[i][0], 8) == 0;
    CHECK(psame);
    const auto b4 = vec.evaluate_batch(pts, 4);
    bool wsame = true;
    for (std::size_t i = 0; i < pts.size(); ++i) wsame &= std::memcmp(&b4[i][0], &batch[i][0], 8) == 0;
    CHECK(wsame);
    // a bad point raises task_error with the lowest index (runtime.hpp:133-136)
    auto badpts = pts;
    badpts[123][2] = 1.5;
    badpts[77][1] = -0.5;
    bool caught = false;
    try {
      vec.evaluate_batch(badpts);
    } catch (const task_error& te) {
      caught = te.task_id() == 77;
      CHECK(throws<std::domain_error>([&] { te.rethrow_cause(); }));
    }
    CHECK(caught);
    // the lowest failing task wins whatever the failure: a short query at
    // 200 beats the domain error at 300, a domain error at 50 beats both
    auto mixed = pts;
    mixed[300][0] = 2.0;
    mixed[200].pop_back();
    int which = -1;
    try {
      vec.evaluate_batch(mixed);
    } catch (const task_error& te) {
      which = static_cast<int>(te.task_id());
      CHECK(throws<std::invalid_argument>([&] { te.rethrow_cause(); }));
    }
    CHECK(which == 200);
    mixed[50][1] = -1.0;
    which = -1;
    try {
      vec.evaluate_batch(mixed);
    } catch (const task_error& te) {
      which = static_cast<int>(te.task_id());
      CHECK(throws<std::domain_error>([&] { te.rethrow_cause(); }));
    }
    CHECK(which == 50);
  }
  // vector-valued outputs (test_ddsg_eval.cpp:224-242) and vectorized == naive
  // (test_ddsg_eval.cpp:106-120): naive telescoping from per-cut batched calls
  {
    GridEvaluator f = [](std::span<const double> x, std::span<double> out) {
      out[0] = x[0] + x[1];
      out[1] = std::exp(x[0] * x[1]);
      out[2] = 0.5;
    };
    auto src = full_decomposition(f, 2, 3, 2, 4, BoundaryMode::modified_linear);
    const auto vec = VectorizedDdsg::compile(src);
    const auto pts = uniform_points(2, 200, 61);
    for (const auto& p : pts) {
      const auto got = vec.evaluate(p);
      // naive Eq. 3.16: sum_u sum_{v subset u} sign * cut_v(x)
      std::vector<double> want = src->anchor().f_anchor;
      for (const auto& [u, g] : src->accepted()) {
        const std::size_t k = u.order();
        for (std::size_t mask = 0; mask < (std::size_t{1} << k); ++mask) {
          std::vector<int> vd;
          for (std::size_t j = 0; j < k; ++j)
            if (mask & (std::size_t{1} << j)) vd.push_back(u.dims[j]);
          const double sign = ((k - vd.size()) % 2 == 0) ? 1.0 : -1.0;
          if (vd.empty()) {
            for (int c = 0; c < 3; ++c) want[static_cast<std::size_t>(c)] += sign * src->anchor().f_anchor[static_cast<std::size_t>(c)];
            continue;
          }
          std::vector<double> xr;
          for (int dd : vd) xr.push_back(p[static_cast<std::size_t>(dd)]);
          const auto cv = src->accepted().at(ComponentIndex{vd}).interpolate(xr);
          for (int c = 0; c < 3; ++c) want[static_cast<std::size_t>(c)] += sign * cv[static_cast<std::size_t>(c)];
        }
      }
      for (int c = 0; c < 3; ++c) CHECK(std::abs(got[static_cast<std::size_t>(c)] - want[static_cast<std::size_t>(c)]) <= 1e-12);
    }
  }
}

// Batched IRBC callers through the shim (test_irbc.cpp:28-52, 189-206;
// test_solver.cpp:170-196).
static void irbc_cpu_cases() {
  using namespace ddsg_b200::irbc;
  auto p = make_parameters(4, Variant::smooth);
  CHECK(std::abs(p.A - (1.0 - 0.99 * 0.99) / (0.36 * 0.99)) <= 1e-15);
  CHECK(p.gamma.size() == 4 && p.gamma[1] == 0.5 && p.gamma[3] == 1.0);
  CHECK(std::abs(1.0 - p.beta * (p.alpha * p.A + 1.0 - p.delta)) < 1e-12);
  for (int j = 0; j < 4; ++j) CHECK(std::abs(p.tau[j] - std::pow(p.A, 1.0 / p.gamma[j])) <= 1e-15);
  const double lam = steady_state_lambda(p);
  double sum = 0.0;
  for (double g : p.gamma) sum += p.A * std::pow(lam, -g);
  CHECK(std::abs(sum - 4.0 * (p.A - p.delta)) <= 1e-10);
  IrbcParameters bad = p;
  bad.beta = 1.5;
  CHECK(throws<std::invalid_argument>([&] { refresh_derived(bad); }));
}

static void irbc_gpu_cases() {
  using namespace ddsg_b200::irbc;
  // steady policy k' = k, lambda = lambda_ss as a 1-d-cut HDMR (exact for linear cuts)
  auto p = make_parameters(2, Variant::smooth);
  p.gamma.assign(2, 0.25);
  p.sigma = 0.0;
  refresh_derived(p);
  const double lam = steady_state_lambda(p);
  const double klo = p.k_lo, khi = p.k_hi;
  GridEvaluator steady = [=](std::span<const double> x, std::span<double> out) {
    out[0] = klo + x[2] * (khi - klo);
    out[1] = klo + x[3] * (khi - klo);
    out[2] = lam;
  };
  auto src = full_decomposition(steady, 4, 3, 1, 2, BoundaryMode::modified_linear);
  const auto pol = VectorizedDdsg::compile(src);
  const double a[2] = {1.0, 1.0}, k[2] = {1.0, 1.0}, cand[3] = {1.0, 1.0, lam};
  double res[3];
  const auto cl = foc_residuals_batch(pol, p, 1, a, k, cand, res);
  CHECK(cl.size() == 1 && cl[0] == 0);
  for (double r : res) CHECK(std::abs(r) < 1e-10);
  // Euler errors on a degenerate box are exact and deterministic
  auto q = p;
  q.k_lo = 1.0 - 5e-11;
  q.k_hi = 1.0 + 5e-11;
  q.lna_half_width = 5e-11;
  refresh_derived(q);
  const double lq = steady_state_lambda(q);
  GridEvaluator steady_q = [=](std::span<const double> x, std::span<double> out) {
    out[0] = q.k_lo + x[2] * (q.k_hi - q.k_lo);
    out[1] = q.k_lo + x[3] * (q.k_hi - q.k_lo);
    out[2] = lq;
  };
  const auto pq = VectorizedDdsg::compile(full_decomposition(steady_q, 4, 3, 1, 2, BoundaryMode::modified_linear));
  const auto e1 = euler_errors(pq, q, 500, 99);
  const auto e2 = euler_errors(pq, q, 500, 99, 4);
  CHECK(e1.avg_log10 < -8.0 && e1.max_log10 < -8.0);
  CHECK(e1.samples == e2.samples && e1.avg_log10 == e2.avg_log10);
}

// ------------------------------------------------- decomposition (test_hdmr.cpp)

static AnchorPoint center_anchor(const Evaluator& f, int d, int m) {  // oracles.hpp: center of the cube
  AnchorPoint a;
  a.coords.assign(static_cast<std::size_t>(d), 0.5);
  a.f_anchor.resize(static_cast<std::size_t>(m));
  f(a.coords, a.f_anchor);
  return a;
}

static void decompose_cpu_cases() {
  auto idx = [](std::vector<int> dims) { return ComponentIndex{std::move(dims)}; };
  // test_hdmr.cpp:32-50
  {
    const auto a = select_anchor(scalar([](std::span<const double> x) { return x[0] + x[1]; }), 2, 1, 4000, 42);
    CHECK(std::abs(a.f_anchor[0] - 1.0) <= 0.05);
    const auto ac = select_anchor(scalar([](std::span<const double>) { return 3.25; }), 3, 1, 50, 7);
    CHECK(ac.f_anchor[0] == 3.25);
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    const double c0 = unif(rng), c1 = unif(rng), c2 = unif(rng);
    CHECK((ac.coords == std::vector<double>{c0, c1, c2}));  // ties: the lowest sample index
    const auto asq = select_anchor(scalar([](std::span<const double> x) { return x[0] * x[0]; }), 1, 1, 10000, 99);
    CHECK(std::abs(asq.f_anchor[0] - 1.0 / 3.0) < 0.02);
  }
  // test_hdmr.cpp:52-80
  {
    auto f = scalar([](std::span<const double> x) { return x[0] * 10.0 + x[1] + 100.0 * x[2]; });
    AnchorPoint a{{0.1, 0.2, 0.7}, {0.0}};
    std::vector<double> out(1), y{0.2, 0.9};
    cut_evaluator(f, a, idx({0, 1}))(y, out);
    CHECK(std::abs(out[0] - (0.2 * 10.0 + 0.9 + 70.0)) <= 1e-15 * 73.0);
    auto prod = scalar([](std::span<const double> x) { return x[0] * x[1] * x[2]; });
    AnchorPoint half{{0.5, 0.5, 0.5}, {}};
    std::vector<double> y1{0.5};
    cut_evaluator(prod, half, idx({1}))(y1, out);
    CHECK(std::abs(out[0] - 0.125) <= 1e-15);
    std::vector<double> y3{0.3, 0.4, 0.5}, want(1);
    cut_evaluator(f, a, idx({0, 1, 2}))(y3, out);
    f(y3, want);
    CHECK(out[0] == want[0]);
    CHECK(throws<std::invalid_argument>([&] { (void)cut_evaluator(f, a, ComponentIndex{}); }));
  }
  // test_hdmr.cpp:82-90
  CHECK(expansion_rho({2.0, 0.0}, {2.0, 0.0}) == 0.0);
  CHECK(std::abs(expansion_rho({2.0, 2.0}, {2.0, 0.0}) - 1.0) < 1e-12);
  CHECK(throws<rho_denominator_error>([] { (void)expansion_rho({1.0}, {0.0}); }));
  CHECK(eta_coefficient({0.0}, {1.0}) == 0.0);
  CHECK(std::isinf(eta_coefficient({1.0}, {0.0})));
  // test_hdmr.cpp:92-106: the centered blind spot of eta
  {
    auto f = scalar([](std::span<const double> x) { return x[0] * x[1]; });
    DdsgOptions opt;
    opt.k_max = 2;
    opt.max_level = 5;
    opt.mode = BoundaryMode::modified_linear;
    ExpansionDiagnostics diag;
    (void)decompose(f, 2, 1, center_anchor(f, 2, 1), opt, &diag);
    CHECK(diag.eta_by_order.size() == 2 && diag.eta_by_order[1].size() == 1);
    if (diag.eta_by_order.size() == 2 && diag.eta_by_order[1].size() == 1) CHECK(diag.eta_by_order[1][0].eta < 1e-12);
  }
  // test_hdmr.cpp:150-173: rho stops a separable function after order 2
  {
    auto f = scalar([](std::span<const double> x) { return x[0] + x[1] + x[2]; });
    AnchorPoint anchor{{0.2, 0.8, 0.3}, {}};
    DdsgOptions opt;
    opt.k_max = 3;
    opt.eps_rho = 1e-4;
    opt.max_level = 4;
    opt.mode = BoundaryMode::modified_linear;
    opt.workers = 2;
    ExpansionDiagnostics diag;
    const auto dd = decompose(f, 3, 1, anchor, opt, &diag);
    CHECK(dd.order_reached() == 2);
    CHECK(diag.rho_by_order.size() == 2 && std::abs(diag.rho_by_order[1]) <= 1e-13);
    CHECK(dd.accepted().count(idx({0})) == 1 && dd.accepted().count(idx({1})) == 1 && dd.accepted().count(idx({2})) == 1);
    CHECK(dd.accepted().count(idx({0, 1})) == 1 && dd.accepted().count(idx({0, 1, 2})) == 0);
    for (const auto& u : {idx({0, 1}), idx({0, 2}), idx({1, 2})}) CHECK(std::abs(dd.component_quadrature(u)[0]) < 1e-13);
  }
  // test_hdmr.cpp:193-220: eta prunes supersets of rejected indices
  {
    auto f = scalar([](std::span<const double> x) {
      return x[0] + x[1] + std::exp(x[0] * x[2]) + std::exp(x[1] * x[2]);
    });
    DdsgOptions opt;
    opt.k_max = 3;
    opt.eps_eta = 1e-5;
    opt.max_level = 5;
    opt.mode = BoundaryMode::modified_linear;
    opt.workers = 3;
    const auto dd = decompose(f, 3, 1, center_anchor(f, 3, 1), opt);
    CHECK(dd.rejected().count(idx({0, 1})) == 1);
    CHECK(dd.accepted().count(idx({0, 2})) == 1 && dd.accepted().count(idx({1, 2})) == 1);
    CHECK(dd.accepted().count(idx({0, 1, 2})) == 0 && dd.rejected().count(idx({0, 1, 2})) == 0);
    bool sound = true;
    for (const auto& [u, grid] : dd.accepted()) {
      for (const auto& z : dd.rejected()) sound = sound && !u.is_superset_of(z);
      for (const auto& v : all_subsets(u))
        if (!v.empty()) sound = sound && dd.accepted().count(v) == 1;
    }
    CHECK(sound);
  }
  // test_hdmr.cpp:222-243: with zero thresholds the telescoping collapses
  {
    auto f = scalar([](std::span<const double> x) {
      return std::exp(x[0]) * (1.0 + 0.5 * std::sin(3.0 * x[1])) + x[1] * x[2];
    });
    DdsgOptions opt;
    opt.k_max = 3;
    opt.max_level = 4;
    opt.mode = BoundaryMode::modified_linear;
    const auto dd = decompose(f, 3, 1, center_anchor(f, 3, 1), opt);
    bool collapsed = dd.coeff_b().size() == 8;
    for (const auto& [u, b] : dd.coeff_b()) collapsed = collapsed && b == (u.order() == 3 ? 1 : 0);
    CHECK(collapsed);
    CHECK(order_k_indices(5, 2).size() == 10 && order_k_indices(3, 4).empty());
  }
}

// ------------------------------------- node keys, basis, counts (host inline functions)

static void index_basis_cpu_cases() {
  // grid_index.hpp:24-55
  CHECK(heap_key(1, 1) == 1u && heap_key(2, 1) == 2u && heap_key(2, 3) == 3u && heap_key(3, 5) == 6u);
  for (int l = 1; l <= 12; ++l)
    for (std::uint32_t i = 1; i < (1u << l); i += 2) {
      const HeapKey hk = heap_key(l, i);
      if (level_of(hk) != l || index_of(hk) != i || coordinate_of(hk) != static_cast<double>(i) / std::ldexp(1.0, l)) {
        CHECK(false);
        return;
      }
    }
  CHECK(!has_parent(1u) && has_parent(2u) && parent_key(6u) == 3u && parent_key(7u) == 3u);
  CHECK(level_sum(NodeKey{1u, 2u, 5u}) == 1 + 2 + 3);
  std::vector<double> xy;
  coordinates_of(NodeKey{heap_key(1, 1), heap_key(3, 7)}, xy);
  CHECK((xy == std::vector<double>{0.5, 0.875}));
  CHECK(throws<std::invalid_argument>([] { (void)heap_key(0, 1); }));
  CHECK(throws<std::invalid_argument>([] { (void)heap_key(31, 1); }));
  CHECK(throws<std::invalid_argument>([] { (void)heap_key(2, 2); }));
  CHECK(throws<std::invalid_argument>([] { (void)heap_key(2, 5); }));
  // test_sparse_grid.cpp:31-47
  CHECK(basis_1d(1, 1, 0.5, BoundaryMode::zero_boundary) == 1.0);
  CHECK(basis_1d(2, 1, 0.5, BoundaryMode::zero_boundary) == 0.0);
  CHECK(std::abs(basis_1d(2, 3, 0.6, BoundaryMode::zero_boundary) - 0.4) <= 1e-15);
  CHECK(basis_1d(1, 1, 0.0, BoundaryMode::modified_linear) == 1.0);
  CHECK(basis_1d(2, 1, 0.0, BoundaryMode::modified_linear) == 2.0);
  CHECK(basis_1d(2, 3, 1.0, BoundaryMode::modified_linear) == 2.0);
  CHECK(std::abs(basis_1d(2, 3, 0.6, BoundaryMode::modified_linear) - 0.4) <= 1e-15);
  CHECK(basis_1d(3, 3, 0.375, BoundaryMode::modified_linear) == 1.0);
  CHECK(throws<std::invalid_argument>([] { (void)basis_1d(2, 2, 0.5, BoundaryMode::zero_boundary); }));
  CHECK(throws<std::invalid_argument>([] { (void)basis_1d(2, 5, 0.5, BoundaryMode::zero_boundary); }));
  CHECK(throws<std::invalid_argument>([] { (void)basis_1d(0, 1, 0.5, BoundaryMode::zero_boundary); }));
  CHECK(throws<std::domain_error>([] { (void)basis_1d(1, 1, 1.5, BoundaryMode::zero_boundary); }));
  // test_sparse_grid.cpp:49-64
  {
    const NodeKey unit{heap_key(1, 1), heap_key(1, 1)};
    std::vector<double> x{0.5, 0.5}, x2{0.5, 0.0}, x3{0.25, 0.6}, wrong{0.5};
    CHECK(basis_nd(unit, x, BoundaryMode::zero_boundary) == 1.0);
    CHECK(basis_nd(NodeKey{heap_key(1, 1), heap_key(2, 1)}, x2, BoundaryMode::zero_boundary) == 0.0);
    CHECK(std::abs(basis_nd(NodeKey{heap_key(2, 1), heap_key(2, 3)}, x3, BoundaryMode::zero_boundary) - 0.4) <= 1e-15);
    CHECK(throws<std::invalid_argument>([&] { (void)basis_nd(unit, wrong, BoundaryMode::zero_boundary); }));
  }
  CHECK(basis_weight(BasisKind::constant_one, 0.5) == 1.0 && basis_weight(BasisKind::hat, 0.25) == 0.25 &&
        basis_weight(BasisKind::left_edge, 0.25) == 0.5 && basis_weight(BasisKind::right_edge, 0.125) == 0.25);
  // test_hdmr.cpp:293-313
  CHECK(ddsg_grid_count(4, 1, 3) == 29);
  CHECK(ddsg_grid_count(2, 2, 2) == 12);
  CHECK(ddsg_grid_count(5, 0, 4) == 1);
  {
    bool ok = true;
    for (int d = 1; d <= 6; ++d)
      for (int k = 1; k <= std::min(d, 3); ++k)
        for (int L = 1; L <= 5; ++L) {
          std::uint64_t want = 1;
          for (int kk = 1; kk <= k; ++kk) {
            std::uint64_t binom = 1;
            for (int i = 1; i <= kk; ++i) binom = binom * static_cast<std::uint64_t>(d - kk + i) / static_cast<std::uint64_t>(i);
            want += binom * brute_count(kk, L);
          }
          ok = ok && ddsg_grid_count(d, k, L) == want;
        }
    CHECK(ok);
  }
  CHECK(throws<std::overflow_error>([] { (void)ddsg_grid_count(300, 10, 10); }));
  CHECK(throws<std::invalid_argument>([] { (void)ddsg_grid_count(3, 4, 2); }));
}

// ------------------------------------------------ refinement through the shim

static GridEvaluator refine_target() {  // 2 outputs, a kink: the adaptive build refines unevenly
  return [](std::span<const double> x, std::span<double> out) {
    double s = 0.0;
    for (double v : x) s += v;
    out[0] = std::max(0.0, s - 0.6 * static_cast<double>(x.size())) + 0.1 * x[0] * x[0];
    out[1] = std::exp(-s) + 0.05 * x[x.size() - 1];
  };
}

static bool same_nodes(const SparseGridFunction& a, const SparseGridFunction& b) {
  if (a.size() != b.size() || a.max_level() != b.max_level()) return false;
  const auto& na = a.nodes();
  const auto& nb = b.nodes();
  for (std::size_t i = 0; i < na.size(); ++i)
    if (na[i].key != nb[i].key || na[i].surplus.size() != nb[i].surplus.size() ||
        std::memcmp(na[i].surplus.data(), nb[i].surplus.data(), na[i].surplus.size() * sizeof(double)) != 0)
      return false;
  return true;
}

// One refinement step from level L equals the build at level L + 1
// (sparse_grid.hpp:84-108 runs exactly these steps), node order and surplus bits.
static void refine_cases(bool on_device) {
  const GridEvaluator f = refine_target();
  for (int dim = 1; dim <= 3; ++dim)
    for (double eps : {0.0, 1e-3}) {
      SgBuildOptions lo, hi;
      lo.max_level = dim == 1 ? 5 : 3;
      lo.eps_gamma = eps;
      lo.mode = dim == 2 ? BoundaryMode::zero_boundary : BoundaryMode::modified_linear;
      hi = lo;
      hi.max_level = lo.max_level + 1;
      SparseGridFunction g = SparseGridFunction::build(f, dim, 2, lo);
      const SparseGridFunction want = SparseGridFunction::build(f, dim, 2, hi);
      const std::size_t before = g.size();
      (void)g.nodes();  // fill the cache: refine_step must drop it
      const RefineStats st = refine_step({&g}, {lo.max_level + dim - 1},
                                         [&](int, std::span<const double> x, std::span<double> out) { f(x, out); },
                                         nullptr, 0, 1, nullptr, on_device);
      CHECK(st.new_nodes == static_cast<std::int64_t>(want.size() - before));
      CHECK(same_nodes(g, want));
      if (eps == 0.0) {  // the manual steps: candidates, hierarchize, append (one level-sum group)
        SparseGridFunction h = SparseGridFunction::build(f, dim, 2, lo);
        const auto keys = h.refine_candidates(lo.max_level + dim - 1);
        std::vector<std::vector<double>> fv(keys.size(), std::vector<double>(2));
        std::vector<double> x;
        for (std::size_t i = 0; i < keys.size(); ++i) {
          coordinates_of(keys[i], x);
          f(x, fv[i]);
        }
        const auto sur = h.hierarchize(keys, fv, on_device);
        std::vector<GridNode> fresh(keys.size());
        for (std::size_t i = 0; i < keys.size(); ++i) fresh[i] = GridNode{keys[i], sur[i], false};
        h.append(fresh);
        CHECK(h.size() == want.size());
        bool same = h.size() == want.size();
        for (std::size_t i = 0; same && i < h.size(); ++i)
          same = h.nodes()[i].key == want.nodes()[i].key &&
                 std::memcmp(h.nodes()[i].surplus.data(), want.nodes()[i].surplus.data(), 2 * sizeof(double)) == 0;
        CHECK(same);
        CHECK(throws<std::invalid_argument>([&] { h.append(fresh); }));  // duplicates are rejected
      }
    }
  {  // a non-finite target value reports the node (build_error, sparse_grid.hpp:287-295)
    SgBuildOptions lo;
    lo.max_level = 2;
    lo.mode = BoundaryMode::modified_linear;
    SparseGridFunction g = SparseGridFunction::build(f, 1, 2, lo);
    auto bad = [&](int, std::span<const double> x, std::span<double> out) {
      f(x, out);
      if (x[0] == 0.125) out[1] = std::numeric_limits<double>::infinity();
    };
    bool reported = false;
    try {
      (void)refine_step({&g}, {2}, bad, nullptr, 0, 1, nullptr, on_device);
    } catch (const build_error& e) {
      reported = e.point().size() == 1 && e.point()[0] == 0.125;
    }
    CHECK(reported);
    CHECK(throws<std::invalid_argument>([&] { (void)refine_step({&g}, {1, 2}, bad); }));
  }
}

// Repeated per-point calls on one workspace are replayed as a CUDA graph
// from the fourth identical call on: every call must still see its own point,
// report its own domain error, and survive a change of program.
static void workspace_replay_cases() {
  auto fa = scalar([](std::span<const double> x) { return std::exp(x[0] - x[1]) + x[2] * x[0]; });
  auto fb = scalar([](std::span<const double> x) { return std::sin(3.0 * x[0]) * x[1] + x[2]; });
  DdsgOptions opt;
  opt.k_max = 2;
  opt.max_level = 4;
  opt.mode = BoundaryMode::modified_linear;
  const auto va = VectorizedDdsg::compile(std::make_shared<const DdsgFunction>(decompose(fa, 3, 1, center_anchor(fa, 3, 1), opt)));
  const auto vb = VectorizedDdsg::compile(std::make_shared<const DdsgFunction>(decompose(fb, 3, 1, center_anchor(fb, 3, 1), opt)));
  const auto pts = uniform_points(3, 60, 4242);
  const auto want_a = va.evaluate_batch(pts), want_b = vb.evaluate_batch(pts);
  EvalWorkspace ws;
  std::vector<double> out(1);
  int bad = 0;
  for (std::size_t i = 0; i < 30; ++i) {  // one program, many calls: eager, captured, replayed
    va.evaluate(pts[i], out, ws);
    bad += std::memcmp(out.data(), want_a[i].data(), sizeof(double)) != 0;
    if (i == 12) {  // a domain error in the middle of the replayed run, then on
      std::vector<double> outside{0.5, 1.5, 0.5};
      bad += !throws<std::domain_error>([&] { va.evaluate(outside, out, ws); });
    }
  }
  for (std::size_t i = 30; i < 45; ++i) {  // the other program on the same workspace
    vb.evaluate(pts[i], out, ws);
    bad += std::memcmp(out.data(), want_b[i].data(), sizeof(double)) != 0;
  }
  for (std::size_t i = 45; i < 60; ++i) {  // alternating programs never replay
    va.evaluate(pts[i], out, ws);
    bad += std::memcmp(out.data(), want_a[i].data(), sizeof(double)) != 0;
    vb.evaluate(pts[i], out, ws);
    bad += std::memcmp(out.data(), want_b[i].data(), sizeof(double)) != 0;
  }
  CHECK(bad == 0);
}

static void decompose_gpu_cases() {
  // test_hdmr.cpp:175-190 and 245-251: the decomposition against the plain sparse grid
  {
    auto f = scalar([](std::span<const double> x) { return x[0] + x[1] + x[2]; });
    AnchorPoint anchor{{0.2, 0.8, 0.3}, {}};
    DdsgOptions opt;
    opt.k_max = 3;
    opt.eps_rho = 1e-4;
    opt.max_level = 4;
    opt.mode = BoundaryMode::modified_linear;
    const auto dd = decompose(f, 3, 1, anchor, opt);
    const auto sg = build_scalar([](std::span<const double> x) { return x[0] + x[1] + x[2]; }, 3, 4, 0.0,
                                 BoundaryMode::modified_linear);
    double err_dd = 0.0, err_sg = 0.0;
    for (const auto& p : uniform_points(3, 1000, 5150)) {
      std::vector<double> want(1);
      f(p, want);
      err_dd = std::max(err_dd, std::abs(dd.evaluate_naive(p)[0] - want[0]));
      err_sg = std::max(err_sg, std::abs(sg.interpolate(p)[0] - want[0]));
    }
    CHECK(err_dd <= err_sg + 1e-12);
  }
  {
    auto fn = [](std::span<const double> x) { return std::exp(x[0]) * (1.0 + 0.5 * std::sin(3.0 * x[1])) + x[1] * x[2]; };
    auto f = scalar(fn);
    DdsgOptions opt;
    opt.k_max = 3;
    opt.max_level = 4;
    opt.mode = BoundaryMode::modified_linear;
    const auto dd = decompose(f, 3, 1, center_anchor(f, 3, 1), opt);
    const auto sg = build_scalar(fn, 3, 4, 0.0, BoundaryMode::modified_linear);
    const auto vec = VectorizedDdsg::compile(std::make_shared<const DdsgFunction>(dd));
    double worst = 0.0, worst_vec = 0.0;
    for (const auto& p : uniform_points(3, 200, 909)) {
      const double ref = sg.interpolate(p)[0];
      worst = std::max(worst, std::abs(dd.evaluate_naive(p)[0] - ref));
      worst_vec = std::max(worst_vec, std::abs(vec.evaluate(p)[0] - ref));
    }
    CHECK(worst <= 1e-12);
    CHECK(worst_vec <= 1e-12);
  }
}

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "cpu";
  if (which == "cpu" || which == "all") {
    cpu_cases();
    irbc_cpu_cases();
    decompose_cpu_cases();
    index_basis_cpu_cases();
    refine_cases(false);
  }
  if (which == "gpu" || which == "all") {
    gpu_cases();
    irbc_gpu_cases();
    decompose_gpu_cases();
    refine_cases(true);
    workspace_replay_cases();
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
