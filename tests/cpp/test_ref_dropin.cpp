// TEST INFRASTRUCTURE: the reference headers (ddsg::, compiled in place from
// /root/reference/proj/include) beside the B200 shim (ddsg_b200::), driven
// through the reference's own call shapes with only the namespace changed.
// Built by `make -C oracle dropin` (where the reference exists) into
// oracle/_ref/test_ref_dropin; run by tests/test_cpp_dropin.py on the GPU.
//
//   1. ddsg::decompose (hdmr.hpp:364) builds a vector-valued decomposition
//      (adaptive cut grids, so stored node orders are not canonical);
//   2. INTEGRATION.md's to_b200() -- #included verbatim (to_b200.inc) --
//      converts it;
//   3. compiled_evaluator (time_iteration.hpp:86-91) is written once per
//      namespace, identical text; evaluate(x, out, ws, &calls)
//      (tools/ddsg.cpp:376), evaluate(x, out) and evaluate_batch(xs,
//      workers) must agree bit for bit, with equal interp_calls;
//   4. the reference writes policy.json (save_json(to_json(...)),
//      tools/ddsg.cpp:217); ddsg_b200::ddsg_from_json(load_json(path)) loads
//      it through the C-ABI (tools/ddsg.cpp:261-268 shape) and evaluates it
//      on the GPU bit-exactly; the shim's writer is read back by the
//      reference's ddsg_from_json, same bits;
//   5. slots(), cut quadratures, exception types;
//   6. ddsg_b200::decompose / select_anchor (the shim's own restatement of
//      hdmr.hpp:45-133,364-483) against ddsg::decompose: identical accepted /
//      rejected sets, b, cut grids, quadratures and eta / rho diagnostics.
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <functional>
#include <memory>
#include <random>
#include <span>
#include <string>
#include <vector>

#include <unistd.h>

#include "ddsg/ddsg_eval.hpp"
#include "ddsg/hdmr.hpp"
#include "ddsg/serialize.hpp"
#include "ddsg_b200.hpp"

#include "to_b200.inc"  // INTEGRATION.md, BEGIN/END to_b200, verbatim

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) {                                                            \
      ++g_pass;                                                            \
    } else {                                                               \
      ++g_fail;                                                            \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)

using PolicyEvaluator = std::function<void(std::span<const double>, std::span<double>)>;  // irbc.hpp:211

// time_iteration.hpp:86-91, once per namespace (identical text)
namespace ref_side {
using namespace ddsg;
inline PolicyEvaluator compiled_evaluator(std::shared_ptr<const VectorizedDdsg> vec) {
  return [vec](std::span<const double> x, std::span<double> out) {
    thread_local EvalWorkspace ws;
    vec->evaluate(x, out, ws);
  };
}
}  // namespace ref_side
namespace b200_side {
using namespace ddsg_b200;
inline PolicyEvaluator compiled_evaluator(std::shared_ptr<const VectorizedDdsg> vec) {
  return [vec](std::span<const double> x, std::span<double> out) {
    thread_local EvalWorkspace ws;
    vec->evaluate(x, out, ws);
  };
}
}  // namespace b200_side

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

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

// A kinked vector-valued target on [0,1]^6 (3 outputs) with sparse
// coupling: the cut grids refine adaptively, pairs without interaction are
// rejected by eta, and the coefficients include zero and negative b.
static void target(std::span<const double> x, std::span<double> out) {
  out[0] = std::exp(-0.5 * (x[0] + x[1])) + 0.3 * x[2] * x[3];
  out[1] = std::max(0.0, x[0] + x[4] - 1.1) + 0.1 * x[5] * x[5];
  out[2] = std::log(1.0 + x[3] + 0.5 * x[4]) + x[1];
}

int main() {
  const int d = 6, m = 3;
  ddsg::AnchorPoint anchor;
  anchor.coords.assign(d, 0.5);
  ddsg::DdsgOptions opt;
  opt.k_max = 2;
  opt.max_level = 5;
  opt.eps_gamma = 1e-3;
  opt.eps_eta = 1e-8;  // prunes the non-interacting pairs: a non-trivial rejected set
  opt.mode = ddsg::BoundaryMode::modified_linear;
  opt.workers = 4;
  auto dd = std::make_shared<const ddsg::DdsgFunction>(ddsg::decompose(target, d, m, anchor, opt));
  auto vec_ref = std::make_shared<const ddsg::VectorizedDdsg>(ddsg::VectorizedDdsg::compile(dd));
  auto vec_gpu = std::make_shared<const ddsg_b200::VectorizedDdsg>(to_b200(*dd));
  std::printf("decompose: %zu accepted, %zu rejected, %zu slots\n", dd->accepted().size(), dd->rejected().size(),
              vec_ref->slots().size());
  std::fflush(stdout);
  CHECK(!dd->rejected().empty());

  // seeded points, as oracles.hpp:45-53 (plus cell boundaries and the faces)
  std::mt19937_64 rng(2022);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  std::vector<std::vector<double>> pts(3000, std::vector<double>(d));
  for (auto& x : pts)
    for (auto& c : x) c = unif(rng);
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < d; ++j) pts[i][j] = static_cast<double>((i * 7 + j * 3) % 33) / 32.0;

  // 3. compiled_evaluator, counted evaluate, two-argument evaluate, batch
  {
    auto f_ref = ref_side::compiled_evaluator(vec_ref);
    auto f_gpu = b200_side::compiled_evaluator(vec_gpu);
    std::vector<double> a(m), b(m);
    int diff = 0;
    for (const auto& x : pts) {
      f_ref(x, a);
      f_gpu(x, b);
      diff += !same_bits(a, b);
    }
    CHECK(diff == 0);
    std::printf("compiled_evaluator: %d of %zu points differ\n", diff, pts.size());

    std::uint64_t calls_ref = 0, calls_gpu = 0;
    ddsg::EvalWorkspace ws_ref;
    ddsg_b200::EvalWorkspace ws_gpu;
    diff = 0;
    for (std::size_t i = 0; i < 256; ++i) {
      vec_ref->evaluate(pts[i], a, ws_ref, &calls_ref);
      vec_gpu->evaluate(pts[i], b, ws_gpu, &calls_gpu);
      diff += !same_bits(a, b);
    }
    CHECK(diff == 0);
    CHECK(calls_ref == calls_gpu && calls_ref > 0);
    std::uint64_t c2r = 0, c2g = 0;
    vec_ref->evaluate(pts[5], a, &c2r);
    vec_gpu->evaluate(pts[5], b, &c2g);
    CHECK(same_bits(a, b) && c2r == c2g);
    vec_ref->evaluate(pts[6], a);
    vec_gpu->evaluate(pts[6], b);
    CHECK(same_bits(a, b));

    const auto yr = vec_ref->evaluate_batch(pts, 4);
    const auto yg = vec_gpu->evaluate_batch(pts, 4);
    diff = 0;
    for (std::size_t i = 0; i < pts.size(); ++i) diff += !same_bits(yr[i], yg[i]);
    CHECK(diff == 0);
    std::printf("evaluate_batch: %d differ; interp_calls %llu / %llu\n", diff,
                static_cast<unsigned long long>(calls_ref), static_cast<unsigned long long>(calls_gpu));
  }

  // 5. slots(), quadratures, exceptions
  {
    const auto& sr = vec_ref->slots();
    const auto& sg = vec_gpu->slots();
    CHECK(sr.size() == sg.size());
    bool ok = sr.size() == sg.size();
    for (std::size_t i = 0; ok && i < sr.size(); ++i) {
      ok = ok && sr[i].index.dims == sg[i].index.dims && sr[i].b == sg[i].b;
      ok = ok && ((sr[i].grid == nullptr) == (sg[i].grid == nullptr));
      if (sr[i].grid && sg[i].grid) ok = ok && sr[i].grid->size() == sg[i].grid->size();
    }
    CHECK(ok);
    CHECK(same_bits(vec_ref->quadrature(), vec_gpu->quadrature()));
    const auto& src = vec_gpu->source();
    for (const auto& [u, b] : dd->coeff_b())
      CHECK(same_bits(dd->cut_quadrature(u), src.cut_quadrature(ddsg_b200::ComponentIndex{u.dims})));
    CHECK(src.rejected().size() == dd->rejected().size());
    for (const auto& [u, g] : dd->accepted())
      CHECK(same_bits(dd->component_quadrature(u), src.component_quadrature(ddsg_b200::ComponentIndex{u.dims})));
    CHECK(same_bits(dd->cumulative_quadrature(1), src.cumulative_quadrature(1)));
    CHECK(same_bits(dd->cumulative_quadrature(2), src.cumulative_quadrature(2)));
    {  // node lookup (sparse_grid.hpp:151-157)
      const auto& [u0, g0] = *dd->accepted().rbegin();
      const auto& gb = src.accepted().at(ddsg_b200::ComponentIndex{u0.dims});
      const auto& nd = g0.nodes()[g0.size() / 2];
      CHECK(gb.contains(nd.key) && same_bits(gb.node_at(nd.key).surplus, nd.surplus));
      ddsg_b200::NodeKey absent(nd.key.size(), (1u << 29) + 7u);
      CHECK(!gb.contains(absent) && !g0.contains(absent));
      CHECK(throws<std::out_of_range>([&] { (void)gb.node_at(absent); }));
      CHECK(&gb.nodes() == &gb.nodes());  // cached: a stable reference, like the reference's
    }
    CHECK(throws<std::out_of_range>([&] { (void)src.cut_quadrature(ddsg_b200::ComponentIndex{{0, 1, 2}}); }));
    std::vector<double> out(m), bad_x(d, 0.5), short_x(d - 1, 0.5);
    bad_x[3] = 1.5;
    ddsg_b200::EvalWorkspace ws;
    CHECK(throws<std::domain_error>([&] { vec_ref->evaluate(bad_x, out); }));
    CHECK(throws<std::domain_error>([&] { vec_gpu->evaluate(bad_x, out, ws); }));
    CHECK(throws<std::invalid_argument>([&] { vec_ref->evaluate(short_x, out); }));
    CHECK(throws<std::invalid_argument>([&] { vec_gpu->evaluate(short_x, out, ws); }));
    std::vector<double> short_out(m - 1);
    CHECK(throws<std::invalid_argument>([&] { vec_gpu->evaluate(pts[0], short_out, ws); }));
  }

  // 4. JSON documents: reference writes, B200 loads (C-ABI) and evaluates on
  //    the GPU; B200 writes, reference loads.
  {
    namespace fs = std::filesystem;
    const fs::path dir = fs::temp_directory_path() / ("ddsg_ref_dropin_" + std::to_string(::getpid()));
    fs::create_directories(dir);
    const std::string p_ref = (dir / "policy.json").string(), p_b200 = (dir / "policy_b200.json").string();
    ddsg::save_json(ddsg::to_json(*dd), p_ref);  // tools/ddsg.cpp:217
    auto loaded =
        std::make_shared<const ddsg_b200::DdsgFunction>(ddsg_b200::ddsg_from_json(ddsg_b200::load_json(p_ref)));
    auto vec_loaded = std::make_shared<const ddsg_b200::VectorizedDdsg>(ddsg_b200::VectorizedDdsg::compile(loaded));
    auto frozen = [vec_loaded](std::span<const double> x, std::span<double> out) {  // tools/ddsg.cpp:263-266
      thread_local ddsg_b200::EvalWorkspace ws;
      vec_loaded->evaluate(x, out, ws);
    };
    std::vector<double> a(m), b(m);
    int diff = 0;
    for (const auto& x : pts) {
      vec_ref->evaluate(x, a);
      frozen(x, b);
      diff += !same_bits(a, b);
    }
    CHECK(diff == 0);
    std::printf("reference-written policy.json on the GPU: %d of %zu points differ\n", diff, pts.size());
    CHECK(loaded->k_max() == dd->k_max());
    CHECK(loaded->rejected().size() == dd->rejected().size());
    CHECK(same_bits(loaded->anchor().coords, dd->anchor().coords));

    ddsg_b200::save_json(ddsg_b200::to_json(*loaded), p_b200);
    auto back = std::make_shared<const ddsg::DdsgFunction>(ddsg::ddsg_from_json(ddsg::load_json(p_b200)));
    auto vec_back = ddsg::VectorizedDdsg::compile(back);
    diff = 0;
    for (std::size_t i = 0; i < 500; ++i) {
      vec_ref->evaluate(pts[i], a);
      vec_back.evaluate(pts[i], b);
      diff += !same_bits(a, b);
    }
    CHECK(diff == 0);
    // the two documents hold the same values: re-serialising the read-back
    // with the reference gives the reference's own text
    CHECK(ddsg::to_json(*back) == ddsg::to_json(*dd));

    // one grid document both ways
    const auto& [u0, g0] = *std::next(dd->accepted().begin(), static_cast<std::ptrdiff_t>(dd->accepted().size() - 1));
    const std::string gdoc = ddsg::to_json(g0).dump(2);
    auto g_b200 = ddsg_b200::sparse_grid_from_json(ddsg_b200::JsonDocument{gdoc});
    CHECK(g_b200.size() == g0.size());
    auto g_back = ddsg::sparse_grid_from_json(nlohmann::json::parse(ddsg_b200::to_json(g_b200).text));
    bool nodes_same = g_back.size() == g0.size();
    for (std::size_t i = 0; nodes_same && i < g0.size(); ++i)
      nodes_same = g_back.nodes()[i].key == g0.nodes()[i].key && same_bits(g_back.nodes()[i].surplus, g0.nodes()[i].surplus);
    CHECK(nodes_same);
    CHECK(throws<std::invalid_argument>([] { (void)ddsg_b200::sparse_grid_from_json(ddsg_b200::JsonDocument{"{\"schema_version\": 2}"}); }));
    CHECK(throws<std::invalid_argument>([] { (void)ddsg_b200::ddsg_from_json(ddsg_b200::JsonDocument{"[1, 2"}); }));
    fs::remove_all(dir);
  }

  // 6. the decomposition itself (hdmr.hpp:364-483) through the shim: same
  //    target, anchor and options under both namespaces; accepted / rejected
  //    sets, b, every cut grid (stored order, keys, surplus bits), cut
  //    quadratures and the eta / rho diagnostics must be identical.
  for (int variant = 0; variant < 3; ++variant) {
    ddsg::DdsgOptions ro = opt;
    ddsg_b200::DdsgOptions bo;
    if (variant == 1) {  // order 3, everything kept, rho stops nothing
      ro.k_max = 3;
      ro.max_level = 3;
      ro.eps_eta = 0.0;
      ro.eps_gamma = 0.0;
    } else if (variant == 2) {  // zero-boundary cuts, rho stops after order 1
      ro.mode = ddsg::BoundaryMode::zero_boundary;
      ro.max_level = 4;
      ro.eps_rho = 10.0;
    }
    bo.k_max = ro.k_max;
    bo.eps_rho = ro.eps_rho;
    bo.eps_eta = ro.eps_eta;
    bo.max_level = ro.max_level;
    bo.eps_gamma = ro.eps_gamma;
    bo.mode = ro.mode == ddsg::BoundaryMode::modified_linear ? ddsg_b200::BoundaryMode::modified_linear
                                                             : ddsg_b200::BoundaryMode::zero_boundary;
    bo.workers = 3;
    ddsg::ExpansionDiagnostics dr;
    ddsg_b200::ExpansionDiagnostics db;
    const auto ref_anchor = ddsg::select_anchor(target, d, m, 64, 11);
    const auto b200_anchor = ddsg_b200::select_anchor(target, d, m, 64, 11);
    CHECK(same_bits(ref_anchor.coords, b200_anchor.coords) && same_bits(ref_anchor.f_anchor, b200_anchor.f_anchor));
    ddsg::AnchorPoint ar = variant == 0 ? anchor : ref_anchor;
    ddsg_b200::AnchorPoint ab{ar.coords, ar.f_anchor};
    const ddsg::DdsgFunction fr = ddsg::decompose(target, d, m, ar, ro, &dr);
    const ddsg_b200::DdsgFunction fb = ddsg_b200::decompose(target, d, m, ab, bo, &db);
    bool same = fr.accepted().size() == fb.accepted().size() && fr.rejected().size() == fb.rejected().size() &&
                fr.order_reached() == fb.order_reached() && fr.total_grid_points() == fb.total_grid_points() &&
                same_bits(fr.anchor().f_anchor, fb.anchor().f_anchor);
    for (const auto& z : fr.rejected()) same = same && fb.rejected().count(ddsg_b200::ComponentIndex{z.dims}) == 1;
    for (const auto& [u, b] : fr.coeff_b()) {
      const auto it = fb.coeff_b().find(ddsg_b200::ComponentIndex{u.dims});
      same = same && it != fb.coeff_b().end() && it->second == b;
      same = same && same_bits(fr.cut_quadrature(u), fb.cut_quadrature(ddsg_b200::ComponentIndex{u.dims}));
    }
    std::size_t nodes = 0;
    for (const auto& [u, g] : fr.accepted()) {
      const auto it = fb.accepted().find(ddsg_b200::ComponentIndex{u.dims});
      if (it == fb.accepted().end() || it->second.size() != g.size()) {
        same = false;
        continue;
      }
      const auto& nb = it->second.nodes();
      for (std::size_t i = 0; i < g.size(); ++i)
        same = same && nb[i].key == g.nodes()[i].key && same_bits(nb[i].surplus, g.nodes()[i].surplus);
      nodes += g.size();
    }
    CHECK(same);
    bool diag_same = dr.rho_by_order.size() == db.rho_by_order.size() && dr.eta_by_order.size() == db.eta_by_order.size();
    for (std::size_t k = 0; diag_same && k < dr.rho_by_order.size(); ++k)
      diag_same = std::memcmp(&dr.rho_by_order[k], &db.rho_by_order[k], sizeof(double)) == 0;
    for (std::size_t k = 0; diag_same && k < dr.eta_by_order.size(); ++k) {
      diag_same = dr.eta_by_order[k].size() == db.eta_by_order[k].size();
      for (std::size_t i = 0; diag_same && i < dr.eta_by_order[k].size(); ++i)
        diag_same = dr.eta_by_order[k][i].index.dims == db.eta_by_order[k][i].index.dims &&
                    dr.eta_by_order[k][i].accepted == db.eta_by_order[k][i].accepted &&
                    std::memcmp(&dr.eta_by_order[k][i].eta, &db.eta_by_order[k][i].eta, sizeof(double)) == 0;
    }
    CHECK(diag_same);
    // the native decomposition evaluates like the reference's (vectorized and naive)
    auto vb = ddsg_b200::VectorizedDdsg::compile(std::make_shared<const ddsg_b200::DdsgFunction>(fb));
    auto vr = ddsg::VectorizedDdsg::compile(std::make_shared<const ddsg::DdsgFunction>(fr));
    std::vector<double> a(m), b(m);
    int diff = 0, diff_naive = 0;
    for (std::size_t i = 0; i < 200; ++i) {
      vr.evaluate(pts[i], a);
      vb.evaluate(pts[i], b);
      diff += !same_bits(a, b);
      if (i < 20) {
        std::uint64_t cr = 0, cb = 0;
        fr.evaluate_naive(pts[i], a, &cr);
        fb.evaluate_naive(pts[i], b, &cb);
        diff_naive += !same_bits(a, b) || cr != cb;
      }
    }
    CHECK(diff == 0);
    CHECK(diff_naive == 0);
    std::printf("decompose variant %d through the shim: %zu accepted, %zu rejected, order %zu, %zu nodes: %s\n", variant,
                fb.accepted().size(), fb.rejected().size(), fb.order_reached(), nodes, same && diag_same ? "identical" : "DIFFERENT");
  }
  {  // argument checks and the failing-component report (hdmr.hpp:366-373, 425-429)
    ddsg_b200::DdsgOptions bo;
    bo.k_max = 1;
    bo.max_level = 2;
    ddsg_b200::AnchorPoint ab{std::vector<double>(d, 0.5), {}};
    CHECK(throws<std::invalid_argument>([&] { (void)ddsg_b200::decompose(target, 0, m, ab, bo); }));
    ddsg_b200::DdsgOptions bad = bo;
    bad.k_max = d + 1;
    CHECK(throws<std::invalid_argument>([&] { (void)ddsg_b200::decompose(target, d, m, ab, bad); }));
    bad = bo;
    bad.eps_eta = -1.0;
    CHECK(throws<std::invalid_argument>([&] { (void)ddsg_b200::decompose(target, d, m, ab, bad); }));
    ddsg_b200::AnchorPoint short_anchor{std::vector<double>(d - 1, 0.5), {}};
    CHECK(throws<std::invalid_argument>([&] { (void)ddsg_b200::decompose(target, d, m, short_anchor, bo); }));
    auto nan_target = [](std::span<const double> x, std::span<double> out) {
      target(x, out);
      if (x[2] != 0.5) out[1] = std::nan("");
    };
    bool reported = false;
    try {
      (void)ddsg_b200::decompose(nan_target, d, m, ab, bo);
    } catch (const std::runtime_error& e) {
      reported = std::string(e.what()).rfind("decompose: component {2} failed: ", 0) == 0;
    }
    CHECK(reported);
    CHECK(throws<std::invalid_argument>([&] { (void)ddsg_b200::select_anchor(target, d, m, 0, 1); }));
    CHECK(throws<std::invalid_argument>([&] { (void)ddsg_b200::cut_evaluator(target, ab, ddsg_b200::ComponentIndex{}); }));
  }

  // 6b. the time iteration's policy-change measure (time_iteration.hpp:213-223)
  {
    ddsg::DdsgOptions o2 = opt;
    o2.max_level = 4;
    o2.eps_eta = 0.0;
    auto d2 = std::make_shared<const ddsg::DdsgFunction>(ddsg::decompose(target, d, m, anchor, o2));
    auto prev_ref = std::make_shared<const ddsg::VectorizedDdsg>(ddsg::VectorizedDdsg::compile(d2));
    const ddsg_b200::VectorizedDdsg prev_gpu = to_b200(*d2);
    double change = 0.0;  // the reference's loop, verbatim shape
    {
      auto p_new = ref_side::compiled_evaluator(vec_ref);
      auto p_prev = ref_side::compiled_evaluator(prev_ref);
      std::vector<double> a(static_cast<std::size_t>(m)), b(static_cast<std::size_t>(m));
      for (const auto& x : pts) {
        p_new(x, a);
        p_prev(x, b);
        for (int c = 0; c < m; ++c)
          change = std::max(change, std::abs(a[static_cast<std::size_t>(c)] - b[static_cast<std::size_t>(c)]));
      }
    }
    const double change_gpu = ddsg_b200::policy_change(*vec_gpu, prev_gpu, pts);
    CHECK(change > 0.0 && std::memcmp(&change, &change_gpu, sizeof(double)) == 0);
    std::printf("policy change over %zu points: %.17g (reference) %.17g (batched)\n", pts.size(), change, change_gpu);
  }

  // 7. the host inline functions of rows a1 / a2 (grid_index.hpp, basis.hpp)
  //    and the node-count formulas against the reference's, bit for bit
  {
    std::mt19937_64 r2(77);
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    int bad = 0;
    for (int l = 1; l <= 14; ++l)
      for (std::uint32_t i = 1; i < (1u << l); i += (l > 8 ? 37u * 2u : 2u)) {
        const auto hk = ddsg::heap_key(l, i);
        bad += hk != ddsg_b200::heap_key(l, i) || ddsg::level_of(hk) != ddsg_b200::level_of(hk) ||
               ddsg::index_of(hk) != ddsg_b200::index_of(hk) || ddsg::parent_key(hk) != ddsg_b200::parent_key(hk);
        const double cr = ddsg::coordinate_of(hk), cb = ddsg_b200::coordinate_of(hk);
        bad += std::memcmp(&cr, &cb, sizeof(double)) != 0;
        for (int rep = 0; rep < 6; ++rep) {
          const double xs[6] = {u01(r2), cr, 0.0, 1.0, cr - std::ldexp(1.0, -l), cr + std::ldexp(1.0, -l) * u01(r2)};
          const double x = std::min(1.0, std::max(0.0, xs[rep]));
          for (int md = 0; md < 2; ++md) {
            const double vr = ddsg::basis_1d(l, i, x, md ? ddsg::BoundaryMode::modified_linear : ddsg::BoundaryMode::zero_boundary);
            const double vb = ddsg_b200::basis_1d(l, i, x, md ? ddsg_b200::BoundaryMode::modified_linear
                                                              : ddsg_b200::BoundaryMode::zero_boundary);
            bad += std::memcmp(&vr, &vb, sizeof(double)) != 0;
            bad += static_cast<int>(ddsg::basis_kind(l, i, md ? ddsg::BoundaryMode::modified_linear : ddsg::BoundaryMode::zero_boundary)) !=
                   static_cast<int>(ddsg_b200::basis_kind(l, i, md ? ddsg_b200::BoundaryMode::modified_linear
                                                                    : ddsg_b200::BoundaryMode::zero_boundary));
          }
        }
      }
    CHECK(bad == 0);
    bad = 0;
    for (int rep = 0; rep < 2000; ++rep) {
      ddsg::NodeKey key(4);
      std::vector<double> x(4);
      for (int j = 0; j < 4; ++j) {
        const int l = 1 + static_cast<int>(r2() % 6);
        key[j] = ddsg::heap_key(l, 2u * static_cast<std::uint32_t>(r2() % (1u << (l - 1))) + 1u);
        x[j] = u01(r2);
      }
      const double vr = ddsg::basis_nd(key, x, ddsg::BoundaryMode::modified_linear);
      const double vb = ddsg_b200::basis_nd(key, x, ddsg_b200::BoundaryMode::modified_linear);
      bad += std::memcmp(&vr, &vb, sizeof(double)) != 0 || ddsg::level_sum(key) != ddsg_b200::level_sum(key);
    }
    CHECK(bad == 0);
    bad = 0;
    for (int dd2 = 1; dd2 <= 40; ++dd2)
      for (int L = 1; L <= 12; ++L) {
        bad += ddsg::sg_node_count(dd2, L) != ddsg_b200::sg_node_count(dd2, L);
        for (int k = 0; k <= std::min(dd2, 3); ++k) bad += ddsg::ddsg_grid_count(dd2, k, L) != ddsg_b200::ddsg_grid_count(dd2, k, L);
      }
    CHECK(bad == 0);
    CHECK(throws<std::overflow_error>([] { (void)ddsg_b200::sg_node_count(300, 70); }));
    CHECK(throws<std::overflow_error>([] { (void)ddsg::sg_node_count(300, 70); }));
  }

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
