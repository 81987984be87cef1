// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI driver around the UNMODIFIED reference implementation
// (/root/reference/proj/include/ddsg/*.hpp, #included in place, nothing
// copied).  Built by oracle/Makefile into oracle/_ref/libddsg_ref.so, it is
// (1) the pin for the C restatement in oracle/ddsg_oracle.c, (2) the source of
// the golden fixtures under tests/golden/, and (3) the CPU baseline timed by
// bench.py (cpu_baseline.kind = "reference").
//
// Entry points wrap: SparseGridFunction::{from_nodes, build, interpolate,
// quadrature} (sparse_grid.hpp:84-179), DdsgFunction::{from_parts,
// evaluate_naive} (hdmr.hpp:257-325), decompose (hdmr.hpp:364-483),
// VectorizedDdsg::{compile, evaluate, evaluate_batch, quadrature}
// (ddsg_eval.hpp:40-151), detail::for_each_index (runtime.hpp:104-137),
// basis_1d / basis_nd (basis.hpp:67-84) and oracle::uniform_points
// (proj/tests/oracles.hpp:45-53), and the IRBC policy callers: the
// reference's own foc_residuals (irbc.hpp:306-361), refresh_derived and
// steady_state_lambda, plus Eigen-free restatements of foc_jacobian
// (solver.hpp:129-165) and euler_errors (solver.hpp:377-436) on top of them
// (solver.hpp needs Eigen, which is absent here).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ddsg/basis.hpp"
#include "ddsg/ddsg_eval.hpp"
#include "ddsg/hdmr.hpp"
#include "ddsg/irbc.hpp"
#include "ddsg/runtime.hpp"
#include "ddsg/sparse_grid.hpp"
#include "oracles.hpp"
#ifdef DDSG_REF_WITH_JSON
#include "ddsg/serialize.hpp"  // needs nlohmann json.hpp
#endif

using namespace ddsg;

namespace {
thread_local std::string g_err;
thread_local int64_t g_task = -1;

// 0 ok, 1 invalid_argument, 2 domain_error, 6 build_error, 7 out_of_range, 9 other
template <typename F>
int guarded(F&& f) {
  g_task = -1;
  try {
    f();
    return 0;
  } catch (const task_error& te) {
    g_task = static_cast<int64_t>(te.task_id());
    g_err = te.what();
    try {
      te.rethrow_cause();
    } catch (const std::domain_error&) {
      return 2;
    } catch (const std::invalid_argument&) {
      return 1;
    } catch (...) {
      return 9;
    }
  } catch (const build_error& e) {
    g_err = e.what();
    return 6;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
  return 9;
}

BoundaryMode to_mode(int m) { return m == 1 ? BoundaryMode::modified_linear : BoundaryMode::zero_boundary; }

std::vector<GridNode> make_nodes(int dim, int m, int64_t n, const uint32_t* keys, const double* surplus) {
  std::vector<GridNode> nodes(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    nodes[i].key.assign(keys + i * dim, keys + (i + 1) * dim);
    nodes[i].surplus.assign(surplus + i * m, surplus + (i + 1) * m);
  }
  return nodes;
}

using batch_cb = int (*)(const double* xs, int64_t count, double* out, void* ctx);

}  // namespace

struct ref_grid {
  SparseGridFunction g;
};

struct ref_hdmr {
  std::shared_ptr<const DdsgFunction> src;
  VectorizedDdsg vec;
};

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int64_t ref_last_task() { return g_task; }

int ref_basis_1d(int level, uint32_t index, double x, int mode, double* out) {
  return guarded([&] { *out = basis_1d(level, index, x, to_mode(mode)); });
}

int ref_heap_key(int level, uint32_t index, uint32_t* out) {
  return guarded([&] { *out = heap_key(level, index); });
}

int ref_grid_from_nodes(int dim, int m, int mode, int max_level, double eps, int64_t n, const uint32_t* keys,
                        const double* surplus, ref_grid** out) {
  return guarded([&] {
    auto h = std::make_unique<ref_grid>();
    h->g = SparseGridFunction::from_nodes(dim, m, max_level, eps, to_mode(mode),
                                          make_nodes(dim, m, n, keys, surplus));
    *out = h.release();
  });
}

int ref_grid_build(int dim, int m, int mode, int max_level, double eps, int norm, unsigned workers, batch_cb f,
                   void* ctx, ref_grid** out) {
  return guarded([&] {
    SgBuildOptions opt;
    opt.max_level = max_level;
    opt.eps_gamma = eps;
    opt.mode = to_mode(mode);
    opt.norm = norm == 1 ? SurplusNorm::l2 : SurplusNorm::inf;
    opt.workers = workers;
    GridEvaluator ev = [f, ctx](std::span<const double> x, std::span<double> o) {
      if (f(x.data(), 1, o.data(), ctx) != 0) throw std::runtime_error("evaluator callback failed");
    };
    auto h = std::make_unique<ref_grid>();
    h->g = SparseGridFunction::build(ev, dim, m, opt);
    *out = h.release();
  });
}

void ref_grid_free(ref_grid* g) { delete g; }
int64_t ref_grid_size(const ref_grid* g) { return static_cast<int64_t>(g->g.size()); }

void ref_grid_nodes(const ref_grid* g, uint32_t* keys, double* surplus) {
  const int dim = g->g.dim(), m = g->g.out_dim();
  int64_t i = 0;
  for (const auto& node : g->g.nodes()) {
    if (keys) std::copy(node.key.begin(), node.key.end(), keys + i * dim);
    if (surplus) std::copy(node.surplus.begin(), node.surplus.end(), surplus + i * m);
    ++i;
  }
}

int ref_grid_quadrature(const ref_grid* g, double* out) {
  return guarded([&] {
    const auto q = g->g.quadrature();
    std::copy(q.begin(), q.end(), out);
  });
}

// detail::for_each_index over SparseGridFunction::interpolate (the plain-grid
// CPU baseline of SURVEY.md §8(d)).  x: [n][dim], y: [n][m].
int ref_grid_eval(const ref_grid* g, const double* x, int64_t n, double* y, unsigned workers) {
  return guarded([&] {
    const int dim = g->g.dim(), m = g->g.out_dim();
    detail::for_each_index(static_cast<size_t>(n), workers, [&](size_t i) {
      g->g.interpolate(std::span<const double>(x + i * dim, dim), std::span<double>(y + i * m, m));
    });
  });
}

// DdsgFunction::from_parts + VectorizedDdsg::compile.  Slots in coeff_b order
// (empty index first); grids[s] is null for the empty slot.
int ref_hdmr_from_parts(int d, int m, const double* f_anchor, int n_slots, const int32_t* slot_order,
                        const int32_t* slot_dims, const int32_t* b, ref_grid* const* grids, ref_hdmr** out) {
  return guarded([&] {
    AnchorPoint anchor;
    anchor.coords.assign(d, 0.5);
    anchor.f_anchor.assign(f_anchor, f_anchor + m);
    std::map<ComponentIndex, SparseGridFunction> accepted;
    std::map<ComponentIndex, int> coeff;
    std::map<ComponentIndex, std::vector<double>> quads;
    int64_t off = 0;
    for (int s = 0; s < n_slots; ++s) {
      ComponentIndex u;
      u.dims.assign(slot_dims + off, slot_dims + off + slot_order[s]);
      off += slot_order[s];
      coeff[u] = b[s];
      if (u.empty()) {
        quads[u] = anchor.f_anchor;
      } else {
        accepted[u] = grids[s]->g;
        quads[u] = grids[s]->g.quadrature();
      }
    }
    DdsgOptions opt;
    auto src = std::make_shared<const DdsgFunction>(DdsgFunction::from_parts(
        d, m, opt, anchor, std::move(accepted), {}, std::move(coeff), std::move(quads)));
    auto h = std::make_unique<ref_hdmr>();
    h->vec = VectorizedDdsg::compile(src);
    h->src = std::move(src);
    *out = h.release();
  });
}

void ref_hdmr_free(ref_hdmr* h) { delete h; }

// VectorizedDdsg::evaluate_batch (ddsg_eval.hpp:130-139).
int ref_hdmr_eval(const ref_hdmr* h, const double* x, int64_t n, double* y, unsigned workers) {
  return guarded([&] {
    const int d = h->vec.dim(), m = h->vec.out_dim();
    std::vector<std::vector<double>> xs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) xs[i].assign(x + i * d, x + (i + 1) * d);
    const auto ys = h->vec.evaluate_batch(xs, workers);
    for (int64_t i = 0; i < n; ++i) std::copy(ys[i].begin(), ys[i].end(), y + i * m);
  });
}

// Same, but without the vector-of-vectors marshalling (for timing the kernel
// the reference runs, with its thread_local workspace).
int ref_hdmr_eval_flat(const ref_hdmr* h, const double* x, int64_t n, double* y, unsigned workers) {
  return guarded([&] {
    const int d = h->vec.dim(), m = h->vec.out_dim();
    detail::for_each_index(static_cast<size_t>(n), workers, [&](size_t i) {
      thread_local EvalWorkspace ws;
      h->vec.evaluate(std::span<const double>(x + i * d, d), std::span<double>(y + i * m, m), ws);
    });
  });
}

// VectorizedDdsg::evaluate with the interpolation-call counter.
int ref_hdmr_eval_one(const ref_hdmr* h, const double* x, double* y, uint64_t* calls) {
  return guarded([&] {
    const int d = h->vec.dim(), m = h->vec.out_dim();
    *calls = 0;
    h->vec.evaluate(std::span<const double>(x, d), std::span<double>(y, m), calls);
  });
}

// DdsgFunction::evaluate_naive (hdmr.hpp:257-270).
int ref_hdmr_eval_naive(const ref_hdmr* h, const double* x, int64_t n, double* y) {
  return guarded([&] {
    const int d = h->vec.dim(), m = h->vec.out_dim();
    for (int64_t i = 0; i < n; ++i)
      h->src->evaluate_naive(std::span<const double>(x + i * d, d), std::span<double>(y + i * m, m));
  });
}

int ref_hdmr_quadrature(const ref_hdmr* h, double* out) {
  return guarded([&] {
    const auto q = h->vec.quadrature();
    std::copy(q.begin(), q.end(), out);
  });
}

// decompose (hdmr.hpp:364-483) with a center anchor; the result is exported
// as parts (slots in coeff_b order + one ref_grid per accepted slot).
struct ref_decomp {
  std::shared_ptr<const DdsgFunction> src;
  std::vector<ComponentIndex> slots;
  std::vector<int> b;
};

int ref_decompose(int d, int m, int k_max, double eps_rho, double eps_eta, int max_level, double eps_gamma,
                  int mode, unsigned workers, batch_cb f, void* ctx, ref_decomp** out) {
  return guarded([&] {
    Evaluator ev = [f, ctx](std::span<const double> x, std::span<double> o) {
      if (f(x.data(), 1, o.data(), ctx) != 0) throw std::runtime_error("evaluator callback failed");
    };
    AnchorPoint a;
    a.coords.assign(d, 0.5);
    a.f_anchor.resize(m);
    ev(a.coords, a.f_anchor);
    DdsgOptions opt;
    opt.k_max = k_max;
    opt.eps_rho = eps_rho;
    opt.eps_eta = eps_eta;
    opt.max_level = max_level;
    opt.eps_gamma = eps_gamma;
    opt.mode = to_mode(mode);
    opt.workers = workers;
    auto h = std::make_unique<ref_decomp>();
    h->src = std::make_shared<const DdsgFunction>(decompose(ev, d, m, a, opt));
    for (const auto& [u, b] : h->src->coeff_b()) {
      h->slots.push_back(u);
      h->b.push_back(b);
    }
    *out = h.release();
  });
}

void ref_decomp_free(ref_decomp* h) { delete h; }
int ref_decomp_n_slots(const ref_decomp* h) { return static_cast<int>(h->slots.size()); }

// slot s: order, dims (<= capacity), b; returns a new ref_grid handle for
// non-empty slots (caller frees) or null.
ref_grid* ref_decomp_slot(const ref_decomp* h, int s, int32_t* order, int32_t* dims, int32_t* b) {
  const auto& u = h->slots[s];
  *order = static_cast<int32_t>(u.order());
  for (size_t j = 0; j < u.order(); ++j) dims[j] = u.dims[j];
  *b = h->b[s];
  if (u.empty()) return nullptr;
  auto g = std::make_unique<ref_grid>();
  g->g = h->src->accepted().at(u);
  return g.release();
}

void ref_decomp_anchor(const ref_decomp* h, double* f_anchor) {
  const auto& fa = h->src->anchor().f_anchor;
  std::copy(fa.begin(), fa.end(), f_anchor);
}

#ifdef DDSG_REF_WITH_JSON
// serialize.hpp:31-145: to_json / sparse_grid_from_json / ddsg_from_json.
// Returned strings are owned by the driver until the next call on this thread.
thread_local std::string g_json;
const char* ref_grid_to_json(const ref_grid* g) {
  g_json = to_json(g->g).dump();
  return g_json.c_str();
}
int ref_grid_from_json(const char* text, ref_grid** out) {
  return guarded([&] {
    auto h = std::make_unique<ref_grid>();
    h->g = sparse_grid_from_json(nlohmann::json::parse(text));
    *out = h.release();
  });
}
const char* ref_decomp_to_json(const ref_decomp* h) {
  g_json = to_json(*h->src).dump();
  return g_json.c_str();
}
// ddsg_from_json + compile; evaluation through ref_hdmr_eval.
int ref_hdmr_from_json(const char* text, ref_hdmr** out) {
  return guarded([&] {
    auto h = std::make_unique<ref_hdmr>();
    h->src = std::make_shared<const DdsgFunction>(ddsg_from_json(nlohmann::json::parse(text)));
    h->vec = VectorizedDdsg::compile(h->src);
    *out = h.release();
  });
}
int ref_json_enabled() { return 1; }
#else
int ref_json_enabled() { return 0; }
#endif

// oracle::uniform_points (proj/tests/oracles.hpp:45-53), point-major.
void ref_uniform_points(int dim, int64_t count, uint64_t seed, double* out) {
  const auto pts = oracle::uniform_points(dim, static_cast<size_t>(count), seed);
  for (int64_t i = 0; i < count; ++i) std::copy(pts[i].begin(), pts[i].end(), out + i * dim);
}

// oracle::sg_node_count_bruteforce (oracles.hpp:21-43) and sg_node_count (hdmr.hpp:134-151).
uint64_t ref_sg_node_count_bruteforce(int n, int L) { return oracle::sg_node_count_bruteforce(n, L); }

unsigned ref_default_workers() { return default_worker_count(); }

// oracle::b_coefficients_bruteforce (oracles.hpp:72-81): the telescopic
// coefficient of every family member (family incl. the empty index, each
// member given as order[s] dims concatenated in dims).
int ref_b_coefficients(int n_family, const int32_t* order, const int32_t* dims, int32_t* b_out) {
  return guarded([&] {
    std::vector<ComponentIndex> fam;
    int64_t off = 0;
    for (int s = 0; s < n_family; ++s) {
      ComponentIndex u;
      u.dims.assign(dims + off, dims + off + order[s]);
      off += order[s];
      fam.push_back(std::move(u));
    }
    const auto b = oracle::b_coefficients_bruteforce(fam);
    for (int s = 0; s < n_family; ++s) {
      auto it = b.find(fam[s]);
      b_out[s] = it == b.end() ? 0 : it->second;
    }
  });
}

}  // extern "C"

// ------------------------------------------------------------- IRBC callers

namespace {

irbc::IrbcParameters irbc_from_flat(int countries, int variant, const double* scal, const double* gamma) {
  // scal = {beta, alpha, delta, sigma, rho_a, phi_adj, gamma_base, lna_half_width, k_lo, k_hi}
  irbc::IrbcParameters p;
  p.countries = countries;
  p.variant = variant ? irbc::Variant::nonsmooth : irbc::Variant::smooth;
  p.beta = scal[0];
  p.alpha = scal[1];
  p.delta = scal[2];
  p.sigma = scal[3];
  p.rho_a = scal[4];
  p.phi_adj = scal[5];
  p.gamma_base = scal[6];
  p.lna_half_width = scal[7];
  p.k_lo = scal[8];
  p.k_hi = scal[9];
  if (gamma) p.gamma.assign(gamma, gamma + countries);
  irbc::refresh_derived(p);
  return p;
}

// compiled_evaluator (time_iteration.hpp:86-91) over a ref_hdmr, or the
// plain grid's interpolate.
irbc::PolicyEvaluator ref_policy(const ref_hdmr* h, const ref_grid* g) {
  if (h)
    return [h](std::span<const double> x, std::span<double> out) {
      thread_local EvalWorkspace ws;
      h->vec.evaluate(x, out, ws);
    };
  return [g](std::span<const double> x, std::span<double> out) { g->g.interpolate(x, out); };
}

irbc::EconomicState state_of(int N, const double* a, const double* k) {
  irbc::EconomicState st;
  st.a.assign(a, a + N);
  st.k.assign(k, k + N);
  return st;
}

}  // namespace

extern "C" {

// refresh_derived (irbc.hpp:59-92): writes gamma[N], tau[N] and A.
int ref_irbc_refresh(int countries, int variant, const double* scal, const double* gamma_in, double* gamma_out,
                     double* tau_out, double* A_out) {
  return guarded([&] {
    const auto p = irbc_from_flat(countries, variant, scal, gamma_in);
    std::copy(p.gamma.begin(), p.gamma.end(), gamma_out);
    std::copy(p.tau.begin(), p.tau.end(), tau_out);
    *A_out = p.A;
  });
}

int ref_irbc_steady_lambda(int countries, int variant, const double* scal, const double* gamma, double* out) {
  return guarded([&] { *out = irbc::steady_state_lambda(irbc_from_flat(countries, variant, scal, gamma)); });
}

// foc_residuals (irbc.hpp:306-361) per state; clamped[i] = its return value.
// States are spread over `workers` threads with detail::for_each_index, as
// the time iteration's per-point solves are (time_iteration.hpp).
int ref_irbc_foc_residuals(const ref_hdmr* h, const ref_grid* g, int countries, int variant, const double* scal,
                           const double* gamma, int64_t n, const double* a, const double* k, const double* cand,
                           unsigned workers, double* res, int32_t* clamped) {
  return guarded([&] {
    const auto p = irbc_from_flat(countries, variant, scal, gamma);
    const auto quad = irbc::make_shock_quadrature(countries);
    const auto pol = ref_policy(h, g);
    const int pd = p.policy_dim();
    detail::for_each_index(static_cast<size_t>(n), workers, [&](size_t i) {
      thread_local irbc::FocWorkspace ws;
      const auto st = state_of(countries, a + i * countries, k + i * countries);
      const auto cv = irbc::PolicyValue::from_flat(std::span<const double>(cand + i * pd, pd), p);
      const int c = irbc::foc_residuals(st, cv, pol, p, quad, std::span<double>(res + i * pd, pd), ws);
      if (clamped) clamped[i] = c;
    });
  });
}

// foc_jacobian (solver.hpp:129-165) restated without Eigen: jac[i][r][c].
int ref_irbc_foc_jacobian(const ref_hdmr* h, const ref_grid* g, int countries, int variant, const double* scal,
                          const double* gamma, int64_t n, const double* a, const double* k, const double* z,
                          const double* r0, double fd_epsilon, double* jac) {
  return guarded([&] {
    const auto p = irbc_from_flat(countries, variant, scal, gamma);
    const auto quad = irbc::make_shock_quadrature(countries);
    const auto pol = ref_policy(h, g);
    const int nn = p.policy_dim(), N = countries;
    irbc::FocWorkspace ws;
    std::vector<double> zp(nn), res(nn);
    for (int64_t i = 0; i < n; ++i) {
      const auto st = state_of(N, a + i * N, k + i * N);
      const double* zi = z + i * nn;
      const double* ri = r0 + i * nn;
      double* J = jac + i * nn * nn;
      zp.assign(zi, zi + nn);
      for (int c = 0; c < nn; ++c) {
        const double hh = fd_epsilon * std::max(std::abs(zi[c]), 1e-2);
        zp[c] = zi[c] + hh;
        const auto cand = irbc::PolicyValue::from_flat(std::span<const double>(zp.data(), zp.size()), p);
        irbc::foc_residuals(st, cand, pol, p, quad, res, ws);
        for (int rr = 0; rr < nn; ++rr) J[rr * nn + c] = (res[rr] - ri[rr]) / hh;
        zp[c] = zi[c];
      }
      if (p.variant == irbc::Variant::nonsmooth) {
        for (int j = 0; j < N; ++j) {
          const int row = N + j;
          const double mu = zi[N + j];
          const double s = zi[j] - (1.0 - p.delta) * st.k[j];
          const double norm = std::sqrt(mu * mu + s * s);
          double dmu, ds;
          if (norm == 0.0) {
            dmu = 1.0 - 1.0 / std::sqrt(2.0);
            ds = 1.0 - 1.0 / std::sqrt(2.0);
          } else {
            dmu = 1.0 - mu / norm;
            ds = 1.0 - s / norm;
          }
          for (int c = 0; c < nn; ++c) J[row * nn + c] = 0.0;
          J[row * nn + N + j] = dmu;
          J[row * nn + j] = ds;
        }
      }
    }
  });
}

// euler_errors (solver.hpp:377-436) restated without Eigen, on the samples
// xs[n][2N] (the caller draws them as the reference does).  stats = {mean,
// worst}; workers as the reference's for_each_index over 64 blocks.
int ref_irbc_euler_errors(const ref_hdmr* h, const ref_grid* g, int countries, int variant, const double* scal,
                          const double* gamma, int64_t n, const double* xs, unsigned workers, double* errs,
                          double* stats, uint64_t* clamp_count) {
  return guarded([&] {
    const auto p = irbc_from_flat(countries, variant, scal, gamma);
    const auto quad = irbc::make_shock_quadrature(countries);
    const auto policy = ref_policy(h, g);
    const size_t N = static_cast<size_t>(countries), d = 2 * N, m = static_cast<size_t>(p.policy_dim());
    std::vector<uint64_t> clamps_per_block(64, 0);
    const size_t n_blocks = std::min<size_t>(64, static_cast<size_t>(n));
    detail::for_each_index(n_blocks, workers, [&](size_t b) {
      irbc::FocWorkspace ws;
      std::vector<double> pol(m), res(m);
      uint64_t local = 0;
      for (size_t i = b; i < static_cast<size_t>(n); i += n_blocks) {
        const std::span<const double> x(xs + i * d, d);
        const auto st = irbc::from_canonical(x, p);
        policy(x, pol);
        const auto pv = irbc::PolicyValue::from_flat(pol, p);
        local += static_cast<uint64_t>(irbc::foc_residuals(st, pv, policy, p, quad, res, ws));
        double worst = 0.0;
        for (size_t j = 0; j < N; ++j) {
          const double g1 = pv.k_next[j] / st.k[j] - 1.0;
          const double denom = pv.lambda * (1.0 + p.phi_adj * g1);
          const double numerator = denom - res[j];
          worst = std::max(worst, std::abs(numerator / denom - 1.0));
        }
        errs[i] = worst;
      }
      clamps_per_block[b] = local;
    });
    double mean = 0.0, worst = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      mean += errs[i];
      worst = std::max(worst, errs[i]);
    }
    stats[0] = mean / static_cast<double>(n);
    stats[1] = worst;
    if (clamp_count) {
      *clamp_count = 0;
      for (uint64_t c : clamps_per_block) *clamp_count += c;
    }
  });
}

}  // extern "C"
