// Batched IRBC policy callers.
//
// The reference calls the policy interpolant once per successor state inside
// per-point loops: foc_residuals (irbc.hpp:306-361) evaluates the 2(N+1)
// successor states of one state, foc_jacobian (solver.hpp:129-165) repeats
// that for each of the pdim forward-difference columns, and euler_errors
// (solver.hpp:377-436) does it for every sample.  Here one call handles a
// whole batch of states:
//
//   successor_kernel   every successor state of every (state, set) in the
//                      batch as a canonical point x[P][2N] (law_of_motion,
//                      irbc.hpp:132-137; to_canonical_clamped, :198-214),
//                      plus the clamp flags
//   policy             ONE batched evaluation of all those points (the eval
//                      kernels of this library)
//   assemble_kernel    one CTA per (state, case): expectation over the
//                      quadrature nodes in the reference's order, Euler /
//                      Fischer-Burmeister / resource rows, and either the
//                      residuals, one Jacobian column or the Euler error
//
// A forward-difference column that perturbs mu_j or lambda leaves every
// successor state unchanged (only k' enters them), so the Jacobian needs
// 1 + N successor sets per state instead of pdim + 1.
//
// Arithmetic follows the reference expression by expression (the library
// is compiled with --fmad=false, so nothing is contracted).  exp / log /
// pow are CUDA's (<= 2 ulp) rather than glibc's, so results agree with the
// reference to rounding, not bit for bit (tests/test_irbc.py tolerances).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "device.cuh"
#include "irbc.cuh"

namespace ddsg_b200 {
namespace irbc {

namespace {

struct Model {
  int N, pdim, Q, kink;
  double beta, alpha, delta, sigma, rho_a, phi_adj, lw, k_lo, k_hi, A;
  double r;  // sqrt(N + 1): node magnitude (irbc.hpp:155)
  double w;  // 1 / (2(N + 1)): node weight (irbc.hpp:158)
  const double* gamma;
  const double* tau;
};

thread_local int64_t g_launches = 0;
thread_local double g_eval_ms = 0.0;  // dominant eval-kernel time of the policy calls

// h = fd_epsilon * std::max(std::abs(z), 1e-2) (solver.hpp:137), NaN kept
__device__ __forceinline__ double fd_step(double eps, double z) {
  const double az = fabs(z);
  return eps * (az < 1e-2 ? 1e-2 : az);
}

// One thread per (successor point P, coordinate j); P = ((s * sets + v) * Q + q).
// Set 0 uses the candidate's k'; set v >= 1 perturbs k'_{v-1} by its step.
__global__ void successor_kernel(Model M, int64_t n, int sets, const double* __restrict__ a,
                                 const double* __restrict__ z, double fd_eps, double* __restrict__ x,
                                 int32_t* __restrict__ flag) {
  const int D = 2 * M.N;
  const int64_t total = n * sets * M.Q * D;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx % D);
    const int64_t P = idx / D;
    const int q = static_cast<int>(P % M.Q);
    const int64_t sv = P / M.Q;
    const int v = static_cast<int>(sv % sets);
    const int64_t s = sv / sets;
    double c;
    if (j < M.N) {
      // node q: axis q/2 (N = the global shock), sign + for even q
      const int axis = q >> 1;
      const double e = (q & 1) ? -M.r : M.r;
      const double ec = axis == j ? e : 0.0, eg = axis == M.N ? e : 0.0;
      const double an = exp(M.rho_a * log(a[s * M.N + j]) + M.sigma * (ec + eg));
      c = (log(an) + M.lw) / (2.0 * M.lw);
    } else {
      const int jj = j - M.N;
      double kp = z[s * M.pdim + jj];
      if (v >= 1 && v - 1 == jj) kp = kp + fd_step(fd_eps, kp);
      c = (kp - M.k_lo) / (M.k_hi - M.k_lo);
    }
    bool cl = false;
    if (c < 0.0) {
      c = 0.0;
      cl = true;
    } else if (c > 1.0) {
      c = 1.0;
      cl = true;
    }
    x[P * D + j] = c;
    if (cl) atomicOr(&flag[P], 1);
  }
}

// from_canonical (irbc.hpp:216-226) for the Euler samples.
__global__ void states_kernel(Model M, int64_t n, const double* __restrict__ xs, double* __restrict__ a,
                              double* __restrict__ k) {
  const int64_t total = n * M.N;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = idx / M.N;
    const int j = static_cast<int>(idx % M.N);
    const double* x = xs + s * 2 * M.N;
    a[idx] = exp(x[j] * 2.0 * M.lw - M.lw);
    k[idx] = M.k_lo + x[M.N + j] * (M.k_hi - M.k_lo);
  }
}

enum { kResiduals = 0, kJacobian = 1, kEuler = 2 };

// One CTA per case.  kResiduals / kEuler: case = state s (set 0, no
// perturbation).  kJacobian: case = (s, c), perturbation of column c, set
// c + 1 for a capital column and set 0 otherwise.
template <int kMode>
__global__ void assemble_kernel(Model M, int64_t n_cases, int sets, const double* __restrict__ a,
                                const double* __restrict__ kst, const double* __restrict__ z,
                                const double* __restrict__ y, const int32_t* __restrict__ flag,
                                const double* __restrict__ r0, double fd_eps, double* __restrict__ out,
                                int32_t* __restrict__ clamped) {
  extern __shared__ double sh[];  // [N] resource terms, then [N] Euler errors
  const int N = M.N, pdim = M.pdim, Q = M.Q;
  const double omd = 1.0 - M.delta;
  for (int64_t cs = blockIdx.x; cs < n_cases; cs += gridDim.x) {
    const int64_t s = kMode == kJacobian ? cs / pdim : cs;
    const int c = kMode == kJacobian ? static_cast<int>(cs % pdim) : -1;
    const int v = (c >= 0 && c < N) ? c + 1 : 0;
    const double* zs = z + s * pdim;
    const double h = c >= 0 ? fd_step(fd_eps, zs[c]) : 0.0;
    const double lam = (pdim - 1 == c) ? zs[pdim - 1] + h : zs[pdim - 1];
    const double* ys = y + (s * sets + v) * Q * static_cast<int64_t>(pdim);
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      const double kp = (j == c) ? zs[j] + h : zs[j];
      const double mu = M.kink ? ((N + j == c) ? zs[N + j] + h : zs[N + j]) : 0.0;
      const double aj = a[s * N + j], kj = kst[s * N + j];
      const double pw = pow(kp, M.alpha - 1.0);
      // the successor productivity of country j takes five values:
      // no own / global shock, own +-, global +-
      const double base = M.rho_a * log(aj);
      const double an0 = exp(base + M.sigma * (0.0 + 0.0));
      const double anp = exp(base + M.sigma * (M.r + 0.0)), anm = exp(base + M.sigma * (-M.r + 0.0));
      const double agp = exp(base + M.sigma * (0.0 + M.r)), agm = exp(base + M.sigma * (0.0 + -M.r));
      double E = 0.0;
      for (int q = 0; q < Q; ++q) {
        const int axis = q >> 1;
        const double an = axis == j ? ((q & 1) ? anm : anp) : (axis == N ? ((q & 1) ? agm : agp) : an0);
        const double* row = ys + static_cast<int64_t>(q) * pdim;
        const double g2 = row[j] / kp - 1.0;
        double term = row[pdim - 1] * (an * M.A * M.alpha * pw + omd + 0.5 * M.phi_adj * g2 * (g2 + 2.0));
        if (M.kink) term -= omd * row[N + j];
        E += M.w * term;
      }
      const double g1 = kp / kj - 1.0;
      double r = lam * (1.0 + M.phi_adj * g1) - M.beta * E;
      if (M.kink) r -= mu;
      sh[j] = aj * M.A * pow(kj, M.alpha) + kj * (omd - 0.5 * M.phi_adj * g1 * g1) - kp -
              pow(lam / M.tau[j], -M.gamma[j]);
      double fb = 0.0;
      if (M.kink) {
        const double slack = kp - omd * kj;
        fb = mu + slack - sqrt(mu * mu + slack * slack);  // fischer_burmeister (irbc.hpp:265-267)
      }
      if (kMode == kResiduals) {
        out[s * pdim + j] = r;
        if (M.kink) out[s * pdim + N + j] = fb;
      } else if (kMode == kJacobian) {
        double* js = out + s * static_cast<int64_t>(pdim) * pdim;
        js[static_cast<int64_t>(j) * pdim + c] = (r - r0[s * pdim + j]) / h;
        if (M.kink) js[static_cast<int64_t>(N + j) * pdim + c] = (fb - r0[s * pdim + N + j]) / h;
      } else {
        const double denom = lam * (1.0 + M.phi_adj * g1);
        const double numerator = denom - r;
        sh[N + j] = fabs(numerator / denom - 1.0);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double resource = 0.0;
      for (int j = 0; j < N; ++j) resource += sh[j];
      if (kMode == kResiduals) {
        out[s * pdim + pdim - 1] = resource;
      } else if (kMode == kJacobian) {
        out[s * static_cast<int64_t>(pdim) * pdim + static_cast<int64_t>(pdim - 1) * pdim + c] =
            (resource - r0[s * pdim + pdim - 1]) / h;
      } else {
        double worst = 0.0;
        for (int j = 0; j < N; ++j) worst = worst < sh[N + j] ? sh[N + j] : worst;  // std::max
        out[s] = worst;
      }
      if (kMode != kJacobian && clamped) {
        int cnt = 0;
        for (int q = 0; q < Q; ++q) cnt += flag[(s * sets + v) * Q + q] != 0;
        clamped[s] = cnt;
      }
    }
    __syncthreads();
  }
}

// Generalized derivative of the Fischer-Burmeister rows (solver.hpp:144-162).
__global__ void fb_rows_kernel(Model M, int64_t n, const double* __restrict__ z, const double* __restrict__ kst,
                               double* __restrict__ jac) {
  const int N = M.N, pdim = M.pdim;
  const int64_t total = n * N;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = idx / N;
    const int j = static_cast<int>(idx % N);
    const double mu = z[s * pdim + N + j];
    const double sl = z[s * pdim + j] - (1.0 - M.delta) * kst[s * N + j];
    const double norm = sqrt(mu * mu + sl * sl);
    double dmu, ds;
    if (norm == 0.0) {
      dmu = 1.0 - 1.0 / sqrt(2.0);
      ds = 1.0 - 1.0 / sqrt(2.0);
    } else {
      dmu = 1.0 - mu / norm;
      ds = 1.0 - sl / norm;
    }
    double* row = jac + s * static_cast<int64_t>(pdim) * pdim + static_cast<int64_t>(N + j) * pdim;
    for (int c = 0; c < pdim; ++c) row[c] = 0.0;
    row[N + j] = dmu;
    row[j] = ds;
  }
}

// Sequential mean / max / clamp total (solver.hpp:426-434), one thread.
__global__ void euler_reduce_kernel(int64_t n, const double* __restrict__ errs, const int32_t* __restrict__ clamped,
                                    double* __restrict__ stats, unsigned long long* __restrict__ clamps) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double mean = 0.0, worst = 0.0;
  unsigned long long cl = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double e = errs[i];
    mean += e;
    worst = worst < e ? e : worst;
    cl += static_cast<unsigned long long>(clamped[i]);
  }
  stats[0] = mean / static_cast<double>(n);
  stats[1] = worst;
  *clamps = cl;
}

// Stream-ordered device scratch.
struct DBuf {
  void* p = nullptr;
  cudaStream_t st;
  DBuf(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) DDSG_CUDA(cudaMallocAsync(&p, bytes, st));
  }
  ~DBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

void copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes) DDSG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
}

unsigned grid_for(int64_t threads, int block) {
  const int64_t g = (threads + block - 1) / block;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 64)));
}

Model make_model(const Params& p, const double* dgamma, const double* dtau) {
  Model M{};
  M.N = p.countries;
  M.pdim = p.pdim();
  M.Q = p.nodes();
  M.kink = p.nonsmooth;
  M.beta = p.beta;
  M.alpha = p.alpha;
  M.delta = p.delta;
  M.sigma = p.sigma;
  M.rho_a = p.rho_a;
  M.phi_adj = p.phi_adj;
  M.lw = p.lna_half_width;
  M.k_lo = p.k_lo;
  M.k_hi = p.k_hi;
  M.A = p.A;
  M.r = std::sqrt(static_cast<double>(p.countries + 1));
  M.w = 1.0 / static_cast<double>(2 * (p.countries + 1));
  M.gamma = dgamma;
  M.tau = dtau;
  return M;
}

// States per chunk so that the successor points of one chunk stay within
// ~1 GiB of x + y.
int64_t chunk_states(const Params& p, int sets) {
  const int64_t per_state = static_cast<int64_t>(sets) * p.nodes() * (p.state_dim() + p.pdim()) * 8;
  return std::max<int64_t>(1, (int64_t{1} << 30) / per_state);
}

enum class Job { residuals, jacobian, euler };

// Shared driver.  Inputs per state: a, k [N], z [pdim] (candidate), r0 (Jacobian).
int64_t run(Job job, const Params& p, const PolicyFn& policy, int64_t n, const double* a_in, const double* k_in,
            const double* z_in, const double* r0_in, double fd_eps, const double* xs_in, double* out,
            int32_t* clamped_out, double* stats_out, uint64_t* clamps_out, cudaStream_t st) {
  g_launches = 0;
  g_eval_ms = 0.0;
  if (n <= 0) return -1;
  const int N = p.countries, pdim = p.pdim(), Q = p.nodes(), D = p.state_dim();
  const int sets = job == Job::jacobian ? N + 1 : 1;
  DBuf dgamma(N * 8, st), dtau(N * 8, st);
  copy(dgamma.p, p.gamma.data(), N * 8, st);
  copy(dtau.p, p.tau.data(), N * 8, st);
  const Model M = make_model(p, dgamma.as<double>(), dtau.as<double>());
  const int64_t chunk = std::min(n, chunk_states(p, sets));
  const int64_t pts_max = chunk * sets * Q;
  DBuf da(chunk * N * 8, st), dk(chunk * N * 8, st), dz(chunk * pdim * 8, st);
  DBuf dx(pts_max * D * 8, st), dy(pts_max * pdim * 8, st), dflag(pts_max * 4, st);
  DBuf dr0(job == Job::jacobian ? chunk * pdim * 8 : 0, st);
  const int64_t out_per_state = job == Job::jacobian ? int64_t{pdim} * pdim : (job == Job::euler ? 1 : pdim);
  DBuf dout(chunk * out_per_state * 8, st), dcl(chunk * 4, st);
  // Euler: all errors and clamp counts stay on the device for the reduction
  DBuf derrs(job == Job::euler ? n * 8 : 0, st), dclall(job == Job::euler ? n * 4 : 0, st);
  DBuf dxs(job == Job::euler ? chunk * D * 8 : 0, st);
  const int block = 256;
  for (int64_t off = 0; off < n; off += chunk) {
    const int64_t cnt = std::min(chunk, n - off);
    const int64_t pts = cnt * sets * Q;
    if (job == Job::euler) {
      // states and candidate policy at the samples (solver.hpp:413-415)
      copy(dxs.p, xs_in + off * D, cnt * D * 8, st);
      states_kernel<<<grid_for(cnt * N, block), block, 0, st>>>(M, cnt, dxs.as<double>(), da.as<double>(),
                                                                dk.as<double>());
      DDSG_CUDA(cudaGetLastError());
      ++g_launches;
      const int64_t bad = policy(dxs.as<double>(), cnt, dz.as<double>(), st);
      g_launches += last_stats().launches;
      g_eval_ms += last_stats().main_ms;
      if (bad >= 0) return off + bad;
    } else {
      copy(da.p, a_in + off * N, cnt * N * 8, st);
      copy(dk.p, k_in + off * N, cnt * N * 8, st);
      copy(dz.p, z_in + off * pdim, cnt * pdim * 8, st);
      if (job == Job::jacobian) copy(dr0.p, r0_in + off * pdim, cnt * pdim * 8, st);
    }
    DDSG_CUDA(cudaMemsetAsync(dflag.p, 0, pts * 4, st));
    successor_kernel<<<grid_for(pts * D, block), block, 0, st>>>(M, cnt, sets, da.as<double>(), dz.as<double>(),
                                                                 fd_eps, dx.as<double>(), dflag.as<int32_t>());
    DDSG_CUDA(cudaGetLastError());
    ++g_launches;
    const int64_t bad = policy(dx.as<double>(), pts, dy.as<double>(), st);
    g_launches += last_stats().launches;
    g_eval_ms += last_stats().main_ms;
    if (bad >= 0) return off + bad / (static_cast<int64_t>(sets) * Q);
    const size_t smem = static_cast<size_t>(2 * N) * 8;
    const int ablock = std::min(256, ((N + 31) / 32) * 32);
    if (job == Job::residuals) {
      assemble_kernel<kResiduals><<<grid_for(cnt, 1), ablock, smem, st>>>(
          M, cnt, sets, da.as<double>(), dk.as<double>(), dz.as<double>(), dy.as<double>(),
          dflag.as<int32_t>(), nullptr, fd_eps, dout.as<double>(), dcl.as<int32_t>());
    } else if (job == Job::jacobian) {
      assemble_kernel<kJacobian><<<grid_for(cnt * pdim, 1), ablock, smem, st>>>(
          M, cnt * pdim, sets, da.as<double>(), dk.as<double>(), dz.as<double>(), dy.as<double>(),
          dflag.as<int32_t>(), dr0.as<double>(), fd_eps, dout.as<double>(), nullptr);
      if (p.nonsmooth) {
        DDSG_CUDA(cudaGetLastError());
        ++g_launches;
        fb_rows_kernel<<<grid_for(cnt * N, block), block, 0, st>>>(M, cnt, dz.as<double>(), dk.as<double>(),
                                                                   dout.as<double>());
      }
    } else {
      assemble_kernel<kEuler><<<grid_for(cnt, 1), ablock, smem, st>>>(
          M, cnt, sets, da.as<double>(), dk.as<double>(), dz.as<double>(), dy.as<double>(),
          dflag.as<int32_t>(), nullptr, fd_eps, derrs.as<double>() + off, dclall.as<int32_t>() + off);
    }
    DDSG_CUDA(cudaGetLastError());
    ++g_launches;
    if (job == Job::residuals) {
      copy(out + off * pdim, dout.p, cnt * pdim * 8, st);
      if (clamped_out) copy(clamped_out + off, dcl.p, cnt * 4, st);
    } else if (job == Job::jacobian) {
      copy(out + off * pdim * pdim, dout.p, cnt * pdim * pdim * 8, st);
    }
  }
  if (job == Job::euler) {
    DBuf dstats(2 * 8 + 8, st);
    euler_reduce_kernel<<<1, 1, 0, st>>>(n, derrs.as<double>(), dclall.as<int32_t>(), dstats.as<double>(),
                                         reinterpret_cast<unsigned long long*>(dstats.as<double>() + 2));
    DDSG_CUDA(cudaGetLastError());
    ++g_launches;
    copy(out, derrs.p, n * 8, st);
    double host_stats[3];
    DDSG_CUDA(cudaMemcpyAsync(host_stats, dstats.p, 24, cudaMemcpyDeviceToHost, st));
    DDSG_CUDA(cudaStreamSynchronize(st));
    stats_out[0] = host_stats[0];
    stats_out[1] = host_stats[1];
    if (clamps_out) {
      unsigned long long cl;
      std::memcpy(&cl, &host_stats[2], 8);
      *clamps_out = cl;
    }
  }
  DDSG_CUDA(cudaStreamSynchronize(st));
  EvalStats& es = last_stats();
  es.launches = g_launches;
  es.kernel_ms = 0.0;
  es.main_ms = g_eval_ms;
  return -1;
}

}  // namespace

int64_t foc_residuals(const Params& p, const PolicyFn& policy, int64_t n, const double* a, const double* k,
                      const double* cand, double* res, int32_t* clamped, cudaStream_t st) {
  return run(Job::residuals, p, policy, n, a, k, cand, nullptr, 0.0, nullptr, res, clamped, nullptr, nullptr, st);
}

int64_t foc_jacobian(const Params& p, const PolicyFn& policy, int64_t n, const double* a, const double* k,
                     const double* z, const double* r0, double fd_epsilon, double* jac, cudaStream_t st) {
  return run(Job::jacobian, p, policy, n, a, k, z, r0, fd_epsilon, nullptr, jac, nullptr, nullptr, nullptr, st);
}

int64_t euler_errors(const Params& p, const PolicyFn& policy, int64_t n, const double* xs, double* errs,
                     double* mean, double* worst, uint64_t* clamps, cudaStream_t st) {
  double stats[2] = {0.0, 0.0};
  const int64_t bad = run(Job::euler, p, policy, n, nullptr, nullptr, nullptr, nullptr, 0.0, xs, errs, nullptr,
                          stats, clamps, st);
  if (bad < 0) {
    *mean = stats[0];
    *worst = stats[1];
  }
  return bad;
}

int64_t last_launches() { return g_launches; }

}  // namespace irbc
}  // namespace ddsg_b200
