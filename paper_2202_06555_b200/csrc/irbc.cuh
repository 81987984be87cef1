// Batched IRBC policy callers: FOC residuals,
// their forward-difference Jacobian and the Euler-error estimate for whole
// batches of states, with every successor state of the batch evaluated by
// one batched policy call on the device (see irbc.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <vector>

namespace ddsg_b200 {
namespace irbc {

// IrbcParameters (irbc.hpp:27-53) after refresh_derived.
struct Params {
  int countries = 0;
  int nonsmooth = 0;
  double beta = 0, alpha = 0, delta = 0, sigma = 0, rho_a = 0, phi_adj = 0;
  double lna_half_width = 0, k_lo = 0, k_hi = 0, A = 0;
  std::vector<double> gamma, tau;
  int pdim() const { return nonsmooth ? 2 * countries + 1 : countries + 1; }
  int state_dim() const { return 2 * countries; }
  int nodes() const { return 2 * (countries + 1); }  // make_shock_quadrature (irbc.hpp:151-166)
};

// Batched policy: y[n][pdim] = policy(x[n][2N]) on device buffers; returns
// the lowest point index outside the domain (NaN) or -1.
using PolicyFn = std::function<int64_t(const double* dx, int64_t n, double* dy, cudaStream_t st)>;

// Each returns the lowest failing state / sample index or -1.  Buffers may
// be host or device memory.
int64_t foc_residuals(const Params& p, const PolicyFn& policy, int64_t n, const double* a, const double* k,
                      const double* cand, double* res, int32_t* clamped, cudaStream_t st);
int64_t foc_jacobian(const Params& p, const PolicyFn& policy, int64_t n, const double* a, const double* k,
                     const double* z, const double* r0, double fd_epsilon, double* jac, cudaStream_t st);
int64_t euler_errors(const Params& p, const PolicyFn& policy, int64_t n, const double* xs, double* errs,
                     double* mean, double* worst, uint64_t* clamps, cudaStream_t st);

// Launches of the last call on this thread (kernels of this module plus the
// policy evaluations' own).
int64_t last_launches();

}  // namespace irbc
}  // namespace ddsg_b200
