/*
 * Synthetic workloads: the target functions of BASELINE.json's five configs
 * and of the reference's test suite, as C batch evaluators
 * (ddsg_batch_evaluator: xs[count][dim] -> out[count][m]).
 *
 * Built into libddsg_workloads.so, separate from the product library.  Both
 * our grid builder and the reference's (through oracle/_ref) call the same
 * compiled function, so grid-construction parity compares identical f bits.
 *
 * Seeded coefficients come from std::mt19937_64-compatible draws (the same
 * generator the reference's tests use, proj/tests/oracles.hpp:45-53) so every
 * config is reproducible from its seed; DESIGN.md records the choices
 * BASELINE.json leaves open (coefficients, pairs, kink offsets).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}
static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (s->mt[i] & 0xFFFFFFFF80000000ull) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      s->mt[i] = s->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
    }
    s->idx = 0;
  }
  uint64_t z = s->mt[s->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}
static double unif(mt64* s, double a, double b) {
  double r = (double)mt64_next(s) / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return a + (b - a) * r;
}

/* ------------------------------------------------- reference test targets */

/* test_ddsg_eval.cpp:37-42 "coupled" */
int wl_coupled(const double* xs, int64_t count, double* out, void* ctx) {
  const int d = *(const int*)ctx;
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * d;
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += exp(-0.5 * x[j]) + 0.2 * x[j] * x[j];
    for (int j = 0; j + 1 < d; ++j) s += 0.3 * sin(x[j] * x[j + 1]);
    out[i] = s;
  }
  return 0;
}

/* test_sparse_grid.cpp:89-93 round-trip product target */
int wl_exp_product(const double* xs, int64_t count, double* out, void* ctx) {
  const int d = *(const int*)ctx;
  for (int64_t i = 0; i < count; ++i) {
    double s = 1.0;
    for (int j = 0; j < d; ++j) s *= exp(-2.0 * xs[i * d + j]) + 0.3 * xs[i * d + j];
    out[i] = s;
  }
  return 0;
}

/* test_sparse_grid.cpp:103-105 adaptive round-trip target (d = 2) */
int wl_bump(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * 2;
    out[i] = exp(-40.0 * (x[0] - 0.3) * (x[0] - 0.3)) + 0.1 * x[1];
  }
  return 0;
}

/* test_sparse_grid.cpp:228-230 x(1-x)y(1-y) */
int wl_parabola2(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * 2;
    out[i] = x[0] * (1.0 - x[0]) * x[1] * (1.0 - x[1]);
  }
  return 0;
}

/* test_ddsg_eval.cpp:226-230 vector-valued target (d = 2, m = 3) */
int wl_vector3(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * 2;
    out[i * 3 + 0] = x[0] + x[1];
    out[i * 3 + 1] = exp(x[0] * x[1]);
    out[i * 3 + 2] = 0.5;
  }
  return 0;
}

/* constant 4.25 (test_ddsg_eval.cpp:122-133) */
int wl_constant(const double* xs, int64_t count, double* out, void* ctx) {
  (void)xs;
  (void)ctx;
  for (int64_t i = 0; i < count; ++i) out[i] = 4.25;
  return 0;
}

/* test_hdmr.cpp:223-225 (d = 3) */
int wl_hdmr_full(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * 3;
    out[i] = exp(x[0]) * (1.0 + 0.5 * sin(3.0 * x[1])) + x[1] * x[2];
  }
  return 0;
}

/* pruned-family target (test_ddsg_eval.cpp:145-147, d = 3) */
int wl_pruned3(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * 3;
    out[i] = x[0] + exp(x[1] * x[2]) + 0.1 * x[2];
  }
  return 0;
}

/* ------------------------------------------------------- BASELINE configs */

/* config 1: exp(-sum_k (x_k - 1/2)^2), m = 1 */
int wl_config1(const double* xs, int64_t count, double* out, void* ctx) {
  const int d = ctx ? *(const int*)ctx : 4;
  for (int64_t i = 0; i < count; ++i) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = xs[i * d + k] - 0.5;
      s += t * t;
    }
    out[i] = exp(-s);
  }
  return 0;
}

/* config 2: f_j = prod_k (1 + 0.1 j x_k)^0.3, j = 0..10, d = 10 */
int wl_config2(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  for (int64_t i = 0; i < count; ++i) {
    for (int j = 0; j <= 10; ++j) {
      double p = 1.0;
      for (int k = 0; k < 10; ++k) p *= pow(1.0 + 0.1 * j * xs[i * 10 + k], 0.3);
      out[i * 11 + j] = p;
    }
  }
  return 0;
}

/* config 3: f_j = max(0, sum x - 10) + 0.1 sum x^2 + 0.01 j x_{j mod 20}, j = 0..20, d = 20 */
int wl_config3(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * 20;
    double s = 0.0, q = 0.0;
    for (int k = 0; k < 20; ++k) {
      s += x[k];
      q += x[k] * x[k];
    }
    const double base = (s - 10.0 > 0.0 ? s - 10.0 : 0.0) + 0.1 * q;
    for (int j = 0; j <= 20; ++j) out[i * 21 + j] = base + 0.01 * j * x[j % 20];
  }
  return 0;
}

/* IRBC-shaped HDMR targets (configs 4 and 5).  States X = 0.8 + 0.4 x in
 * [0.8, 1.2]^d.  Output j < m-1 is a policy
 *   g_j(X) = kappa_j + sum_k a_jk log X_k + sum_{r in R_j} c_jr X_p(r) X_q(r)
 * (config 5 adds the irreversibility kink max(0, g_j)); output m-1 is a
 * smooth multiplier-like aggregate.  Coefficients are drawn once from the
 * config seed. */
typedef struct {
  int d, m, n_pairs, kink;
  double* a;      /* [m][d] */
  double* kappa;  /* [m] */
  int* pp;        /* [n_pairs] */
  int* pq;        /* [n_pairs] */
  double* c;      /* [n_pairs] coefficient of pair r on output owner[r] */
  int* owner;     /* [n_pairs] output index */
} irbc_target;

static irbc_target* g_cfg[6];

static irbc_target* make_irbc(int config) {
  irbc_target* t = (irbc_target*)calloc(1, sizeof(irbc_target));
  mt64* rng = (mt64*)malloc(sizeof(mt64));
  if (config == 4) {
    t->d = 100;
    t->m = 51;
    t->n_pairs = 45;
    t->kink = 0;
    mt64_seed(rng, 20220213ull + 4);
  } else {
    t->d = 300;
    t->m = 151;
    t->n_pairs = 300;
    t->kink = 1;
    mt64_seed(rng, 20220213ull + 5);
  }
  const int d = t->d, m = t->m;
  t->a = (double*)malloc(sizeof(double) * (size_t)m * d);
  t->kappa = (double*)malloc(sizeof(double) * (size_t)m);
  t->pp = (int*)malloc(sizeof(int) * (size_t)t->n_pairs);
  t->pq = (int*)malloc(sizeof(int) * (size_t)t->n_pairs);
  t->c = (double*)malloc(sizeof(double) * (size_t)t->n_pairs);
  t->owner = (int*)malloc(sizeof(int) * (size_t)t->n_pairs);
  for (int j = 0; j < m; ++j)
    for (int k = 0; k < d; ++k) t->a[j * d + k] = unif(rng, -1.0, 1.0) / (config == 4 ? 10.0 : 30.0);
  if (config == 4) {
    /* all 45 pairs among the first 10 dims, lexicographic */
    int r = 0;
    for (int p = 0; p < 10; ++p)
      for (int q = p + 1; q < 10; ++q) {
        t->pp[r] = p;
        t->pq[r] = q;
        ++r;
      }
  } else {
    /* 300 distinct random pairs among 300 dims, sorted lexicographically */
    int r = 0;
    while (r < t->n_pairs) {
      int p = (int)(mt64_next(rng) % (uint64_t)d), q = (int)(mt64_next(rng) % (uint64_t)d);
      if (p == q) continue;
      if (p > q) {
        int tmp = p;
        p = q;
        q = tmp;
      }
      int dup = 0;
      for (int s = 0; s < r; ++s) dup |= (t->pp[s] == p && t->pq[s] == q);
      if (dup) continue;
      t->pp[r] = p;
      t->pq[r] = q;
      ++r;
    }
    for (int i = 1; i < r; ++i) /* insertion sort (p, q) */
      for (int k = i; k > 0 && (t->pp[k - 1] > t->pp[k] || (t->pp[k - 1] == t->pp[k] && t->pq[k - 1] > t->pq[k])); --k) {
        int a = t->pp[k], b = t->pq[k];
        t->pp[k] = t->pp[k - 1];
        t->pq[k] = t->pq[k - 1];
        t->pp[k - 1] = a;
        t->pq[k - 1] = b;
      }
  }
  for (int r = 0; r < t->n_pairs; ++r) {
    t->owner[r] = (int)(mt64_next(rng) % (uint64_t)(m - 1));
    t->c[r] = unif(rng, -0.5, 0.5);
  }
  for (int j = 0; j < m; ++j) {
    /* kappa: the policy argument at the anchor (X = 1) is a small positive
     * delta, so cuts through dims with large |a_jk| cross the kink */
    double pair_at_anchor = 0.0;
    for (int r = 0; r < t->n_pairs; ++r)
      if (t->owner[r] == j) pair_at_anchor += t->c[r];
    t->kappa[j] = unif(rng, 0.002, 0.02) - pair_at_anchor;
  }
  free(rng);
  return t;
}

static irbc_target* irbc(int config) {
  if (!g_cfg[config]) g_cfg[config] = make_irbc(config);
  return g_cfg[config];
}

static int irbc_eval(int config, const double* xs, int64_t count, double* out) {
  irbc_target* t = irbc(config);
  const int d = t->d, m = t->m;
  double* lx = (double*)malloc(sizeof(double) * (size_t)d);
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * d;
    double* o = out + i * m;
    for (int k = 0; k < d; ++k) lx[k] = log(0.8 + 0.4 * x[k]);
    for (int j = 0; j < m; ++j) {
      double s = t->kappa[j];
      const double* a = t->a + (size_t)j * d;
      for (int k = 0; k < d; ++k) s += a[k] * lx[k];
      o[j] = s;
    }
    for (int r = 0; r < t->n_pairs; ++r) {
      const double xp = 0.8 + 0.4 * x[t->pp[r]], xq = 0.8 + 0.4 * x[t->pq[r]];
      o[t->owner[r]] += t->c[r] * xp * xq;
    }
    if (t->kink)
      for (int j = 0; j < m - 1; ++j) o[j] = o[j] > 0.0 ? o[j] : 0.0;
    /* multiplier-like last output: smooth aggregate of the policies */
    double agg = 0.0;
    for (int j = 0; j < m - 1; ++j) agg += o[j];
    o[m - 1] = exp(0.1 * agg / (m - 1)) + 0.05 * lx[0];
  }
  free(lx);
  return 0;
}

int wl_config4(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  return irbc_eval(4, xs, count, out);
}
int wl_config5(const double* xs, int64_t count, double* out, void* ctx) {
  (void)ctx;
  return irbc_eval(5, xs, count, out);
}

/* Pair list of an HDMR config: writes n_pairs (p, q) into pairs[2*r]. */
int wl_config_pairs(int config, int32_t* pairs) {
  irbc_target* t = irbc(config);
  for (int r = 0; r < t->n_pairs; ++r) {
    pairs[2 * r] = t->pp[r];
    pairs[2 * r + 1] = t->pq[r];
  }
  return t->n_pairs;
}

/* ----------------------------------------------------------- cut wrapper */

/* Restriction of a d-dim target to the cut through the anchor along `dims`
 * (hdmr.hpp:248-259): g(y) = f(x) with x_dims = y, x_j = anchor_j elsewhere. */
typedef int (*wl_fn)(const double*, int64_t, double*, void*);
typedef struct {
  wl_fn f;
  void* fctx;
  int d, m, k;
  int32_t dims[16];
  double* anchor; /* [d] */
} wl_cut;

wl_cut* wl_cut_new(wl_fn f, void* fctx, int d, int m, int k, const int32_t* dims, const double* anchor) {
  if (k < 1 || k > 16) return NULL;
  wl_cut* c = (wl_cut*)calloc(1, sizeof(wl_cut));
  c->f = f;
  c->fctx = fctx;
  c->d = d;
  c->m = m;
  c->k = k;
  for (int j = 0; j < k; ++j) c->dims[j] = dims[j];
  c->anchor = (double*)malloc(sizeof(double) * (size_t)d);
  memcpy(c->anchor, anchor, sizeof(double) * (size_t)d);
  return c;
}

void wl_cut_free(wl_cut* c) {
  if (!c) return;
  free(c->anchor);
  free(c);
}

int wl_cut_eval(const double* ys, int64_t count, double* out, void* ctx) {
  wl_cut* c = (wl_cut*)ctx;
  const int64_t chunk = 256;
  double* xs = (double*)malloc(sizeof(double) * (size_t)chunk * c->d);
  int rc = 0;
  for (int64_t off = 0; off < count && rc == 0; off += chunk) {
    const int64_t n = count - off < chunk ? count - off : chunk;
    for (int64_t i = 0; i < n; ++i) {
      memcpy(xs + i * c->d, c->anchor, sizeof(double) * (size_t)c->d);
      for (int j = 0; j < c->k; ++j) xs[i * c->d + c->dims[j]] = ys[(off + i) * c->k + j];
    }
    rc = c->f(xs, n, out + off * c->m, c->fctx);
  }
  free(xs);
  return rc;
}

/* --------------------------------------------------- IRBC policy targets */

/* Policy-shaped targets for the batched IRBC callers (SURVEY.md §8(f) rows
 * 2-3).  Canonical state x in [0,1]^(2N): N log-productivities, then N
 * capitals (irbc.hpp:188-226); flat policy k'[N], (mu[N]), lambda
 * (irbc.hpp:230-246):
 *   lna_j = 2 w x_j - w,  k_j = k_lo + x_{N+j} (k_hi - k_lo)
 *   inv_j = delta k_j + ca_j lna_j + ck_j (1 - k_j)
 *           + sum_{pairs r owned by j} cc_r (x_p - 1/2)(x_q - 1/2)
 *   k'_j  = (1 - delta) k_j + max(0, inv_j)   (irreversible investment)
 *   mu_j  = 0.1 max(0, -inv_j)                (non-smooth variant)
 *   lambda = lam0 exp(-0.1 mean_j lna_j + 0.05 mean_j (k_j - 1))
 * steady = 1 gives the reference tests' steady policy instead
 * (test_irbc.cpp:14-24): k' = k, mu = 0, lambda = lam0. */
typedef struct {
  int N, nonsmooth, steady, n_pairs;
  double delta, k_lo, k_hi, lw, lam0;
  double *ca, *ck, *cc;
  int *pp, *pq, *owner;
} wl_irbc;

wl_irbc* wl_irbc_new(int N, int nonsmooth, int steady, int n_pairs, uint64_t seed, double delta, double k_lo,
                     double k_hi, double lw, double lam0) {
  if (N < 1 || n_pairs < 0 || (n_pairs > 0 && 2 * N < 2)) return NULL;
  wl_irbc* t = (wl_irbc*)calloc(1, sizeof(wl_irbc));
  t->N = N;
  t->nonsmooth = nonsmooth;
  t->steady = steady;
  t->delta = delta;
  t->k_lo = k_lo;
  t->k_hi = k_hi;
  t->lw = lw;
  t->lam0 = lam0;
  const int d = 2 * N;
  const long maxp = (long)d * (d - 1) / 2;
  if (n_pairs > maxp) n_pairs = (int)maxp;
  t->n_pairs = n_pairs;
  t->ca = (double*)malloc(sizeof(double) * (size_t)N);
  t->ck = (double*)malloc(sizeof(double) * (size_t)N);
  t->cc = (double*)malloc(sizeof(double) * (size_t)(n_pairs + 1));
  t->pp = (int*)malloc(sizeof(int) * (size_t)(n_pairs + 1));
  t->pq = (int*)malloc(sizeof(int) * (size_t)(n_pairs + 1));
  t->owner = (int*)malloc(sizeof(int) * (size_t)(n_pairs + 1));
  mt64 rng;
  mt64_seed(&rng, seed);
  for (int j = 0; j < N; ++j) {
    t->ca[j] = unif(&rng, 0.01, 0.05);
    t->ck[j] = unif(&rng, 0.01, 0.05);
  }
  int r = 0;
  while (r < n_pairs) {
    int p = (int)(mt64_next(&rng) % (uint64_t)d), q = (int)(mt64_next(&rng) % (uint64_t)d);
    if (p == q) continue;
    if (p > q) {
      int tmp = p;
      p = q;
      q = tmp;
    }
    int dup = 0;
    for (int s = 0; s < r; ++s) dup |= (t->pp[s] == p && t->pq[s] == q);
    if (dup) continue;
    t->pp[r] = p;
    t->pq[r] = q;
    ++r;
  }
  for (int i = 1; i < r; ++i) /* insertion sort (p, q) */
    for (int k = i; k > 0 && (t->pp[k - 1] > t->pp[k] || (t->pp[k - 1] == t->pp[k] && t->pq[k - 1] > t->pq[k])); --k) {
      int a = t->pp[k], b = t->pq[k];
      t->pp[k] = t->pp[k - 1];
      t->pq[k] = t->pq[k - 1];
      t->pp[k - 1] = a;
      t->pq[k - 1] = b;
    }
  for (int s = 0; s < r; ++s) {
    t->owner[s] = (int)(mt64_next(&rng) % (uint64_t)N);
    t->cc[s] = unif(&rng, -0.2, 0.2);
  }
  return t;
}

void wl_irbc_free(wl_irbc* t) {
  if (!t) return;
  free(t->ca);
  free(t->ck);
  free(t->cc);
  free(t->pp);
  free(t->pq);
  free(t->owner);
  free(t);
}

int wl_irbc_pairs(const wl_irbc* t, int32_t* pairs) {
  for (int r = 0; r < t->n_pairs; ++r) {
    pairs[2 * r] = t->pp[r];
    pairs[2 * r + 1] = t->pq[r];
  }
  return t->n_pairs;
}

int wl_irbc_policy(const double* xs, int64_t count, double* out, void* ctx) {
  const wl_irbc* t = (const wl_irbc*)ctx;
  const int N = t->N, d = 2 * N, m = t->nonsmooth ? 2 * N + 1 : N + 1;
  double* inv = (double*)malloc(sizeof(double) * (size_t)N);
  for (int64_t i = 0; i < count; ++i) {
    const double* x = xs + i * d;
    double* o = out + i * m;
    double mlna = 0.0, mk = 0.0;
    for (int j = 0; j < N; ++j) {
      const double lna = x[j] * 2.0 * t->lw - t->lw;
      const double k = t->k_lo + x[N + j] * (t->k_hi - t->k_lo);
      inv[j] = t->delta * k + t->ca[j] * lna + t->ck[j] * (1.0 - k);
      mlna += lna;
      mk += k - 1.0;
    }
    for (int r = 0; r < t->n_pairs; ++r) inv[t->owner[r]] += t->cc[r] * (x[t->pp[r]] - 0.5) * (x[t->pq[r]] - 0.5);
    for (int j = 0; j < N; ++j) {
      const double k = t->k_lo + x[N + j] * (t->k_hi - t->k_lo);
      o[j] = t->steady ? k : (1.0 - t->delta) * k + (inv[j] > 0.0 ? inv[j] : 0.0);
      if (t->nonsmooth) o[N + j] = t->steady ? 0.0 : 0.1 * (inv[j] < 0.0 ? -inv[j] : 0.0);
    }
    o[m - 1] = t->steady ? t->lam0 : t->lam0 * exp(-0.1 * mlna / N + 0.05 * mk / N);
  }
  free(inv);
  return 0;
}
