/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the DDSG evaluation path.
 *
 * A plain-C restatement of the reference's evaluation algorithm, used by
 * tests/ (parity checker), __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  Never linked into, or called by, the product library.
 *
 * Each function follows the reference file:line it cites
 * (/root/reference/proj/include/ddsg/...).  The restatement is pinned against
 * the reference itself (oracle/_ref/libddsg_ref.so, built from the reference
 * headers in place) and against the reference's own known-answer tests
 * (tests/test_oracle_pins.py); the golden fixtures under tests/golden/ were
 * produced by the reference (tests/golden/make_golden.py).
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off is load-bearing: the reference's Release build rounds
 * every product and sum separately (no FMA).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* grid_index.hpp:24-29 */
static int level_of(uint32_t hk) { return hk == 0 ? 0 : 32 - __builtin_clz(hk); }
static uint32_t index_of(uint32_t hk) {
  const int l = level_of(hk);
  return 2u * (hk - (1u << (l - 1))) + 1u;
}

/* basis.hpp:27-54: basis_kind + basis_value with inv_h = ldexp(1, l),
 * center = index / inv_h.  mode 0 = zero_boundary, 1 = modified_linear. */
double oracle_basis_value(int mode, int level, uint32_t index, double x) {
  const double inv_h = ldexp(1.0, level);
  const double center = (double)index / inv_h;
  double v;
  if (mode == 1) {
    if (level == 1) return 1.0;
    if (index == 1u) {
      v = 2.0 - x * inv_h;
      return v > 0.0 ? v : 0.0;
    }
    if (index == (1u << level) - 1u) {
      v = 2.0 - (1.0 - x) * inv_h;
      return v > 0.0 ? v : 0.0;
    }
  }
  v = 1.0 - fabs(x - center) * inv_h;
  return v > 0.0 ? v : 0.0;
}

/* sparse_grid.hpp:111-128: linear scan over the nodes in stored order,
 * w = prod_j basis_value with early exit on 0, out[c] += w * s[c]. */
static void interpolate_one(int dim, int m, int mode, int64_t n_nodes, const uint32_t* keys,
                            const double* surplus, const double* x, double* out) {
  for (int c = 0; c < m; ++c) out[c] = 0.0;
  for (int64_t nn = 0; nn < n_nodes; ++nn) {
    double w = 1.0;
    const uint32_t* key = keys + nn * dim;
    for (int j = 0; j < dim; ++j) {
      w *= oracle_basis_value(mode, level_of(key[j]), index_of(key[j]), x[j]);
      if (w == 0.0) break;
    }
    if (w != 0.0) {
      const double* s = surplus + nn * m;
      for (int c = 0; c < m; ++c) out[c] += w * s[c];
    }
  }
}

/* check_query (sparse_grid.hpp:188-196) / check_point (hdmr.hpp:299-304). */
static int point_ok(const double* x, int dim) {
  for (int j = 0; j < dim; ++j)
    if (!(x[j] >= 0.0 && x[j] <= 1.0)) return 0;
  return 1;
}

/* Batch of interpolate calls; returns 0, or 2 with *bad = lowest offending
 * point index (the task_error convention of runtime.hpp:104-137). */
int oracle_grid_eval(int dim, int m, int mode, int64_t n_nodes, const uint32_t* keys, const double* surplus,
                     const double* x, int64_t n, double* y, int64_t* bad) {
  *bad = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (!point_ok(x + i * dim, dim)) {
      *bad = i;
      return 2;
    }
    interpolate_one(dim, m, mode, n_nodes, keys, surplus, x + i * dim, y + i * m);
  }
  return 0;
}

/* Support statistics of one grid at x: nnz and FNV-1a over (slot, node)
 * pairs with w != 0 in node order. */
static void support_one(int slot, int dim, int mode, int64_t n_nodes, const uint32_t* keys, const double* x,
                        int64_t* nnz, uint64_t* h) {
  for (int64_t nn = 0; nn < n_nodes; ++nn) {
    double w = 1.0;
    const uint32_t* key = keys + nn * dim;
    for (int j = 0; j < dim; ++j) {
      w *= oracle_basis_value(mode, level_of(key[j]), index_of(key[j]), x[j]);
      if (w == 0.0) break;
    }
    if (w != 0.0) {
      const uint64_t kk = ((uint64_t)(uint32_t)slot << 32) | (uint32_t)nn;
      ++*nnz;
      for (int b = 0; b < 8; ++b) {
        *h ^= (kk >> (8 * b)) & 0xffull;
        *h *= 0x100000001b3ull;
      }
    }
  }
}

int oracle_grid_support(int dim, int mode, int64_t n_nodes, const uint32_t* keys, const double* x, int64_t n,
                        int64_t* nnz, uint64_t* hash) {
  for (int64_t i = 0; i < n; ++i) {
    if (!point_ok(x + i * dim, dim)) return 2;
    nnz[i] = 0;
    hash[i] = 0xcbf29ce484222325ull;
    support_one(0, dim, mode, n_nodes, keys, x + i * dim, &nnz[i], &hash[i]);
  }
  return 0;
}

/* ddsg_eval.hpp:154-158. */
static double pairwise_sum(const double* v, int64_t n, int64_t stride) {
  if (n == 1) return v[0];
  const int64_t half = n / 2;
  return pairwise_sum(v, half, stride) + pairwise_sum(v + half * stride, n - half, stride);
}

/* HDMR slot table in coeff_b order (empty index first).  Per slot s:
 * slot_order[s] dims (concatenated in slot_dims), b[s], and for non-empty
 * slots a grid: grid_mode[s], grid_n[s] nodes whose keys / surpluses are
 * concatenated (slot order) in grid_keys ([n][order]) / grid_surplus ([n][m]).
 * Evaluation follows VectorizedDdsg::evaluate (ddsg_eval.hpp:83-113):
 * row = b * f_anchor for the empty slot, row = interpolate(x|u) then
 * row[c] *= b otherwise; out[c] = pairwise_sum over the active rows. */
typedef struct {
  int order;
  const int32_t* dims;
  int b;
  int mode;
  int64_t n;
  const uint32_t* keys;
  const double* surplus;
} oracle_slot;

static oracle_slot* make_slots(int m, int n_slots, const int32_t* slot_order, const int32_t* slot_dims,
                               const int32_t* b, const int32_t* grid_mode, const int64_t* grid_n,
                               const uint32_t* grid_keys, const double* grid_surplus) {
  oracle_slot* slots = (oracle_slot*)calloc((size_t)n_slots, sizeof(oracle_slot));
  int64_t doff = 0, koff = 0, soff = 0;
  for (int s = 0; s < n_slots; ++s) {
    slots[s].order = slot_order[s];
    slots[s].dims = slot_dims + doff;
    slots[s].b = b[s];
    slots[s].mode = grid_mode[s];
    slots[s].n = slot_order[s] ? grid_n[s] : 0;
    slots[s].keys = grid_keys + koff;
    slots[s].surplus = grid_surplus + soff;
    doff += slot_order[s];
    koff += slots[s].n * slot_order[s];
    soff += slots[s].n * m;
  }
  return slots;
}

int oracle_hdmr_eval(int d, int m, const double* f_anchor, int n_slots, const int32_t* slot_order,
                     const int32_t* slot_dims, const int32_t* b, const int32_t* grid_mode, const int64_t* grid_n,
                     const uint32_t* grid_keys, const double* grid_surplus, const double* x, int64_t n, double* y,
                     int64_t* bad) {
  *bad = -1;
  oracle_slot* slots = make_slots(m, n_slots, slot_order, slot_dims, b, grid_mode, grid_n, grid_keys, grid_surplus);
  int na = 0;
  for (int s = 0; s < n_slots; ++s) na += slots[s].b != 0;
  double* rows = (double*)malloc(sizeof(double) * (size_t)(na > 0 ? na : 1) * (size_t)m);
  double xr[64];
  int rc = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double* xp = x + i * d;
    if (!point_ok(xp, d)) {
      *bad = i;
      rc = 2;
      break;
    }
    int a = 0;
    for (int s = 0; s < n_slots; ++s) {
      if (slots[s].b == 0) continue;
      double* row = rows + (int64_t)a * m;
      if (slots[s].order == 0) {
        for (int c = 0; c < m; ++c) row[c] = slots[s].b * f_anchor[c];
      } else {
        for (int j = 0; j < slots[s].order; ++j) xr[j] = xp[slots[s].dims[j]];
        interpolate_one(slots[s].order, m, slots[s].mode, slots[s].n, slots[s].keys, slots[s].surplus, xr, row);
        for (int c = 0; c < m; ++c) row[c] *= slots[s].b;
      }
      ++a;
    }
    for (int c = 0; c < m; ++c) y[i * m + c] = na == 0 ? 0.0 : pairwise_sum(rows + c, na, m);
  }
  free(rows);
  free(slots);
  return rc;
}

int oracle_hdmr_support(int d, int m, int n_slots, const int32_t* slot_order, const int32_t* slot_dims,
                        const int32_t* b, const int32_t* grid_mode, const int64_t* grid_n, const uint32_t* grid_keys,
                        const double* grid_surplus, const double* x, int64_t n, int64_t* nnz, uint64_t* hash) {
  oracle_slot* slots = make_slots(m, n_slots, slot_order, slot_dims, b, grid_mode, grid_n, grid_keys, grid_surplus);
  double xr[64];
  int rc = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double* xp = x + i * d;
    if (!point_ok(xp, d)) {
      rc = 2;
      break;
    }
    nnz[i] = 0;
    hash[i] = 0xcbf29ce484222325ull;
    for (int s = 0; s < n_slots; ++s) {
      if (slots[s].b == 0 || slots[s].order == 0) continue;
      for (int j = 0; j < slots[s].order; ++j) xr[j] = xp[slots[s].dims[j]];
      support_one(s, slots[s].order, slots[s].mode, slots[s].n, slots[s].keys, xr, &nnz[i], &hash[i]);
    }
  }
  free(slots);
  return rc;
}

/* Telescoping coefficients by the subset-lattice walk of
 * proj/tests/oracles.hpp:72-81 (b_i = sum over family members u >= i of
 * (-1)^(|u|-|i|)), here for a family given as sorted dim lists.
 * family_order[f], family_dims (concatenated); out_b[f]. */
int oracle_b_coefficients(int n_family, const int32_t* family_order, const int32_t* family_dims, int32_t* out_b) {
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_family + 1));
  off[0] = 0;
  for (int f = 0; f < n_family; ++f) off[f + 1] = off[f] + family_order[f];
  for (int i = 0; i < n_family; ++i) {
    int bi = 0;
    for (int u = 0; u < n_family; ++u) {
      /* is family[u] a superset of family[i]? (component_index.hpp:33-35) */
      int ok = 1;
      int64_t p = off[u];
      for (int64_t q = off[i]; q < off[i + 1] && ok; ++q) {
        while (p < off[u + 1] && family_dims[p] < family_dims[q]) ++p;
        if (p == off[u + 1] || family_dims[p] != family_dims[q]) ok = 0;
      }
      if (!ok) continue;
      bi += ((family_order[u] - family_order[i]) % 2 == 0) ? 1 : -1;
    }
    out_b[i] = bi;
  }
  free(off);
  return 0;
}

/* std::mt19937_64 (the standard's parameters) + libstdc++'s
 * generate_canonical<double, 53> (one 64-bit draw: (double)u / 2^64, clamped
 * below 1) = std::uniform_real_distribution<double>(0,1) as used by
 * proj/tests/oracles.hpp:45-53. */
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

void oracle_uniform_points(uint64_t seed, int64_t n, int dim, double* out) {
  mt64* s = (mt64*)malloc(sizeof(mt64));
  mt64_seed(s, seed);
  for (int64_t i = 0; i < n * dim; ++i) {
    double r = (double)mt64_next(s) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    out[i] = r;
  }
  free(s);
}
