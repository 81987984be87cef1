/*
 * ddsg_b200.h — C-ABI of the B200-native DDSG evaluation path.
 *
 * This is the drop-in boundary for the hot path of arXiv 2202.06555 (batched
 * evaluation of piecewise-linear hierarchical sparse-grid interpolants composed
 * as a cut-HDMR sum).  Every entry point replaces one call of the reference's
 * header-only C++ API (/root/reference/proj/include/ddsg/, cited below as
 * file:line); the C++ shim in include/ddsg_b200.hpp re-raises the reference's
 * exception types on top of the status codes returned here.
 *
 * Conventions
 *  - No entry point throws.  Every function returns a ddsg_status; on failure
 *    ddsg_last_error() returns a thread-local message.
 *  - Points are row-major x[n][dim], outputs row-major y[n][m] (replacing the
 *    reference's vector<vector<double>>, ddsg_eval.hpp:130-139).
 *  - x / y may be host or device pointers (detected with
 *    cudaPointerGetAttributes).  Device buffers are used in place; pinned
 *    host buffers are copied in pipelined chunks over three streams;
 *    ordinary (pageable) host buffers -- std::vector, numpy -- are staged
 *    through pinned buffers in pipelined chunks (the same path as the
 *    EvalWorkspace calls below).
 *  - Heap keys follow grid_index.hpp:1-38: a 1-d node (l, i) is packed as
 *    hk = 2^(l-1) + (i-1)/2, l in [1, 30].
 *  - Objects are immutable after creation except through ddsg_grid_append
 *    (refinement), which needs external synchronisation, like the reference
 *    (SPEC.md:109,270).
 */
#ifndef DDSG_B200_H_
#define DDSG_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. */
typedef enum {
  DDSG_OK = 0,
  DDSG_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  DDSG_DOMAIN_ERROR = 2,     /* std::domain_error (x outside [0,1] or NaN) */
  DDSG_CUDA_ERROR = 3,
  DDSG_NCCL_ERROR = 4,
  DDSG_OUT_OF_MEMORY = 5,
  DDSG_BUILD_ERROR = 6,      /* ddsg::build_error: evaluator returned non-finite */
  DDSG_OUT_OF_RANGE = 7      /* std::out_of_range (node lookup) */
} ddsg_status;

/* basis.hpp:22 BoundaryMode. */
typedef enum { DDSG_ZERO_BOUNDARY = 0, DDSG_MODIFIED_LINEAR = 1 } ddsg_boundary_mode;

/* sparse_grid.hpp:53 SurplusNorm. */
typedef enum { DDSG_NORM_INF = 0, DDSG_NORM_L2 = 1 } ddsg_surplus_norm;

/* Evaluation arithmetic.  EXACT (the default) reproduces the reference
 * rounding sequence bit for bit (mul then add per node in canonical order,
 * x b, pairwise slot sum).  FAST contracts the per-node mul+add into one FMA
 * (same order).  FAST carries NO tolerance guarantee: its per-slot rounding
 * differs from the reference's by up to ~n u |row| and HDMR sums cancel
 * (sum |b_s row_s| is ~10^2-10^3 x |y| on the BASELINE configs), so it can
 * exceed 1e-14 abs + 1e-12 rel on a small fraction of outputs (measured
 * rates: DESIGN.md §3.1).  Use it only where that is acceptable. */
typedef enum { DDSG_EVAL_EXACT = 0, DDSG_EVAL_FAST = 1 } ddsg_eval_mode;

typedef struct ddsg_grid ddsg_grid_t; /* SparseGridFunction (sparse_grid.hpp:72) */
typedef struct ddsg_hdmr ddsg_hdmr_t; /* VectorizedDdsg (ddsg_eval.hpp:28) over a DdsgFunction (hdmr.hpp:195) */

/* Thread-local message for the last failing call on this thread. */
const char* ddsg_last_error(void);

/* Library / device information: number of visible CUDA devices (0 if none). */
int ddsg_device_count(void);

/* ------------------------------------------------------------------ grids */

/* Replaces SparseGridFunction::from_nodes (sparse_grid.hpp:160-179).
 * heap_keys: [n_nodes][dim] uint32, surplus: [n_nodes][m] fp64, both in the
 * caller's (stored) node order, which nodes() reports back.  Evaluation walks
 * the nodes in canonical order (level sum, heap-key lexicographic).
 * Errors: INVALID_ARGUMENT on dim/m < 1, key validation failure (level > 30
 * or malformed), duplicate keys (sparse_grid.hpp:172-175). */
ddsg_status ddsg_grid_create(int dim, int m, int mode, int max_level, double eps_gamma,
                             int64_t n_nodes, const uint32_t* heap_keys, const double* surplus,
                             ddsg_grid_t** out);

/* Batched evaluator used by ddsg_grid_build: writes f(xs[i]) into out[i] for
 * i < count (xs: [count][dim], out: [count][m]).  A non-zero return value
 * aborts the build with DDSG_BUILD_ERROR.  Replaces GridEvaluator
 * (sparse_grid.hpp:70), batched so a caller can vectorise. */
typedef int (*ddsg_batch_evaluator)(const double* xs, int64_t count, double* out, void* ctx);

/* Replaces SparseGridFunction::build (sparse_grid.hpp:84-108) with
 * SgBuildOptions{max_level, eps_gamma, mode, norm} (sparse_grid.hpp:61-67):
 * level-sum sweep, children of significant nodes closed under missing
 * ancestors and sorted by (level sum, key), residual hierarchization
 * surplus = f(x) - interpolate(grid so far, x) in insertion order.
 * A non-finite evaluator output yields DDSG_BUILD_ERROR with the offending
 * point reported through ddsg_last_build_point. */
ddsg_status ddsg_grid_build(int dim, int m, int mode, int max_level, double eps_gamma, int norm,
                            ddsg_batch_evaluator f, void* ctx, ddsg_grid_t** out);

/* Coordinates of the point that made the last build fail on this thread
 * (build_error::point, sparse_grid.hpp:40-48).  Returns its length. */
int ddsg_last_build_point(double* out, int capacity);

/* Appends refinement nodes (the only mutation).  Keys must
 * be new.  Device tables are rebuilt lazily on the next evaluation. */
ddsg_status ddsg_grid_append(ddsg_grid_t* g, int64_t n_new, const uint32_t* heap_keys,
                             const double* surplus);

/* Residual hierarchization of new nodes against the current grid on the GPU
 * (sparse_grid.hpp:264-276,302-315): surplus_out[i] = f_values[i] -
 * interpolate(g, x(keys[i])).  f_values / surplus_out: both host or both
 * device memory (device rows stay on the device, e.g. for an all-gather).
 * Does not modify g. */
ddsg_status ddsg_hierarchize(const ddsg_grid_t* g, int64_t n_new, const uint32_t* heap_keys,
                             const double* f_values, double* surplus_out);

/* Host (CPU) residual hierarchization, bit-identical to the reference's
 * insert_batch (sparse_grid.hpp:264-276): interpolation at each new node over
 * the current nodes in stored order.  Used where no GPU is present. */
ddsg_status ddsg_hierarchize_host(const ddsg_grid_t* g, int64_t n_new, const uint32_t* heap_keys,
                                  const double* f_values, double* surplus_out);

/* Refinement candidates from level sum s (sparse_grid.hpp:215-254): children
 * of every node at level sum s whose surplus passes the grid's criterion
 * (eps_gamma, norm), closed under missing ancestors, sorted by (level sum,
 * key) — the next batch the reference's build would insert.  Call with
 * heap_keys == NULL to get the count in *n_out. */
ddsg_status ddsg_grid_refine_candidates(const ddsg_grid_t* g, int level_sum, int64_t* n_out, uint32_t* heap_keys);

ddsg_status ddsg_grid_destroy(ddsg_grid_t* g);

/* Accessors (sparse_grid.hpp:74-81). */
ddsg_status ddsg_grid_info(const ddsg_grid_t* g, int* dim, int* m, int* mode, int* max_level,
                           double* eps_gamma, int64_t* n_nodes);
/* Copies nodes in stored order: keys [n][dim], surplus [n][m] (either may be NULL). */
ddsg_status ddsg_grid_nodes(const ddsg_grid_t* g, uint32_t* heap_keys, double* surplus);
/* SparseGridFunction::contains / node_at (sparse_grid.hpp:151-157): *index =
 * the stored position of the node with this key ([dim] heap keys), or -1. */
ddsg_status ddsg_grid_find(const ddsg_grid_t* g, const uint32_t* heap_key, int64_t* index);
/* SparseGridFunction::quadrature (sparse_grid.hpp:138-149), host, fixed node order. */
ddsg_status ddsg_grid_quadrature(const ddsg_grid_t* g, double* out);

/* Replaces SparseGridFunction::interpolate (sparse_grid.hpp:111-128) over a
 * batch: y[i] = interpolate(x[i]).  *bad_index receives the lowest point index
 * outside [0,1]^dim (or NaN) and the call returns DDSG_DOMAIN_ERROR, mirroring
 * detail::for_each_index's lowest-task-id task_error (runtime.hpp:104-137).
 * stream: a cudaStream_t (NULL = legacy default stream).  Synchronous. */
ddsg_status ddsg_eval_grid(const ddsg_grid_t* g, const double* x, int64_t n, double* y,
                           int64_t* bad_index, void* stream);

/* ------------------------------------------------------------------- HDMR */

/* Replaces DdsgFunction::from_parts (hdmr.hpp:307-325) + VectorizedDdsg::compile
 * (ddsg_eval.hpp:40-74).  Slots must be given in the reference's coeff_b order:
 * the empty index first, then (order, lexicographic) (component_index.hpp:25-28).
 *   slot_order[s]   = |u_s|
 *   slot_dims       = concatenated dims of every slot (strictly increasing per slot)
 *   b[s]            = integer telescoping coefficient
 *   grids[s]        = grid of slot s (NULL for the empty index; dim == |u_s|)
 *   f_anchor        = [m] anchor values
 * Slots with b == 0 are kept but skipped in evaluation (ddsg_eval.hpp:71-72).
 * Errors: INVALID_ARGUMENT on a missing empty slot, unsorted slots, a grid of
 * the wrong dimension or output length, or a family that is not downward
 * closed (ddsg_eval.hpp:61-70). The grids are copied; the caller keeps ownership. */
ddsg_status ddsg_hdmr_create(int d, int m, const double* f_anchor, int n_slots,
                             const int32_t* slot_order, const int32_t* slot_dims, const int32_t* b,
                             const ddsg_grid_t* const* grids, ddsg_hdmr_t** out);

ddsg_status ddsg_hdmr_destroy(ddsg_hdmr_t* h);

ddsg_status ddsg_hdmr_info(const ddsg_hdmr_t* h, int* d, int* m, int* n_slots, int* n_active,
                           int64_t* n_nodes);

/* Replaces VectorizedDdsg::evaluate_batch (ddsg_eval.hpp:130-139): y[i] =
 * sum over active slots (pairwise, ddsg_eval.hpp:154-158) of b_s * interp_s(x[i]|u_s).
 * Errors as ddsg_eval_grid.  Synchronous. */
ddsg_status ddsg_eval_hdmr(const ddsg_hdmr_t* h, const double* x, int64_t n, double* y,
                           int64_t* bad_index, void* stream);

/* VectorizedDdsg::quadrature (ddsg_eval.hpp:143-151), host. */
ddsg_status ddsg_hdmr_quadrature(const ddsg_hdmr_t* h, double* out);

/* Slot s of the table in coeff_b order (VectorizedDdsg::slots(),
 * ddsg_eval.hpp:77; the empty index first): its order, dims (caller buffer
 * of >= order entries, may be NULL), coefficient b, and a NEW grid handle
 * holding a copy of its grid (NULL for the empty index; the caller destroys
 * it; pass grid == NULL to skip the copy).  OUT_OF_RANGE if s is outside
 * [0, n_slots). */
ddsg_status ddsg_hdmr_slot(const ddsg_hdmr_t* h, int s, int* order, int32_t* dims, int32_t* b, ddsg_grid_t** grid);

/* --------------------------------------------------------- JSON documents
 *
 * The reference's versioned documents (serialize.hpp, schema_version 1):
 * surpluses and coordinates are JSON numbers written with shortest
 * round-trip digits, so save/load is bit-exact (serialize.hpp:3-5).  Text in,
 * text out (the caller owns the file I/O, like load_json / save_json,
 * serialize.hpp:147-160).  `len` < 0 means NUL-terminated.  Writers: call
 * with buf == NULL to get the size in *len_out (bytes, without the NUL),
 * then with a buffer of at least *len_out + 1 bytes; the text is the
 * reference's save_json layout (dump(2) plus a newline). */

/* sparse_grid_from_json (serialize.hpp:54-77) -> a grid handle.  Errors:
 * INVALID_ARGUMENT on malformed JSON, a missing key, a wrong schema version
 * or type tag, a bad heap key (grid_index.hpp:32-39) or from_nodes'
 * checks (sparse_grid.hpp:168-175). */
ddsg_status ddsg_grid_from_json(const char* text, int64_t len, ddsg_grid_t** out);
/* to_json(SparseGridFunction) (serialize.hpp:31-52), nodes in stored order. */
ddsg_status ddsg_grid_to_json(const ddsg_grid_t* g, char* buf, int64_t cap, int64_t* len_out);

/* The reference's ddsg_from_json, serialize.hpp:112-145, then VectorizedDdsg::compile
 * (ddsg_eval.hpp:40-74): the document's policy as an evaluator, slots in
 * coeff_b order.  The document's k_max, anchor coordinates, rejected set and
 * cut quadratures are kept for ddsg_hdmr_to_json / ddsg_hdmr_document.
 * Errors: as ddsg_grid_from_json, plus compile's (coefficient for a
 * non-accepted index, missing subset, no empty slot). */
ddsg_status ddsg_hdmr_from_json(const char* text, int64_t len, ddsg_hdmr_t** out);
/* to_json(DdsgFunction) (serialize.hpp:84-110).  Needs the document fields:
 * INVALID_ARGUMENT without anchor coordinates, OUT_OF_RANGE without the cut
 * quadratures (the reference's cut_quadrature throws std::out_of_range,
 * hdmr.hpp:213-218); set them with ddsg_hdmr_set_document. */
ddsg_status ddsg_hdmr_to_json(const ddsg_hdmr_t* h, char* buf, int64_t cap, int64_t* len_out);

/* Document fields of DdsgFunction that evaluation does not use (hdmr.hpp:
 * k_max, anchor().coords, rejected(), cut_quadrature(u)):
 *   anchor_coords   [d] (NULL keeps the current value)
 *   rejected        n_rejected indices: rejected_order[r] = |u_r|, dims
 *                   concatenated in rejected_dims (sorted and validated like
 *                   ComponentIndex::make)
 *   cut_quadratures [n_slots][m] in slot order, or NULL (none) */
ddsg_status ddsg_hdmr_set_document(ddsg_hdmr_t* h, int k_max, const double* anchor_coords, int n_rejected,
                                   const int32_t* rejected_order, const int32_t* rejected_dims,
                                   const double* cut_quadratures);
/* Reads them back, plus the anchor values f_anchor [m] (any output may be
 * NULL; call first with the arrays NULL to get n_rejected / n_rejected_dims).
 * anchor_coords defaults to 0.5 when never set; *has_quadratures = 0 when no
 * quadratures are held. */
ddsg_status ddsg_hdmr_document(const ddsg_hdmr_t* h, int* k_max, double* anchor_coords, double* f_anchor,
                               int* n_rejected, int64_t* n_rejected_dims, int32_t* rejected_order,
                               int32_t* rejected_dims, int* has_quadratures, double* cut_quadratures);

/* ------------------------------------------- distributed refinement step
 *
 * One adaptive refinement step of replicated grids (the
 * path's only collective), orchestrated natively.  For grid g the new batch
 * is the reference's next build batch from level sum level_sums[g]
 * (next_candidates, sparse_grid.hpp:215-254), processed in level-sum groups;
 * per group round the new nodes of all grids are split into equal, padded,
 * contiguous shares over the ranks; each rank evaluates the target at its
 * share (callback), hierarchizes it (surplus = f - interpolate, EXACT, on
 * the GPU when on_device != 0, else on the host), the surplus rows
 * [world][share][m] are all-gathered and every rank appends the whole group
 * in batch order (insert_batch, sparse_grid.hpp:256-298).  The grids stay
 * bit-identical on every rank and equal to the reference's build at the
 * next level.  Mutates the grids (external synchronisation, like
 * ddsg_grid_append). */
typedef int (*ddsg_node_evaluator)(int grid, const double* xs, int64_t count, double* out, void* ctx);
/* All-gather of bytes_per_rank bytes from every rank into recv
 * [world][bytes_per_rank] (device buffers when on_device).  Returns 0 on success. */
typedef int (*ddsg_allgather_fn)(const void* send, void* recv, int64_t bytes_per_rank, void* ctx);
typedef struct {
  int64_t new_nodes, rounds, gathered_bytes;
  double target_s, hierarchize_s, allgather_s;
} ddsg_refine_stats;
/* allgather may be NULL for a single process (world == 1).  Errors:
 * INVALID_ARGUMENT, BUILD_ERROR (non-finite target value; the node through
 * ddsg_last_build_point), NCCL_ERROR (the all-gather returned non-zero). */
ddsg_status ddsg_refine_step(ddsg_grid_t* const* grids, int n_grids, const int* level_sums, ddsg_node_evaluator f,
                             void* f_ctx, int rank, int world, ddsg_allgather_fn allgather, void* ag_ctx,
                             int on_device, ddsg_refine_stats* stats);
/* The same step over a caller's NCCL communicator (an ncclComm_t, e.g. the
 * C++ host's, or torch's ProcessGroupNCCL._comm_ptr()): device buffers,
 * ncclAllGather(ncclFloat64) on `stream` (a cudaStream_t) over NVLink.
 * libnccl.so.2 is resolved at the first call (the library does not link
 * it).  nccl_comm may be NULL only for world == 1. */
ddsg_status ddsg_refine_step_nccl(ddsg_grid_t* const* grids, int n_grids, const int* level_sums,
                                  ddsg_node_evaluator f, void* f_ctx, void* nccl_comm, int rank, int world,
                                  void* stream, ddsg_refine_stats* stats);

/* ---------------------------------------------------- evaluation workspace
 *
 * EvalWorkspace (ddsg_eval.hpp:21-24): reusable buffers for allocation-free
 * evaluation in hot loops.  A workspace owns pinned host staging, device
 * buffers and a stream on the device current at first use; x / y passed to
 * the _ws calls are ordinary (pageable) host memory, staged through the
 * pinned buffers in pipelined chunks.  A workspace is not thread-safe (the
 * reference keeps one per thread: thread_local EvalWorkspace,
 * time_iteration.hpp:88). */
typedef struct ddsg_workspace ddsg_workspace_t;
ddsg_status ddsg_workspace_create(ddsg_workspace_t** out);
ddsg_status ddsg_workspace_destroy(ddsg_workspace_t* ws);
/* VectorizedDdsg::evaluate(x, out, ws, interp_calls) (ddsg_eval.hpp:83-113)
 * over n host points: y[i] = evaluate(x[i]); *interp_calls (may be NULL) is
 * incremented by n x the number of active non-empty slots, the reference's
 * per-point count of cut interpolations.  Errors as ddsg_eval_hdmr. */
ddsg_status ddsg_eval_hdmr_ws(const ddsg_hdmr_t* h, ddsg_workspace_t* ws, const double* x, int64_t n, double* y,
                              int64_t* bad_index, uint64_t* interp_calls);
/* VectorizedDdsg::evaluate_batch in the reference's vector<vector<double>>
 * convention (ddsg_eval.hpp:130-139): point i is read from xrows[i] (dim
 * doubles) and its outputs written to yrows[i] (m doubles); the rows are
 * gathered / scattered straight into / out of the pinned staging buffers
 * (no flattened copy).  Errors as ddsg_eval_hdmr. */
ddsg_status ddsg_eval_hdmr_rows(const ddsg_hdmr_t* h, ddsg_workspace_t* ws, const double* const* xrows, int64_t n,
                                double* const* yrows, int64_t* bad_index);
/* SparseGridFunction::interpolate over n host points through a workspace. */
ddsg_status ddsg_eval_grid_ws(const ddsg_grid_t* g, ddsg_workspace_t* ws, const double* x, int64_t n, double* y,
                              int64_t* bad_index);

/* --------------------------------------------------------------- controls */

/* Selects the arithmetic of subsequent evaluations on this object. */
ddsg_status ddsg_grid_set_eval_mode(ddsg_grid_t* g, int eval_mode);
ddsg_status ddsg_hdmr_set_eval_mode(ddsg_hdmr_t* h, int eval_mode);

/* Kernel statistics of the last evaluation on this thread: number of kernel
 * launches issued, the device time (ms) of the whole evaluation (device-
 * resident calls; 0 for host-buffer calls) and of the dominant evaluation
 * kernel alone, measured with CUDA events on the launching stream(s). */
ddsg_status ddsg_last_eval_stats(int64_t* launches, double* kernel_ms, double* main_kernel_ms);

/* 1 if the HDMR evaluates on the slot-staged kernel (all active slots of
 * order <= 2 within its static level limits), 0 for the generic kernel. */
ddsg_status ddsg_hdmr_kernel_path(const ddsg_hdmr_t* h, int* fast_path);

/* Measures the FP64 DFMA and DMMA (mma.sync f64) peaks of the current device
 * in TFLOP/s (roofline denominators; microbenchmark, ~0.1 s). */
ddsg_status ddsg_measure_fp64_peak(double* dfma_tflops, double* dmma_tflops);

/* Support statistics (test / roofline helper, computed on the device):
 * nnz[i] = number of (slot, node) pairs with w != 0 at x[i]; hash[i] = an
 * order-sensitive FNV-1a hash of the (slot, stored node index) pairs in
 * evaluation order.  x, nnz, hash: host or device. */
ddsg_status ddsg_hdmr_support(const ddsg_hdmr_t* h, const double* x, int64_t n, int64_t* nnz,
                              uint64_t* hash, void* stream);
ddsg_status ddsg_grid_support(const ddsg_grid_t* g, const double* x, int64_t n, int64_t* nnz,
                              uint64_t* hash, void* stream);

/* Seeded uniform points exactly as std::mt19937_64 +
 * std::uniform_real_distribution<double>(0,1) (libstdc++), point-major, as
 * the reference's test oracle generates them (proj/tests/oracles.hpp:45-53). */
void ddsg_uniform_points(uint64_t seed, int64_t n, int dim, double* out);

/* Blocked form of the same generator for sharded benchmarks: block b holds
 * block_points points drawn from std::mt19937_64(seed + b) +
 * uniform_real_distribution(0,1), point-major.  Writes points
 * [first, first + n) of that stream into out[n][dim] (host memory), blocks
 * generated on several host threads; any contiguous range -- a rank's shard
 * -- is therefore generated independently of how the set is split, and the
 * oracle reproduces block b with a plain seeded draw. */
void ddsg_uniform_point_blocks(uint64_t seed, int64_t block_points, int64_t first, int64_t n, int dim,
                               double* out);

/* ------------------------------------------------ batched policy callers
 *
 * the time iteration's consumers of the policy
 * interpolant, restructured so that every successor state of a whole batch
 * of grid points / samples is evaluated in ONE batched policy evaluation on
 * the device.  The policy is a device object: exactly one of policy_hdmr /
 * policy_grid is non-NULL (the reference's PolicyEvaluator built by
 * compiled_evaluator, time_iteration.hpp:86-91).  Its input is the canonical
 * state x in [0,1]^(2N) (N log-productivities, then N capitals) and its
 * output the flat policy (k'[N], mu[N] for the non-smooth variant, lambda)
 * (irbc.hpp:215-236).  Buffers may be host or device memory. */

typedef enum { DDSG_IRBC_SMOOTH = 0, DDSG_IRBC_NONSMOOTH = 1 } ddsg_irbc_variant;

/* IrbcParameters (irbc.hpp:27-53) in flat form.  gamma and tau point to
 * caller-owned arrays of `countries` doubles. */
typedef struct {
  int countries;
  int variant; /* ddsg_irbc_variant */
  double beta, alpha, delta, sigma, rho_a, phi_adj, gamma_base;
  double lna_half_width, k_lo, k_hi;
  double A;      /* derived */
  double* gamma; /* [countries] */
  double* tau;   /* [countries], derived */
} ddsg_irbc_params;

/* refresh_derived (irbc.hpp:59-92): validates, fills gamma when fill_gamma
 * != 0 (gamma_j = gamma_base + 0.75 j/(N-1)), then A and tau.  Errors:
 * INVALID_ARGUMENT with the reference's messages. */
ddsg_status ddsg_irbc_refresh_derived(ddsg_irbc_params* p, int fill_gamma);

/* steady_state_lambda (irbc.hpp:248-263), host bisection. */
ddsg_status ddsg_irbc_steady_state_lambda(const ddsg_irbc_params* p, double* lambda);

/* foc_residuals (irbc.hpp:306-361) for n states at once:
 *   a, k        [n][N]      state (productivity levels, capitals)
 *   candidate   [n][pdim]   flat candidate policy (pdim = N+1 or 2N+1)
 *   residuals   [n][pdim]   out
 *   clamped     [n]         out (may be NULL): successor states clamped into
 *                           the box, the reference's return value
 * All 2(N+1) successor states of all n points are evaluated by one batched
 * policy call.  Errors: INVALID_ARGUMENT (bad parameters/handles),
 * DOMAIN_ERROR when a successor state is NaN (the reference's
 * check_point), *bad_index = the lowest failing state. */
ddsg_status ddsg_irbc_foc_residuals(const ddsg_hdmr_t* policy_hdmr, const ddsg_grid_t* policy_grid,
                                    const ddsg_irbc_params* p, int64_t n, const double* a, const double* k,
                                    const double* candidate, double* residuals, int32_t* clamped,
                                    int64_t* bad_index, void* stream);

/* foc_jacobian (solver.hpp:129-165) for n states at once: forward
 * differences jac[i][r][c] = (res(z_i + h_c e_c)[r] - r0[i][r]) / h_c with
 * h_c = fd_epsilon * max(|z_ic|, 1e-2), then (non-smooth variant) the
 * Fischer-Burmeister rows replaced by their generalized derivative.
 *   z, r0 [n][pdim], jac [n][pdim][pdim] (row-major, jac[i][r][c]).
 * Perturbing mu or lambda leaves the successor states unchanged, so only
 * 1 + N distinct successor sets per point are evaluated (one batched call). */
ddsg_status ddsg_irbc_foc_jacobian(const ddsg_hdmr_t* policy_hdmr, const ddsg_grid_t* policy_grid,
                                   const ddsg_irbc_params* p, int64_t n, const double* a, const double* k,
                                   const double* z, const double* r0, double fd_epsilon, double* jac,
                                   int64_t* bad_index, void* stream);

/* euler_errors (solver.hpp:377-436) on caller-supplied canonical samples
 * xs[n][2N] (the reference draws them with std::mt19937_64(seed) +
 * uniform_real_distribution(0,1), point-major: ddsg_uniform_points):
 *   errs[n]     per-sample worst-country relative Euler error (out)
 *   mean, worst sequential mean / max over errs (out; log10 is the caller's)
 *   clamp_count successor states clamped into the box, summed (out, may be NULL) */
ddsg_status ddsg_irbc_euler_errors(const ddsg_hdmr_t* policy_hdmr, const ddsg_grid_t* policy_grid,
                                   const ddsg_irbc_params* p, int64_t n, const double* xs, double* errs,
                                   double* mean, double* worst, uint64_t* clamp_count, int64_t* bad_index,
                                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DDSG_B200_H_ */
