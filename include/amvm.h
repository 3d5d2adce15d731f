/*
 * amvm.h — C-ABI of the B200-native AMVM inner loop (libamvm.so).
 *
 * The reference (`dmmv`, a pure-Python package) has no FFI: its boundary is
 * the Python call `dmmv.solve(inst, cfg) -> SolveReport`
 * (/root/reference/pkg/src/dmmv/controller.py:211) plus the component
 * functions it is built from.  Every entry point below replaces one of those
 * Python functions; the Python host mirror (`paper_2508_13437_b200`) binds
 * them with ctypes exactly as a maintainer of `dmmv` would.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes; no C++ exceptions cross the ABI.
 *   - Every array pointer is a DEVICE pointer unless the name ends in `_host`.
 *   - All calls are asynchronous on the caller's `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream).
 *   - The caller owns every buffer, including the workspace sized by
 *     amvm_workspace_bytes(); the library keeps no pointer after return and
 *     holds no global mutable state (re-entrant across streams/devices).
 *   - Status: 0 = OK, negative = error; amvm_strerror() names it.  The
 *     Python mirror raises ValueError for AMVM_ERR_INVALID (same messages as
 *     the reference) and RuntimeError otherwise.
 *   - A is stored COLUMN-major (`At`: column j is the m contiguous doubles at
 *     At + j*m).  Every hot loop of the path streams columns of A
 *     (localsearch.py:73,191, core.py:222,242), so that is the layout in HBM.
 *   - Level indices are int32 (the reference uses np.intp; values < 2^31).
 */
#ifndef AMVM_H
#define AMVM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMVM_ABI_VERSION 1

#if defined(__GNUC__)
#define AMVM_API __attribute__((visibility("default")))
#else
#define AMVM_API
#endif

enum {
  AMVM_OK = 0,
  AMVM_ERR_INVALID = -1,     /* bad argument (shape, range, NULL pointer)      */
  AMVM_ERR_CUDA = -2,        /* a CUDA runtime call failed                     */
  AMVM_ERR_WORKSPACE = -3,   /* workspace smaller than amvm_workspace_bytes()  */
  AMVM_ERR_UNSUPPORTED = -4, /* shape outside what this build supports         */
  AMVM_ERR_NO_DEVICE = -5    /* no sm_100 device / kernel image not loadable   */
};

/* One problem family sharing A.  count == 1 is the single-instance solve of
 * controller.py:211; count > 1 is the shared-X batch (PTQ rows of one layer,
 * PAPER.md:147-158) that the reference drives by looping over Instances.   */
typedef struct {
  int64_t m, n, nlev, count;
  const double *At;     /* n x m, column-major A (see header comment)            */
  const double *B;      /* count x m targets b                                    */
  const double *levels; /* count x nlev strictly increasing levels (core.py:26)  */
} amvm_problem;

/* SolverConfig (controller.py:35-68) + module constants, as plain data.     */
typedef struct {
  double alpha;          /* impact decay, operators.py:54                      */
  double sigma1, sigma2, sigma3, decay;  /* controller.py:44-47                */
  double accept_tie_tol; /* ACCEPT_TIE_TOL controller.py:32                    */
  double weight_floor;   /* WEIGHT_FLOOR controller.py:31                      */
  double time_limit_s;   /* < 0: none (controller.py:236)                      */
  int32_t r;             /* removal_count(destroy_rate, n), controller.py:206  */
  int32_t k_eps;         /* FilterConfig.k_eps, localsearch.py:45               */
  int32_t max_candidates;/* <= 0: no cap (None), localsearch.py:46             */
  int32_t max_iters;     /* controller.py:40                                   */
  int32_t l2_tiebreak;   /* accept() tie-break, controller.py:48,179           */
  int32_t refresh_period;       /* REFRESH_PERIOD core.py:18                   */
  int32_t one_opt_max_sweeps;   /* ONE_OPT_MAX_SWEEPS localsearch.py:20        */
  int32_t ls_max_rounds;        /* LOCAL_SEARCH_MAX_ROUNDS localsearch.py:21   */
  int32_t n_segment;            /* N_SEGMENT controller.py:30                  */
  int32_t threads;       /* CTA size: 0 = auto (512 threads, one CTA per SM,  *
                          * when count <= SM count, else 256 x 2 per SM); 256  *
                          * or 512 force one (component calls: 256 only)       */
} amvm_params;

/* numpy PCG64 bit generator state == Generator.bit_generator.state.        */
typedef struct {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
  uint32_t has_uint32, uinteger;
} amvm_pcg64;

/* A Solution (core.py:145-180) for each of `count` instances.              */
typedef struct {
  int32_t *idx;      /* count x n level indices                              */
  double *residual;  /* count x m, s = A x - b                               */
  double *objective; /* count, max |s|                                       */
  int32_t *updates;  /* count, updates_since_refresh                         */
} amvm_solution;

/* Per-instance outputs of a solve (SolveReport, controller.py:194-203).    */
typedef struct {
  amvm_solution best;       /* best solution found                            */
  double *initial_objective;/* count                                          */
  int32_t *iterations;      /* count                                          */
  int64_t *operator_uses;   /* count x 4, PAIRS order controller.py:23-28     */
  double *trace_current_t;  /* count x max_iters (may be NULL = no trace)     */
  double *trace_best_t;     /* count x max_iters                              */
  uint8_t *trace_pair;      /* count x max_iters, PAIRS slot                  */
  uint8_t *trace_accepted;  /* count x max_iters                              */
  int64_t *moves_scored;    /* count x 2: [0] reference-equivalent candidate
                               moves scored (the candidates the reference
                               evaluates on this trajectory: 1-OPT neighbours
                               up to the applied move, 2 per greedy variable,
                               filtered swaps), [1] raw candidates the device
                               scored over all m rows (one_opt columns that
                               survive the exact row screens, greedy trials,
                               swap evaluations); may be NULL                 */
  int64_t *phase_cycles;    /* count x 16: [0..7] SM-clock cycles per phase
                               (select+copy, random destroy, impact+worst
                               destroy, repair, one_opt, find_candidates,
                               swap evaluation, accept+commit); [8..15] event
                               counts (find_candidates calls, survivors, swaps
                               applied, one_opt exact rechecks, one_opt moves,
                               one_opt windows, impact calls, refreshes);
                               may be NULL                                    */
} amvm_result;

/* ---- whole solve: replaces dmmv.solve (controller.py:211-286) ---------- */

/* Workspace bytes for amvm_solve / the component calls on this problem.    */
AMVM_API size_t amvm_workspace_bytes(const amvm_problem *prob, const amvm_params *prm);

/* Runs the ALNS loop for every instance, starting from `start` (the
 * initial_solution of controller.py:134, computed by the host) with
 * `rng[k]` (seeded state in, final state out).  `start` is not modified.   */
AMVM_API int amvm_solve(const amvm_problem *prob, const amvm_params *prm,
               const amvm_solution *start, amvm_pcg64 *rng,
               amvm_result *res, void *ws, size_t ws_bytes, void *stream);

/* ---- whole solve on a SPARSE A (tomography: density <= 1/8) ------------
 * Same semantics and results as amvm_solve (bit for bit: every zero entry
 * the dense path would add is exact), with A given only as CSC and CSR
 * (device arrays, both ascending within a column / row) -- no dense copy of
 * A anywhere, so the workspace is O(slots * (m + n)) plus the parked
 * instances.  one_opt scores each candidate from its column's nonzeros plus
 * the largest |s| among untouched rows (a top list of 2*max_col_nnz + 1
 * rows by |s|); max_col_nnz = the largest column nonzero count.           */
typedef struct {
  int64_t m, n, nlev, count, nnz, max_col_nnz;
  const int64_t *cptr; const int32_t *crow; const double *cval;  /* CSC, n + 1 / nnz / nnz */
  const int64_t *rptr; const int32_t *rcol; const double *rval;  /* CSR, m + 1 / nnz / nnz */
  const double *B;      /* count x m targets b                                    */
  const double *levels; /* count x nlev                                           */
  int64_t max_row_nnz;  /* largest row nonzero count; > 0 enables the column-     *
                         * indexed candidate filter (0: the general filter)       */
} amvm_sparse_problem;

AMVM_API size_t amvm_sparse_workspace_bytes(const amvm_sparse_problem *prob, const amvm_params *prm);
AMVM_API int amvm_solve_sparse(const amvm_sparse_problem *prob, const amvm_params *prm,
                               const amvm_solution *start, amvm_pcg64 *rng, amvm_result *res,
                               void *ws, size_t ws_bytes, void *stream);

/* ---- component calls (count == 1; the Solution is updated in place) ---- */

/* one_opt, localsearch.py:59-88 */
AMVM_API int amvm_one_opt(const amvm_problem *prob, const amvm_params *prm,
                 amvm_solution *sol, void *ws, size_t ws_bytes, void *stream);

/* local_search, localsearch.py:249-269 */
AMVM_API int amvm_local_search(const amvm_problem *prob, const amvm_params *prm,
                      amvm_solution *sol, void *ws, size_t ws_bytes,
                      void *stream);

/* find_candidates, localsearch.py:128-169: writes up to `cap` candidates in
 * reference order (descending delta, then i, then j) and *count (device
 * int32) = number written.                                                  */
AMVM_API int amvm_find_candidates(const amvm_problem *prob, const amvm_params *prm,
                         const amvm_solution *sol, int32_t *out_i,
                         int32_t *out_j, double *out_delta, int32_t *count,
                         int32_t cap, void *ws, size_t ws_bytes, void *stream);

/* best_swap, localsearch.py:211-246: out4 (device double[4]) receives
 * {i, j, delta, predicted_t}; i = -1 when no swap improves.                 */
AMVM_API int amvm_best_swap(const amvm_problem *prob, const amvm_params *prm,
                   const amvm_solution *sol, double *out4, void *ws,
                   size_t ws_bytes, void *stream);

/* best_swap with FilterConfig.l2_tiebreak (localsearch.py:181-246): the
 * candidates split like np.array_split(cands, min(workers, count)); each
 * chunk's smallest improving t' wins its chunk, ties going to the smallest
 * (l2, i, j) with l2 = np.linalg.norm(shifted, axis=1) (pairwise sum of
 * squares; a lone winner carries np.linalg.norm = sqrt(ddot)); chunk
 * winners merge by (t, l2, i, j).  out4 as amvm_best_swap.                 */
AMVM_API int amvm_best_swap_l2(const amvm_problem *prob, const amvm_params *prm,
                               const amvm_solution *sol, int32_t workers, double *out4,
                               void *ws, size_t ws_bytes, void *stream);

/* apply_shift (core.py:208-225): s += (lv[new] - lv[old]) * A[:, j]
 * (DMUL, DADD), idx[j] = new, then _bump (core.py:200-205): the counter +1
 * and objective = max|s|, or the dgemv-order refresh at refresh_period.
 * Shifting to the current level is a no-op (no counter bump).  In place.  */
AMVM_API int amvm_apply_shift(const amvm_problem *prob, const amvm_params *prm,
                              amvm_solution *sol, int64_t j, int32_t new_level,
                              void *ws, size_t ws_bytes, void *stream);

/* apply_swap (core.py:228-245): s += (x_i - x_j) * (A[:, j] - A[:, i]),
 * levels exchanged, _bump.  i != j; the values must differ (checked by the
 * host mirror, which owns the reference's error messages).  In place.     */
AMVM_API int amvm_apply_swap(const amvm_problem *prob, const amvm_params *prm,
                             amvm_solution *sol, int64_t i, int64_t j, void *ws,
                             size_t ws_bytes, void *stream);

/* accept (controller.py:168-183): verdict (device int32[1]) = 1 iff
 * cand_objective < cur_objective, or l2_tiebreak and cand_objective <=
 * cur_objective + tie_tol and ||cand||_2 < ||cur||_2 (np.linalg.norm =
 * sqrt of the OpenBLAS SkylakeX ddot).  Residuals are m doubles; the
 * objectives are device double[1].                                         */
AMVM_API int amvm_accept(int64_t m, const double *cur_residual, const double *cur_objective,
                         const double *cand_residual, const double *cand_objective,
                         int32_t l2_tiebreak, double tie_tol, int32_t *verdict, void *stream);

/* OperatorBank (controller.py:71-85) as device data; PAIRS slot order.     */
typedef struct {
  double weights[4], scores[4];
  int64_t segment_uses[4], lifetime_uses[4], iteration;
  double decay;
} amvm_bank;

/* select_operators (controller.py:88-90): *pair (device int32) =
 * rng.choice(4, p=weights/sum(weights)); advances rng.                      */
AMVM_API int amvm_select_operators(const amvm_bank *bank, amvm_pcg64 *rng, int32_t *pair,
                                   void *stream);

/* update_weights (controller.py:99-131): outcome 0 new best, 1 improved,
 * 2 accepted, 3 rejected; sigma1..3, weight_floor and n_segment from prm,
 * the decay from the bank (OperatorBank.decay).                            */
AMVM_API int amvm_update_weights(amvm_bank *bank, const amvm_params *prm, int32_t pair,
                                 int32_t outcome, void *stream);

/* impact_scores, operators.py:54-74: d (device double[n]).                 */
AMVM_API int amvm_impact_scores(const amvm_problem *prob, const amvm_params *prm,
                       const amvm_solution *sol, double *d, void *ws,
                       size_t ws_bytes, void *stream);

/* destroy operators, operators.py:34-39 (kind 0, random) and 77-105
 * (kind 1, worst-remove).  Writes the ascending `removed` (device int32[r])
 * and advances `rng`.                                                        */
AMVM_API int amvm_destroy(const amvm_problem *prob, const amvm_params *prm, int kind,
                 const amvm_solution *sol, amvm_pcg64 *rng, int32_t *removed,
                 void *ws, size_t ws_bytes, void *stream);

/* repair operators, operators.py:108-117 (kind 0, random; consumes rng) and
 * 120-138 (kind 1, greedy).  `removed` ascending, `saved_idx` the prior
 * levels (device int32[r] each).                                             */
AMVM_API int amvm_repair(const amvm_problem *prob, const amvm_params *prm, int kind,
                amvm_solution *sol, amvm_pcg64 *rng, const int32_t *removed,
                const int32_t *saved_idx, int32_t r, void *ws, size_t ws_bytes,
                void *stream);

/* compute_residual, core.py:183-197, as a device contraction for a batch:
 * residual[k] = A @ levels[k][idx[k]] - B[k], objective[k] = max|residual|.
 * Summed in OpenBLAS 0.3.30's SkylakeX dgemv_t order (4 FMA accumulators
 * per output over 2048-element blocks, ddot for m == 1): bitwise equal to
 * numpy's `A @ x` on such a host with single-threaded BLAS. */
AMVM_API int amvm_compute_residual(const amvm_problem *prob, amvm_solution *sol,
                          void *stream);

/* PTQ front end for one layer sharing X (= A, m calibration rows x n inputs;
 * builders.py:355-372 semantics with a shared X, controller.py:157-165):
 * for each weight row k of W (count x n, device), levels[k] = numpy
 * linspace(min w_k, max w_k, nlev) (range widened by 0.5 when it collapses),
 * idx[k] = nearest level of w_k (ties to the lower level), B[k] = X @ w_k in
 * numpy's BLAS order.  Follow with amvm_compute_residual for the start.    */
AMVM_API int amvm_ptq_prepare(int64_t m, int64_t n, int64_t count, int64_t nlev,
                              const double *At, const double *W, double *B,
                              double *levels, int32_t *idx, void *stream);

/* ---- exact oracle: replaces dmmv.oracle.brute_force (oracle.py:38-111) --
 * Exhaustive enumeration of all nlev^n assignments of ONE instance
 * (count == 1, n <= 64).  Result: the lexicographically smallest level-index
 * vector attaining the minimum max|A x - b| (the reference's first-strict-
 * improvement order), its objective, and its code (sum_j idx_j nlev^(n-1-j)).
 * order 0 evaluates t as `assignments @ A.T - b` (oracle.py:62-64: numpy's
 * dgemm, a sequential FMA chain over j), order 1 as the pruned DFS does
 * (oracle.py:95-111: -b + levels[d_0]*A[:,0] + ..., unfused).  The budget
 * check (BudgetExceededError) stays on the host.  best_idx (int32[n]),
 * best_t (double[1]), best_code (int64[1], may be NULL) are device pointers;
 * ws holds amvm_brute_force_workspace_bytes(prob) bytes.                  */
AMVM_API size_t amvm_brute_force_workspace_bytes(const amvm_problem *prob);
AMVM_API int amvm_brute_force(const amvm_problem *prob, int order, int32_t *best_idx,
                              double *best_t, int64_t *best_code, void *ws,
                              size_t ws_bytes, void *stream);

/* is_improving (localsearch.py:91-125) for nc swap candidates (i, j,
 * delta = x_i - x_j > 0) against the solution (residual, objective):
 * verdict[c] = 1 iff every row keeps (-t-s)/delta < a_j - a_i < (t-s)/delta.
 * The reference's row screen only skips rows that pass, so this is its
 * verdict with or without the screen.  Device pointers; count == 1.       */
AMVM_API int amvm_is_improving(const amvm_problem *prob, const double *residual, double objective,
                               int64_t nc, const int32_t *ci, const int32_t *cj,
                               const double *cd, int32_t *verdict, void *stream);

/* Batched candidate-move scoring: the one_opt candidate objective
 * (localsearch.py:76-78) for every column and candidate level at once,
 * for all `count` instances sharing A:
 *   out_t[(c*n + j)*nv + v] = max_k |s_ck + (lv_c[l] - lv_c[idx_cj]) * A[k,j]|
 * (level difference, then unfused DMUL and DADD; bitwise numpy's value).
 * mode 0: all levels, nv = nlev, l = v (l == idx gives the objective).
 * mode 1: adjacent levels (the reference's one_opt set), nv = 2,
 *         l = idx-1, idx+1; +inf where that level does not exist.
 * best[c] = flat index j*nv + v of the smallest (t, j, l) over candidates
 * that change the level (-1 if none), best_t[c] its t; best and best_t may
 * both be NULL (scores only: no grid-wide reduction).  `idx` is count x n,
 * `residual` count x m; device pointers; replaces the Python loop of
 * localsearch.py:70-80 for scoring (no move is applied).
 * Preconditions: 0 <= idx < nlev; A, residual and levels finite (the
 * abs-max drops NaN where numpy's propagates it).  Workspace (8-byte
 * aligned) of amvm_score_workspace_bytes(prob): per-CTA best slots and one
 * ticket counter per instance; it must be ZEROED before its first use (the
 * kernels leave the counters at zero, so no per-call memset is needed).
 * Adjacent mode with even m <= 8192 runs the TMA-bulk streaming kernel (one
 * CTA per SM, every column of A read from HBM once per instance); other
 * shapes and the all-levels mode run the warp-per-column kernel.          */
AMVM_API size_t amvm_score_workspace_bytes(const amvm_problem *prob);
AMVM_API int amvm_score_moves(const amvm_problem *prob, const int32_t *idx, const double *residual,
                              int mode, double *out_t, int64_t *best, double *best_t,
                              void *ws, size_t ws_bytes, void *stream);

/* exhaustive_swap_check (oracle.py:135-161): for every ordered pair with
 * x_i > x_j, out_t[i*n+j] = objective of the swapped assignment recomputed
 * from scratch in numpy's order (compute_residual, core.py:183-197) and
 * out_v[i*n+j] = the swap test's verdict; other entries are not written.
 * count == 1, n <= 4096 (the reference allows n <= 64).                    */
AMVM_API int amvm_swap_check(const amvm_problem *prob, const int32_t *idx, const double *residual,
                             double objective, double *out_t, int32_t *out_v, void *stream);

/* ---- device warm start: initial_solution without continuous_init --------
 * (controller.py:134-165): (A^T A + 1e-8 I) x = A^T b by Cholesky on the
 * device, idx[j] = nearest level of x_j (ties to the lower level), x = 0 if
 * the factorisation fails or x is not finite.  Agrees with the reference's
 * LAPACK solve to rounding (not bitwise; the host path stays the default).
 * count == 1.  idx (int32[n]), target (double[n], may be NULL) and flag
 * (int32[1]: 0 ok, 1 factorisation failed, 2 not finite; both fall back to
 * zeros as the reference does, with a warning on the host) are device
 * pointers; ws holds amvm_ls_start_workspace_bytes(m, n) bytes.           */
AMVM_API size_t amvm_ls_start_workspace_bytes(int64_t m, int64_t n);
AMVM_API int amvm_ls_start(const amvm_problem *prob, int32_t *idx, double *target,
                           int32_t *flag, void *ws, size_t ws_bytes, void *stream);

/* ---- tomography front end: replaces parallel_beam_matrix / _ray_weights --
 * (builders.py:186-239) as a device CSR build, bit-identical to the
 * reference's dense matrix restricted to its nonzeros (rows = (angle,
 * detector), columns = pixels ascending).  dirs (device double[4*n_angles])
 * = (cos, sin, -sin, cos) of each angle, computed by the host exactly as the
 * reference does (np.cos / np.sin).  amvm_projector_indptr writes
 * indptr[0..side*n_angles] (int64; workspace amvm_projector_workspace_bytes);
 * the caller allocates indptr[rows] entries and calls amvm_projector_fill. */
AMVM_API size_t amvm_projector_workspace_bytes(int64_t side, int64_t n_angles);
AMVM_API int amvm_projector_indptr(int64_t side, int64_t n_angles, const double *dirs,
                                   int64_t *indptr, void *ws, size_t ws_bytes, void *stream);
AMVM_API int amvm_projector_fill(int64_t side, int64_t n_angles, const double *dirs,
                                 const int64_t *indptr, int64_t *indices, double *values,
                                 void *stream);

/* out (S x m) = A @ X[:, s] (+ noise, S x m, may be NULL) for the CSR A
 * (m x n, columns ascending per row) and X (n x S): builders.py:322's
 * projections `A @ truth + noise`, in numpy's dense dgemv_t order (zeros
 * skipped exactly), bit-identical to the reference.                       */
AMVM_API int amvm_csr_gemv(int64_t m, int64_t n, int64_t S, const int64_t *indptr,
                           const int64_t *cols, const double *vals, const double *X,
                           const double *noise, double *out, void *stream);

/* SIRT warm start (builders.py:242-274) for S right-hand sides B (S x m)
 * sharing the CSR A: X (n x S) from 0, `iters` updates
 * x <- clip(x + C A^T R (b - A x), lo, hi) (clamp != 0).  Sums run in CSR /
 * CSC storage order (not numpy's dense BLAS order): agrees with the
 * reference to rounding.  Validation (A >= 0, a live row and column) is the
 * caller's; ws holds amvm_sirt_workspace_bytes(m, n, nnz, S) bytes.       */
AMVM_API size_t amvm_sirt_workspace_bytes(int64_t m, int64_t n, int64_t nnz, int64_t S);
AMVM_API int amvm_sirt(int64_t m, int64_t n, int64_t nnz, int64_t S, const int64_t *indptr,
                       const int64_t *cols, const double *vals, const double *B, int32_t iters,
                       double lo, double hi, int clamp, double *X, void *ws, size_t ws_bytes,
                       void *stream);

/* HOST helper: numpy default_rng(seed).bit_generator.state for each seed
 * (SeedSequence -> PCG64), so per-instance seeds need no Python loop.      */
AMVM_API int amvm_seed_pcg64(const uint64_t *seeds_host, int64_t count,
                             amvm_pcg64 *out_host);

/* Waits for `stream`, then returns the device-side status the last call on
 * this workspace left in its header (AMVM_OK, or e.g. AMVM_ERR_UNSUPPORTED
 * when a swap-candidate buffer overflowed).                                 */
AMVM_API int amvm_status(const void *ws, void *stream);

AMVM_API const char *amvm_strerror(int status);
AMVM_API int amvm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AMVM_H */
