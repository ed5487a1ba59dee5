/*
 * boxscreen_b200.h -- C ABI of the B200-native screened box-constrained
 * least-squares iteration (drop-in for the hot path of the reference
 * `boxscreen` package, arXiv 2202.07258).
 *
 * The reference has no FFI: its solver dispatch is the string if/elif at
 * /root/reference/pkg/src/boxscreen/driver.py:171-178 over the kinds listed at
 * solvers.py:17, operating on the Workspace state contract of
 * solvers.py:48-69.  Every entry point below replaces one reference symbol;
 * the symbol is cited beside it.  A Python binding of exactly these entry
 * points lives in paper_2202_07258_b200/_native.py (ctypes); INTEGRATION.md
 * shows how the reference's own driver would bind them.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers unless the name ends in _host.
 *    Matrices are column-major with a leading dimension `lda >= m`; the column
 *    stride `lda * sizeof(elem)` and the base pointer must be 16-byte aligned
 *    (the bulk-copy engine streams whole columns).
 *  - A is stored in fp64 (BX_F64) or fp32 (BX_F32, BASELINE config 4: half the
 *    streamed bytes, products accumulated in fp32 per CTA); y, bounds, t, the
 *    iterate and every other vector and scalar are fp64 (so fp32 storage never
 *    limits the precision of x -- DESIGN.md, "fp32").
 *  - Upper bounds may be +inf (NNLS / mixed); lower bounds must be finite.
 *  - Every function returns a bx_status.  Nonzero codes map 1:1 onto the
 *    reference exception classes of errors.py (listed per code).  The message
 *    of the last failure is available from bx_last_error().
 *  - One context = one solve = one CUDA stream; no global mutable state
 *    (solves are single-owner and reentrant).
 *  - Device memory is owned by the caller: bx_workspace_bytes() says how much
 *    scratch the context needs, the caller allocates it (PyTorch in the Python
 *    front end) and passes it to bx_ctx_create().  The context never writes A.
 */
#ifndef BOXSCREEN_B200_H
#define BOXSCREEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BX_OK = 0,
  BX_ERR_DIMENSION = 1,            /* errors.py:8   DimensionMismatch          */
  BX_ERR_ZERO_COLUMN = 2,          /* errors.py:69  ZeroColumn                 */
  BX_ERR_NO_INTERIOR = 3,          /* errors.py:29  NoInteriorPoint            */
  BX_ERR_STEP_TOO_LARGE = 4,       /* errors.py:51  StepSizeTooLarge           */
  BX_ERR_INTERNAL_CONSISTENCY = 5, /* errors.py:43  InternalConsistency        */
  BX_ERR_NEGATIVE_GAP = 6,         /* errors.py:39  NegativeGap                */
  BX_ERR_INVALID_ARGUMENT = 7,     /* ValueError (model.py:67-76, solvers.py:29-35) */
  BX_ERR_CUDA = 8,                 /* CUDA runtime failure (no reference analogue) */
  BX_ERR_UNSUPPORTED = 9,          /* shape outside the compiled kernel envelope   */
  BX_ERR_WORKSPACE = 10,           /* caller workspace too small / misaligned      */
  BX_ERR_NOT_INTERIOR = 11,        /* errors.py:25  NotInterior                */
  BX_ERR_SINGULAR = 12,            /* errors.py:56  SingularSubproblem (active set) */
  BX_ERR_PEER_TIMEOUT = 13         /* column-sharded fused exchange: a peer never published
                                      (bounded wait, BX_PEER_TIMEOUT_S, default 30 s)  */
} bx_status;

typedef enum { BX_F64 = 0, BX_F32 = 1 } bx_dtype;

/* solver kinds: solvers.py:17 ("pg", "cd", "active-set"); "apg" is the FISTA
 * extension of BASELINE.json configs 3 and 5 (not in the reference).
 * BX_ACTIVE_SET (bounded Lawson-Hanson, solvers.py:140-204) needs the extra
 * workspace of bx_ctx_set_active_set_workspace. */
typedef enum { BX_PG = 0, BX_CD = 1, BX_APG = 2, BX_ACTIVE_SET = 3 } bx_kind;

typedef struct bx_ctx bx_ctx;

/* SolverConfig (solvers.py:20-35) + the solve() flags (driver.py:131). */
typedef struct {
  int32_t kind;          /* bx_kind                                              */
  int32_t inner_passes;  /* >= 1                                                 */
  int64_t max_rounds;    /* <= 0: reference default (10**6; 10 n for the active
                            set, driver.py:144-150)                              */
  double gap_tol;        /* > 0                                                  */
  double step_size;      /* <= 0 or NaN: auto (power iteration, solvers.py:89)   */
  int32_t power_iters;   /* default 50                                           */
  int32_t screening;     /* 0/1                                                  */
  double alpha;          /* loss strong-concavity constant (model.py:40) = 1     */
  double slack_scale;    /* driver.py:219: 1e-12 for fp64                        */
  int32_t relative_gap;  /* 1: stop when gap <= gap_tol * max(1, P) (fp32 rule,
                            DESIGN.md); 0: absolute gap (reference rule)        */
  int32_t restart;       /* FISTA restart rule (BX_APG): 0 = adaptive (objective
                            increase OR the gradient test);
                            1 = objective increase only (BASELINE config 3's
                            stated rule, mirroring solvers.py:111-114)           */
} bx_solve_cfg;

/* TraceRecord (driver.py:28-38) plus the dual-point internals. */
typedef struct {
  int64_t round;
  double elapsed;
  double primal, dual, gap;
  int64_t preserved_count;
  int64_t newly_screened_lower, newly_screened_upper;
  double eps, radius, step;
  double certified_gap;  /* NaN when not evaluated this round                   */
  int64_t restarts;      /* FISTA restarts so far (cumulative)                  */
  double momentum;       /* FISTA t_k after the round                            */
} bx_trace_rec;

typedef struct {
  int64_t rounds;
  int32_t converged;
  double gap;            /* certified gap when converged, else last reduced gap */
  int64_t n_sat_lower, n_sat_upper;
  int64_t iterations;    /* primal passes (PG/APG steps or CD sweeps)          */
  double step;
  double sigma;          /* last power-iteration estimate                      */
  int64_t kernel_launches;
  int64_t restarts;
  int64_t spec_kept;     /* screening events whose speculative round-boundary step
                            stood                                  */
  int64_t spec_undone;   /* ... and events that undid it and took it again       */
} bx_solve_out;

/* Host callback producing the power-iteration start vector of length k:
 * the Python front end passes numpy default_rng(seed).standard_normal(k),
 * exactly solvers.py:75-76.  NULL selects an internal (non-numpy) generator. */
typedef void (*bx_start_vector_fn)(int64_t k, int64_t seed, double* out_host, void* user);

/* ---- context ------------------------------------------------------------ */

/* bytes of device scratch a context of this shape needs */
size_t bx_workspace_bytes(int64_t m, int64_t n, int32_t dtype);

/* Problem (model.py:47-99) + ScreeningState (screening.py:27-36) +
 * TranslationVector (duality.py:41-59).  `t` may be NULL: neg-ones
 * (duality.py:74-75).  Validates zero columns (ZeroColumn) and, when some
 * upper bound is infinite, strict interiority (NoInteriorPoint). */
int bx_ctx_create(bx_ctx** out, int64_t m, int64_t n, int32_t dtype,
                  const void* a, int64_t lda, const void* y,
                  const void* lower, const void* upper, const void* t,
                  void* workspace, size_t workspace_bytes, void* cuda_stream);
int bx_ctx_destroy(bx_ctx* ctx);
const char* bx_last_error(const bx_ctx* ctx);

/* ---- fine-grained entry points (Workspace contract, solvers.py:48-137) ---- */

/* column norms ||a_j|| (model.py:89-92), length n, fp64 */
int bx_col_norms(bx_ctx* ctx, void* out);
/* A't (duality.py:52), length n, fp64 */
int bx_att(bx_ctx* ctx, void* out);
/* spectral_norm_estimate on the preserved columns (solvers.py:72-86) */
int bx_power_iter(bx_ctx* ctx, int32_t iters, const double* v0_host, double* sigma_out);
/* reset the primal point to clip(0, l, u) and rebuild the workspace
 * (driver.py:149, solvers.py:54-65) */
int bx_reset(bx_ctx* ctx);
/* `passes` primal passes of the given kind on the preserved set:
 * pg_step (solvers.py:101-116), cd_sweep (:119-137), FISTA */
int bx_primal_passes(bx_ctx* ctx, int32_t kind, double eta, int32_t passes);
/* dual point + reduced gap + (optionally) the sphere test for the current
 * iterate: driver.py:183-201 and 213-221.  alpha: the loss's
 * strong-concavity constant (model.py:40, 1 for the quadratic loss).
 * out_scalars_host receives {primal, dual, gap, eps, radius, slack,
 * n_new_lower, n_new_upper}. */
int bx_dual_screen(bx_ctx* ctx, int32_t screening, double slack_scale, double alpha,
                   double* out_scalars_host);
/* apply_screening (screening.py:72-94) + Workspace.refresh (solvers.py:54-65)
 * of the last bx_dual_screen's sphere test: snaps screened x to bounds,
 * updates z, compacts A and the per-column state of the kind the last
 * bx_primal_passes ran (ballot/prefix-sum), updates the residual. */
int bx_compact(bx_ctx* ctx);
/* _certified_gap on the full problem (driver.py:112-117 ->
 * duality.py:159-209); out_host = {gap, primal, dual, eps} */
int bx_certified_gap(bx_ctx* ctx, double alpha, double* out_host);

/* Load a preserved set and a primal point into the workspace -- the state
 * the reference's spec-level updates take as (ScreeningState, PrimalPoint)
 * and rebuild a Workspace from (solvers.py:48-65, 207-227): `preserved`
 * (host, k ascending original indices), x_full (device, n) and the
 * saturated part z = A_S x_S (device, m).  Recomputes r = A_act x + z - y
 * and its objective; FISTA momentum restarts.  sat lists are not tracked. */
int bx_set_state(bx_ctx* ctx, const int64_t* preserved_host, int64_t k, const double* x_full,
                 const double* z);
/* one outer bounded-variable Lawson-Hanson iteration on the preserved set
 * (active_set_step, solvers.py:152-204; needs
 * bx_ctx_set_active_set_workspace): passive_in (device, k; NULL keeps the
 * context's mask) -> passive_out (device, k; may be NULL); *optimal = 1
 * when nothing violates the optimality conditions. */
int bx_active_set_step(bx_ctx* ctx, const uint8_t* passive_in, uint8_t* passive_out, int32_t* optimal);
/* residual r (m) and the restricted gradient A_act' r (k) at the current
 * iterate -- pg_update / cd_update's return values (solvers.py:207-227).
 * Device pointers. */
int bx_gradient(bx_ctx* ctx, double* resid, double* grad);
/* out (m) = A[:, cols] coef (+ z_add when not NULL): forward_product
 * (screening.py:97-104) and the z update of apply_screening (:84-88).
 * cols (device int32, k entries; NULL = all n columns, k = n). */
int bx_apply_a(bx_ctx* ctx, const int32_t* cols, int64_t k, const double* coef, const double* z_add,
               double* out);
/* out (n) = A' v over the full problem (eval_dual, dual_translate,
 * is_dual_feasible: duality.py:103-185).  Device pointers. */
int bx_apply_at(bx_ctx* ctx, const double* v, double* out);
/* dual point of the full problem at x_full (device, n): dual translation
 * with the context's t when some upper bound is infinite
 * (dual_point_nnlr, duality.py:187-209), dual scaling otherwise
 * (dual_point_bvlr, :159-168).  theta (m), a_t_theta (n) device (either may
 * be NULL); out_host = {gap (clamped), primal, dual, eps}. */
int bx_dual_point(bx_ctx* ctx, const double* x_full, double alpha, double* theta, double* a_t_theta,
                  double* out_host);
/* dual objective D(theta) (duality.py:103-124) given A'theta (device, n;
 * NULL: computed here); *d_host receives it. */
int bx_eval_dual(bx_ctx* ctx, const double* theta, const double* a_t_theta, double* d_host);
/* gap-safe sphere test on given inner products (screening.py:46-69):
 * a_t_theta (device, n), preserved (device int32, k), thresholds
 * (radius + slack) ||a_j||, strict comparisons; flags (device, k):
 * 0 keep, 1 lower, 2 upper. */
int bx_sphere_test(bx_ctx* ctx, const double* a_t_theta, const int32_t* preserved, int64_t k, double radius,
                   double slack, uint8_t* flags);
/* preserved count, and the preserved original indices (int32, device) */
int64_t bx_preserved_count(const bx_ctx* ctx);

/* ---- the Algorithm-1 loop (driver.py:131-256) ---------------------------- */
int bx_solve(bx_ctx* ctx, const bx_solve_cfg* cfg, bx_start_vector_fn start_fn,
             void* start_user, bx_trace_rec* trace_host, int64_t trace_cap,
             bx_solve_out* out_host);

/* final state (SolveResult, driver.py:41-50): x (n, fp64), theta
 * (m, fp64), sat_lower / sat_upper (int64, in screening order).  Any
 * pointer may be NULL.  Device pointers. */
int bx_get_state(bx_ctx* ctx, void* x, void* theta, int64_t* sat_lower, int64_t* sat_upper);
/* FISTA's previous iterate x_{k-1} as a full vector (device, n; screened
 * coordinates at their bounds) -- with the momentum scalar of the last trace
 * record it is the state a FISTA round resumes from (used to replay the
 * oracle from the device state mid-solve, tests/test_gpu_headline.py). */
int bx_get_prev_iterate(bx_ctx* ctx, double* x_prev);

/* ---- active-set solver (solvers.py:140-204) ------------------------------ */
/* bytes of the active-set scratch: the passive Cholesky factor R
 * (min(m, n)^2 fp64, updated by column appends and Givens deletions instead
 * of the reference's per-iteration refactorisation) plus O(m + n) vectors */
size_t bx_active_set_workspace_bytes(int64_t m, int64_t n);
/* hand that scratch to a context (required before bx_solve with
 * BX_ACTIVE_SET; the caller owns the memory, as with bx_ctx_create's) */
int bx_ctx_set_active_set_workspace(bx_ctx* ctx, void* workspace, size_t workspace_bytes);

/* ---- multi-GPU column sharding ---------------------------- */
/* 128-byte NCCL unique id, produced on rank 0 and broadcast by the caller */
int bx_nccl_unique_id(unsigned char* id_out_host);
/* attach a communicator: this context holds global columns
 * [col_offset, col_offset + n) of an n_global-column problem */
int bx_ctx_set_comm(bx_ctx* ctx, const unsigned char* id_host, int32_t rank,
                    int32_t nranks, int64_t col_offset, int64_t n_global);

/* Persistent communicator for repeated sharded solves: the NCCL
 * communicator and the fused exchange's IPC-mapped buffers (sized for up to
 * m rows) are set up once per process group and borrowed by every context
 * (bx_ctx_use_comm), instead of bx_ctx_set_comm + bx_peer_* per solve.
 * Setup is collective: every rank calls bx_comm_create with the same unique
 * id, bx_comm_peer_alloc, exchanges the 64-byte handles, bx_comm_peer_open
 * (or, when any rank failed, bx_comm_peer_disable on all ranks).  The
 * communicator must outlive the contexts that use it. */
typedef struct bx_comm bx_comm;
int bx_comm_create(bx_comm** out, const unsigned char* id_host, int32_t rank, int32_t nranks);
int bx_comm_destroy(bx_comm* comm);
int bx_comm_peer_alloc(bx_comm* comm, int64_t m, unsigned char* ipc_handle_out);
int bx_comm_peer_open(bx_comm* comm, const unsigned char* ipc_handles);
int bx_comm_peer_disable(bx_comm* comm);
int bx_ctx_use_comm(bx_ctx* ctx, bx_comm* comm, int64_t col_offset, int64_t n_global);

/* fused reduce + peer exchange for the per-step reduction of the sharded
 * PG / FISTA pass (replaces its NCCL allreduces with ONE kernel that stores
 * each row block straight into every peer's buffer over NVLink and sums the
 * peers' blocks in rank order; csrc/bx_exchange.cuh).  After attaching a
 * communicator: bx_peer_alloc allocates this rank's receive buffer and
 * exports its 64-byte CUDA IPC handle (handle_out may be NULL for the
 * in-process group); bx_peer_open maps every rank's buffer from the
 * nranks x 64 gathered handles (NULL: in-process group).  At most 8 ranks. */
int bx_peer_alloc(bx_ctx* ctx, unsigned char* ipc_handle_out);
int bx_peer_open(bx_ctx* ctx, const unsigned char* ipc_handles);
/* Fall back to the NCCL schedule for the per-step reduction (unmaps the
 * peers): every rank calls it when any rank failed to map its peers, so all
 * ranks run the same schedule. */
int bx_peer_disable(bx_ctx* ctx);

/* in-process rank group: ranks are threads of one process sharing a GPU or
 * several; the allreduce is host-barrier + device sum (test transport of the
 * column-sharded path; production uses NCCL through bx_ctx_set_comm) */
typedef struct bx_group bx_group;
int bx_group_create(bx_group** out, int32_t nranks);
int bx_group_destroy(bx_group* group);
int bx_ctx_set_group(bx_ctx* ctx, bx_group* group, int32_t rank, int64_t col_offset, int64_t n_global);

/* ---- live per-kernel timing (bench.py roofline) ---------------------------- */
/* CUDA events around every kernel launch on the context stream; accumulated
 * per slot with the ALGORITHMIC bytes of each launch. */
enum {
  BX_PROF_PASS_DOT = 0,    /* screening pass: g = A'r + epsilon partial     */
  BX_PROF_PASS_PG_G = 1,   /* PG step from the stored gradient              */
  BX_PROF_PASS_PG = 2,     /* fused PG step (dot + update + A x)            */
  BX_PROF_PASS_APG = 3,    /* fused FISTA step                              */
  BX_PROF_PASS_POWER = 4,  /* power iteration                               */
  BX_PROF_PASS_AX = 5,     /* A x (refresh / certified gap / z update)      */
  BX_PROF_REDUCE = 6,
  BX_PROF_DUAL = 7,
  BX_PROF_SPHERE = 8,
  BX_PROF_GATHER = 9,
  BX_PROF_CD = 10,
  BX_PROF_ACTIVE = 11,     /* active-set selection / factor update / solve  */
  BX_PROF_SMALL = 12,      /* cooperative SM-resident round kernel (small problems) */
  BX_PROF_SLOTS = 13
};
typedef struct {
  int64_t launches;
  double ms;
  double bytes;
} bx_prof_entry;
int bx_set_profiling(bx_ctx* ctx, int32_t on);
int bx_get_profile(bx_ctx* ctx, bx_prof_entry* out_host, int32_t n);

/* ---- batched many-RHS APG (BASELINE config 5) ----------------------------- */
/* K independent NNLS problems sharing one dictionary A (m <= 208), FISTA with
 * per-problem gap-safe screening, both products on fp64 tensor cores (DMMA);
 * semantics in oracle/batched_oracle.py.  Not in the reference (it solves one
 * right-hand side per solve() call, driver.py:131). */
typedef struct bx_batch bx_batch;
typedef struct {
  int64_t rounds, converged, iterations, kernel_launches;
  double max_gap;
  /* tile-rounds (64 right-hand sides each) that ran the per-coordinate sphere
   * test; the others were cleared by the per-problem bound (no coordinate
   * could be screened); tiles = K / 64 */
  int64_t sphere_sweeps, tiles;
  /* summed duration of the round kernels (CUDA events on the solve's stream) */
  double round_kernel_ms;
} bx_batched_out;
size_t bx_batched_workspace_bytes(int64_t m, int64_t n, int64_t k_rhs);
/* A: device, column-major (lda even); Y: device m x K column-major (ldy) */
int bx_batched_create(bx_batch** out, int64_t m, int64_t n, int64_t k_rhs, const double* a, int64_t lda,
                      const double* y, int64_t ldy, void* workspace, size_t workspace_bytes,
                      void* cuda_stream);
/* `rounds` rounds of `passes` FISTA steps + dual point + sphere test; stops
 * early when every problem's gap < gap_tol.  trace_host (optional, 4 doubles
 * per round): {converged, max gap, mean gap, mean preserved}. */
int bx_batched_run(bx_batch* b, double eta, int32_t passes, int32_t rounds, int32_t screening, double gap_tol,
                   double* trace_host, int64_t trace_cap, bx_batched_out* out_host);
/* Convergence is checked (and the host synchronised) every rounds_per_check
 * rounds (default 1, at most 16).  With more than one, a launch runs that many
 * rounds and the rounds of different tiles overlap across it: SMs that finish
 * a round's last wave of tiles start the next round's first tiles (a tile's
 * round r + 1 depends only on its own round r).  The per-round trace is still
 * complete; a batch that converges at one of its inner rounds still runs to
 * the batch's last round. */
int bx_batched_set_check_every(bx_batch* b, int32_t rounds_per_check);
/* bx_batched_run with the result delivered to the host: x_host (pinned,
 * n x K column-major, column stride ldx_host >= n) holds X when the call
 * returns.  In the last round of the budget the tiles run wave by wave and
 * each wave's columns of X are copied out while the next waves compute. */
int bx_batched_run_to_host(bx_batch* b, double eta, int32_t passes, int32_t rounds, int32_t screening,
                           double gap_tol, double* trace_host, int64_t trace_cap, bx_batched_out* out_host,
                           double* x_host, int64_t ldx_host);
/* x: n x K (device, column stride ldx_out); stats: 5 x K (device) per-problem
 * {primal, dual, gap, eps, preserved} of the last round */
int bx_batched_get(bx_batch* b, double* x, int64_t ldx_out, double* stats);
const char* bx_batched_last_error(const bx_batch* b);
int bx_batched_destroy(bx_batch* b);

#ifdef __cplusplus
}
#endif
#endif /* BOXSCREEN_B200_H */
