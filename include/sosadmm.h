/*
 * sosadmm.h — C ABI of the B200-native HSDE-ADMM hot path for SOS-derived SDPs
 * (arXiv 1708.04174, Zheng, Fantuzzi, Papachristodoulou: "Fast ADMM for sum-of-squares programs
 * using partial orthogonality").  Citations "P:n" are lines of the paper's LaTeX source
 * (PAPER.md); "S:n" are lines of SPEC.md; labels are the paper's equation labels.
 *
 * Problem (`eq:generalSDP`):  min c^T xi  s.t.  A xi = b,  xi in K = R^t x S+(N_1) x ...
 * Dual:  max b^T y  s.t.  A^T y + z = c,  z in K*.
 * The library runs the ADMM of `eq:ADMMSteps` on the homogeneous self-dual embedding
 * with u = (xi, y, tau), v = (z, s, kappa):
 *     u_hat = (I + Q)^{-1}(u + v);   u = P_C(u_hat - v);   v = v - u_hat + u.
 * The linear step uses partial orthogonality (Proposition 1; Prop. 3):
 * every PSD column with at most one nonzero (and c_j = 0) is "orthogonal", the rest (the t free
 * columns and any other PSD column) form A_low, and (I + A A^T)^{-1} = P^{-1} - P^{-1} A_low
 * (I + A_low^T P^{-1} A_low)^{-1} A_low^T P^{-1} with P = I + A_orth A_orth^T diagonal,
 * plus the rank-one HSDE correction with cached M^{-1} zeta (`E:MatrixInverseResult`).
 *
 * Layouts (all host pointers unless stated):
 *  - column order of xi, z, c and of A: t free columns, then one svec block per PSD cone;
 *  - svec = LAPACK 'U' packed column-major: position p(i,j) = i + j(j+1)/2 for i <= j, with the
 *    off-diagonal entries scaled by sqrt(2) (an isometry of S^N; reading C1);
 *  - A is CSC (m x n, n = t + sum N_b(N_b+1)/2), 0-based, int64 column pointers, int32 rows;
 *  - FP64 everywhere; indices int32/int64 as declared.
 * Ownership: inputs are borrowed for the duration of the call and copied.  The context owns its
 *  device state, which lives in the caller-provided device workspace (e.g. a torch tensor); the
 *  library allocates no device memory of its own (settings.workspace is required: E_ARG if NULL).
 *  Outputs are written to caller buffers.  A context is not thread-safe; distinct contexts are independent.
 * Errors: every call returns sosadmm_err (0 = OK).  The first error is latched in the context and
 *  returned by every later call; sosadmm_last_error_message() gives a human-readable detail.
 * Initialisation (reading C7): u0 = (0, 0, 1), v0 = (0, 0, 0).  No scaling, no
 *  relaxation (reading C8).  Residuals and termination: DESIGN.md reading C9.
 */
#ifndef SOSADMM_H
#define SOSADMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SOSADMM_OK = 0,
  SOSADMM_E_ARG = -1,       /* malformed input (sizes, pointers, CSC structure) */
  SOSADMM_E_STRUCT = -2,    /* unsupported structure (low-rank width > 16384, a block > SOSADMM_MAX_BLOCK) */
  SOSADMM_E_FACTOR = -3,    /* I + A_low^T P^{-1} A_low not numerically SPD (impossible in exact arithmetic) */
  SOSADMM_E_CUDA = -4,      /* CUDA runtime error (message has the detail) */
  SOSADMM_E_NCCL = -5,      /* NCCL unavailable or failed (sharded mode) */
  SOSADMM_E_NONFINITE = -6, /* non-finite iterate; message names the iteration */
  SOSADMM_E_OOM = -7        /* workspace too small / allocation failed */
} sosadmm_err;

typedef enum {
  SOSADMM_RUNNING = 0,
  SOSADMM_OPTIMAL = 1,            /* max(res_pri, res_dual, res_gap) <= tol */
  SOSADMM_PRIMAL_INFEASIBLE = 2,  /* b^T y > 0 and ||A^T y + z|| / b^T y <= tol (reading C9) */
  SOSADMM_DUAL_INFEASIBLE = 3,    /* c^T xi < 0 and ||A xi|| / (-c^T xi) <= tol (reading C9) */
  SOSADMM_MAX_ITERS = 4,
  SOSADMM_INCONCLUSIVE = 5
} sosadmm_status;

/* Largest supported PSD block dimension (the cluster tridiagonalisation and the divide-and-conquer
 * merge keep per-block state in shared memory); larger blocks make setup fail with E_STRUCT. */
#define SOSADMM_MAX_BLOCK 1280

/* Conic data of `eq:generalSDP`.  psd_dim[b] = N_b; block b owns N_b(N_b+1)/2 svec columns. */
typedef struct {
  int64_t m;
  int64_t n_free;
  int32_t n_psd;
  const int32_t* psd_dim;
  const int64_t* A_colptr; /* n + 1 */
  const int32_t* A_rowidx; /* nnz */
  const double* A_val;     /* nnz */
  const double* b;         /* m */
  const double* c;         /* n */
} sosadmm_problem;

typedef struct {
  double tol;            /* termination tolerance on the C9 residuals (default 1e-4) */
  int64_t max_iters;     /* status MAX_ITERS once this many iterations ran */
  int32_t check_every;   /* residual check stride (1 = every iteration; the only supported value) */
  int32_t device;        /* CUDA device ordinal */
  void* stream;          /* cudaStream_t to launch on (NULL = the library's own stream) */
  void* workspace;       /* device memory of >= sosadmm_workspace_size() bytes (required) */
  size_t workspace_bytes;
} sosadmm_settings;

typedef struct {
  int64_t iter;       /* iterations completed (k of u^k) */
  int32_t status;     /* sosadmm_status */
  double res_pri;     /* ||A xi/tau - b|| / (1 + ||b||) at u^k (inf if tau = 0) */
  double res_dual;    /* ||A^T y/tau + z/tau - c|| / (1 + ||c||) */
  double res_gap;     /* |c^T xi/tau - b^T y/tau| / (1 + |c^T xi/tau| + |b^T y/tau|) */
  double pobj;        /* c^T xi / tau */
  double dobj;        /* b^T y / tau */
  double tau, kappa;
  double pinf, dinf;  /* certificate ratios of reading C9 (inf when the sign test fails) */
} sosadmm_info;

typedef struct sosadmm_ctx sosadmm_ctx;

/* Structural analysis only (no factorisation): device bytes the context needs. 0 on bad input. */
size_t sosadmm_workspace_size(const sosadmm_problem* prob);

/* Setup ("can be cached"): classify columns, build the
 * alpha-map, D and P = I + D, A_low in CSR/CSC, K = I + A_low^T P^{-1} A_low and its inverse,
 * h = M^{-1} zeta (zeta = (c, -b)) and 1 + zeta^T h; copy the data to the device; set u0, v0. */
sosadmm_err sosadmm_setup(const sosadmm_problem* prob, const sosadmm_settings* settings, sosadmm_ctx** out);

/* ---- Multi-GPU block sharding (north_star: "partition the blocks across the GPUs of
 * one 8xB200 box and NCCL-allreduce the length-m A2 x partial sums over NVLink each iteration").
 * Rank r owns the PSD blocks with block_owner[b] == r (the free columns are accounted by rank 0);
 * every iteration each rank forms the partial gather sums over its columns and one
 * ncclAllReduce(sum, FP64, 2m + 3) completes them; the Woodbury / HSDE scalar work is replicated and
 * bit-identical on all ranks, the scatter / PSD projection / dual update touch owned blocks only.
 * NCCL is resolved at run time from the process's libnccl.so.2 (E_NCCL if it cannot be loaded).
 * sosadmm_nccl_unique_id writes SOSADMM_NCCL_ID_BYTES bytes (call on rank 0, broadcast with any
 * transport, e.g. torch.distributed); every rank then calls sosadmm_setup_sharded with the same
 * problem, settings.device = its GPU, the same id and the same block_owner (n_psd entries in
 * [0, world)).  sosadmm_iterate / sosadmm_get_info / sosadmm_get_iterate are collectives on a
 * sharded context (every rank must call them in the same order); sosadmm_get_iterate returns the
 * full iterate on every rank.  The unit entry points return E_ARG on a sharded context.
 * SOSADMM_ALLREDUCE=peer (environment, read at setup) replaces the ncclAllReduce by the reduction over
 * peer memory fused into the gather's consumer: CUDA IPC handles of the workspaces are
 * exchanged with one ncclAllGather at setup, each iteration every rank publishes its partial sums with a
 * release store into the peers' flag slots and k_gather_fin_peer adds all ranks' partials in rank
 * order (requires peer access between the GPUs and a workspace allocated with cudaMalloc). */
#define SOSADMM_NCCL_ID_BYTES 128
sosadmm_err sosadmm_nccl_unique_id(void* id);
sosadmm_err sosadmm_setup_sharded(const sosadmm_problem* prob, const sosadmm_settings* settings, const void* nccl_id,
                                  int32_t rank, int32_t world, const int32_t* block_owner, sosadmm_ctx** out);

/* Run up to k ADMM iterations (`eq:ADMMSteps`) on the device, stopping early when the C9 rule
 * fires or max_iters is reached; every iteration's residuals are checked.  The iterations are
 * CUDA-graph replays enqueued in chunks; once a finished chunk shows the device's latched stop, no
 * further replays are enqueued (replays after the stop would be no-ops), so a large k costs little
 * past the stop.  Asynchronous work is completed before return; *out (may be NULL) receives the
 * state after the last iteration. */
sosadmm_err sosadmm_iterate(sosadmm_ctx* ctx, int64_t k, sosadmm_info* out);

/* Enqueue k ADMM iterations (k CUDA-graph replays) on the context's stream and return without
 * waiting (independent instances, each set up with its own stream, run concurrently
 * on one GPU — e.g. one 16-CTA tridiagonalisation cluster per instance).  The device-side
 * termination rule still applies to every iteration.  sosadmm_get_info (or sosadmm_iterate)
 * completes the work and reports; launch errors are returned here, asynchronous faults there.
 * On a sharded context it is a collective like sosadmm_iterate. */
sosadmm_err sosadmm_iterate_async(sosadmm_ctx* ctx, int64_t k);

/* Scheduling hint for SURVEY §8(f) f1 (no arithmetic: the iterates of `eq:ADMMSteps` are the same bit for
 * bit either way).  shared != 0: the context shares its GPU with other concurrently iterating instances, so
 * its iteration graph keeps the warm-start predictor of the large-block PSD projection in line instead of
 * forking it beside the affine projection (measured: the fork gains 2 % for a lone instance and costs
 * 8-18 % of a batch's aggregate rate).  Default 0.  Waits for the context's enqueued work and drops an
 * already built graph (rebuilt by the next iterate call).  E_ARG on a NULL context. */
sosadmm_err sosadmm_set_shared_gpu(sosadmm_ctx* ctx, int shared);

/* Same iterations launched without the CUDA graph, with CUDA events (on the library's stream)
 * around each phase; adds the phase durations (ms) to ms_phase[0..SOSADMM_NPHASE-1] = {affine
 * gather..row update, scatter, small-block Jacobi projections, large-block tridiagonalisation,
 * divide-and-conquer tridiagonal eigensolver, back-transform + reconstruction, pack / dual
 * update}.  Used by bench.py for the per-kernel-class rooflines. */
#define SOSADMM_NPHASE 7
sosadmm_err sosadmm_iterate_profiled(sosadmm_ctx* ctx, int64_t k, sosadmm_info* out, double* ms_phase);

/* Current info without iterating (residuals of u^k are computed on demand). */
sosadmm_err sosadmm_get_info(sosadmm_ctx* ctx, sosadmm_info* out);

/* Copy the unscaled HSDE iterates u = (xi, y, tau), v = (z, s, kappa) of `eq:ADMMSteps` (
 * u, v in the embedding of P:362-389) to host buffers of n, m, n, m doubles; tau, kappa, iter to
 * scalars.  The scaled solution is xi/tau, y/tau.  Any output pointer may be NULL. */
sosadmm_err sosadmm_get_iterate(sosadmm_ctx* ctx, double* xi, double* y, double* z, double* s,
                                double* tau, double* kappa, int64_t* iter);

/* Overwrite the iterates u = (xi, y, tau), v = (z, s, kappa) of the HSDE with host data
 * (n, m, n, m doubles; resume, warm start and the fixed-point tests of the planted KKT point).
 * s may be NULL (= 0, its value for every k >= 1).  Resets the termination status and residuals. */
sosadmm_err sosadmm_set_iterate(sosadmm_ctx* ctx, const double* xi, const double* y, const double* z,
                                const double* s, double tau, double kappa, int64_t iter);

/* Partial-orthogonality structure found by setup (Proposition 1):
 * row_of[j] for every column j: the row of its single nonzero if the column is orthogonal
 * (-1 for an empty orthogonal column), -2 if it belongs to A_low;  D[alpha] = sum over orthogonal
 * columns of (A_alpha,j / w_j)^2 * w_j^2 with w_j the svec weight, i.e. the exact integer count
 * n_alpha for indicator data;  *t_low = number of A_low columns (t').  Buffers: n, m. */
sosadmm_err sosadmm_get_structure(sosadmm_ctx* ctx, int32_t* row_of, double* D, int64_t* t_low);

/* Unit entry points of the two kernels classes (tests and bench), host buffers:
 * affine projection u_hat = (I + Q)^{-1} w  (`eq:HsdeStep1`, P:396 via P:426-481). */
sosadmm_err sosadmm_project_affine(sosadmm_ctx* ctx, const double* w1, const double* w2, double w3,
                                   double* u1, double* u2, double* u3);
/* PSD projection of one block in svec coordinates (`eq:HsdeStep2`). */
sosadmm_err sosadmm_project_psd(sosadmm_ctx* ctx, int32_t block, const double* a_svec, double* out_svec);

/* Algorithmic FP64 work of the last large-block PSD projections (measurement), 6 doubles per
 * large block (N > 64) in setup order: [tridiagonalisation 4/3 N^3, divide-and-conquer merge GEMM flops
 * sum 2 n k K from the device-side deflated sizes, back-transform 2 N^2 r, reconstruction N (N + 32) r, r,
 * number of fully deflated merges] with r = the selected spectral side's rank.  In: *nblocks = capacity of
 * `work` in blocks (work may be NULL to query); out: *nblocks = number of large blocks. */
sosadmm_err sosadmm_psd_work(sosadmm_ctx* ctx, double* work, int32_t* nblocks);

/* Residual history (measurement; reading C9 residuals of u^k as the in-graph check computed them during
 * iteration k + 1): up to *count entries of 5 doubles [k, pres, dres, gap, pobj], newest first, consecutive
 * k; the ring holds the last 1,024 iterations.  In: *count = capacity in entries; out: entries written. */
sosadmm_err sosadmm_residual_history(sosadmm_ctx* ctx, double* out, int32_t* count);

/* Warm-started large-block projection counters (csrc/warm.cuh), 10 int64 per large block in
 * setup order: [iterations projected by the warm refinement, iterations projected by the cold path
 * (tridiagonalisation + D&C + back-transform), total refinement updates of the warm iterations and of the
 * failed attempts, failed attempts, warm mode on (0/1), r (rank of the last projection's smaller spectral
 * side), N, S evaluations of the last iteration, cold iterations that re-seeded the eigenvectors, reason of
 * the last failed attempt (1 no convergence within the step budget, 2 stalled coupling, 3 cluster above the
 * exact-solve cap, 4 non-finite)].  Same capacity protocol as sosadmm_psd_work. */
sosadmm_err sosadmm_warm_stats(sosadmm_ctx* ctx, int64_t* stats, int32_t* nblocks);

/* Number of kernel launches one iteration issues (for the bench's gpu_launches claim). */
int64_t sosadmm_launches_per_iter(const sosadmm_ctx* ctx);

/* Release the context (its device state lives in the caller's workspace, which the caller frees;
 * the context's streams, events, CUDA graph and NCCL communicator are destroyed here).  NULL is a
 * no-op.  Ownership rule of SURVEY §8(b) (S:227 cache immutable until destroyed). */
void sosadmm_destroy(sosadmm_ctx* ctx);
const char* sosadmm_strerror(sosadmm_err e);
const char* sosadmm_last_error_message(const sosadmm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SOSADMM_H */
