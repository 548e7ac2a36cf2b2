/*
 * sosadmm_debug.h — stage-level entry points of the large-block PSD projection, for unit tests
 * only (tests/test_gpu_stages.py).  Each call allocates its own device memory, runs one stage of
 * the production kernels on a private stream, copies the result to the host buffers and frees.
 * All matrices are column-major FP64 host arrays.  Return 0 on success, a negative sosadmm_err
 * code otherwise.
 */
#ifndef SOSADMM_DEBUG_H
#define SOSADMM_DEBUG_H
#include <stdint.h>
#include "sosadmm.h"
#ifdef __cplusplus
extern "C" {
#endif
/* C (M x N) = A (M x K) * op(B) with op(B) = B (K x N) or B^T (B is N x K): the DMMA GEMM. */
int sosadmm_debug_gemm(int M, int N, int K, const double* A, const double* B, int transB, double* C);
/* C (M x N) = op(A) B with the warm-path DMMA GEMM (dgemm.cuh): op(A) = A (M x K, transA = 0) or A^T (A is
 * K x M, transA = 1); upper = 1 computes only the 64 x 64 tiles meeting the upper triangle (others stay 0);
 * variant: tile configuration (dgemm.cuh DG_VARIANTS; < 0 = the production default); reps > 0 also times
 * reps launches (*ms = mean per launch, CUDA events). */
int sosadmm_debug_dgemm(int M, int N, int K, const double* A, int transA, int upper, const double* B, double* C,
                        int variant, int reps, float* ms);
/* Warm-started projection (csrc/warm.cuh) of one symmetric block, 64 < N <= 1280: a0 through the cold path
 * (seeding the eigenvectors), then a1 through the warm refinement (cold fallback if it does not converge);
 * out0 / out1 = Pi_{S+}(a0), Pi_{S+}(a1) (full, column-major); stats = [status of the a1 projection (1 warm,
 * 2 cold), S evaluations, clusters of its last step, r, side, refinement updates]. */
int sosadmm_debug_warm_project(int N, const double* a0, const double* a1, double* out0, double* out1, int* stats);
/* Householder tridiagonalisation of the symmetric N x N matrix A in one thread-block cluster:
 * d (N), e (N-1), tau (N-1), V (N x N, reflector k in column k, rows k+1..N-1). */
int sosadmm_debug_tridiag(int N, const double* A, double* d, double* e, double* tau, double* V);
/* Divide-and-conquer eigensolver of the tridiagonal (d, e): ascending lam (N), eigenvectors Z (N x N). */
int sosadmm_debug_stedc(int N, const double* d, const double* e, double* lam, double* Z);
/* In-place inverse of the SPD t x t matrix K (setup-time cache of I + A_low^T P^{-1} A_low). */
int sosadmm_debug_spdinv(int t, double* K);
/* Timing probe of the tridiagonalisation: prof ((N-2) x 16 clock64 stamp slots of CTA 0 at the phase
 * boundaries of every Householder step), ms = CUDA-event time of one launch after a warm-up. */
int sosadmm_debug_tridiag_prof(int N, const double* A, long long* prof, float* ms);
/* Two-stage tridiagonalisation, stage 1 (dense -> band, sy2sb.cuh): band (N x 2BW, column c at
 * band[c 2BW + (r - c)], offsets 0..BW), V1 (N x N, reflector k in column k: zeros in rows k+1..k+BW-1,
 * 1 at row k+BW), tau1 (N); *bw = BW, *nref = number of reflector columns.  -2 if N is outside the
 * two-stage envelope. */
int sosadmm_debug_sy2sb(int N, const double* A, double* band, double* V1, double* tau1, int* bw, int* nref);
/* Stage 2 (band -> tridiagonal, sb2st.cuh) of a band in the layout above: d (N), e (N-1), the
 * reflectors V2 (N x KMAX x BW: sweep i, task k at (i KMAX + k) BW) and tau2 (N x KMAX); *kmax = KMAX. */
int sosadmm_debug_sb2st(int N, int BW, const double* band, double* d, double* e, double* V2, double* tau2,
                        int* kmax);
/* Z (N x r, column-major) <- Q2 Z with the stage-2 reflectors (bt2.cuh). */
int sosadmm_debug_bt2(int N, int BW, const double* V2, const double* tau2, int r, double* Z);
/* Both stages on A (the production path): d, e; *ms = CUDA-event time of one run after a warm-up. */
int sosadmm_debug_tridiag2(int N, const double* A, double* d, double* e, float* ms);
/* Two-stage timing (CUDA events, second of two runs): stage 1 and stage 2 milliseconds; optional clock64
 * stamps: prof1 (16 per panel: panel CTA 0..7, worker 0 8..15), prof2 (per task of sweep 0). */
int sosadmm_debug_ts_timing(int N, const double* A, float* ms1, float* ms2, long long* prof1, long long* prof2);
/* Large-block projection stages of A: tridiagonal (d, e), D&C eigenvalues lam, sel = [r, c0, side]. */
int sosadmm_debug_psd_stages(int N, const double* A, double* d, double* e, double* lam, int* sel);
/* One-GPU emulation of a block-sharded solve (the world >= 2 arithmetic of sosadmm_setup_sharded without
 * NCCL): each rank's context is set up with sosadmm_debug_setup_emulated (same arguments as
 * sosadmm_setup_sharded minus the id, world <= 8, all on one device); sosadmm_debug_group_iterate runs k
 * iterations of all ranks, summing the 2m + 3 partial sums with a device add in rank order where the
 * product path calls ncclAllReduce; sosadmm_debug_group_get_iterate assembles the owned columns.
 * ctx[r] must be the rank-r context.  Returns a sosadmm_err. */
int sosadmm_debug_setup_emulated(const sosadmm_problem* prob, const sosadmm_settings* settings, int32_t rank,
                                 int32_t world, const int32_t* block_owner, sosadmm_ctx** out);
int sosadmm_debug_group_iterate(sosadmm_ctx* const* ctx, int world, int64_t k);
/* Switch an emulated group (after setup, before iterating) to the peer-memory reduction of SURVEY §8(f)
 * f4: the partial sums are reduced inside k_gather_fin_peer from every rank's buffer (rank order), after
 * a per-round flag hand-off (k_peer_signal), instead of a separate allreduce.  Real ranks select it with
 * SOSADMM_ALLREDUCE=peer (CUDA IPC handles of the workspaces exchanged by one ncclAllGather at setup). */
int sosadmm_debug_group_link_peers(sosadmm_ctx* const* ctx, int world);
int sosadmm_debug_group_get_iterate(sosadmm_ctx* const* ctx, int world, double* xi, double* y, double* z, double* s,
                                    double* tau, double* kappa, int64_t* iter);
#ifdef __cplusplus
}
#endif
#endif
