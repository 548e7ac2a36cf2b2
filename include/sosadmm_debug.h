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
#ifdef __cplusplus
extern "C" {
#endif
/* C (M x N) = A (M x K) * op(B) with op(B) = B (K x N) or B^T (B is N x K): the DMMA GEMM. */
int sosadmm_debug_gemm(int M, int N, int K, const double* A, const double* B, int transB, double* C);
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
#ifdef __cplusplus
}
#endif
#endif
