// PSD-cone projection of small Gram blocks (N <= 64): Pi(A) = V diag(max(lambda, 0)) V^T
// (PAPER.md P:397-398 `eq:HsdeStep2`, cone S_+ of P:281), eigendecomposition by the cyclic
// two-sided Jacobi method with the parallel (round-robin tournament) ordering: N/2 disjoint
// rotations per round, N-1 rounds per sweep, sweeps until no rotation passes the threshold.
// One CTA per block; A and V live in shared memory; the result overwrites the block matrix.
#pragma once
#include "common.cuh"

constexpr int JAC_NT = 256;
constexpr int JAC_MAXN = 64;

struct JacobiArgs {
  double* mats;
  const long long* blk_mat;
  const int* blk_N;
  const int* small_blk;  // list of block ids handled by this launch
  const DevState* st;
  const IterScal* is;
  int check_state;       // 1 = honour the done/proceed flags
};

// Round r of the tournament for Np players (Np even): slot k -> pair (p, q).
__device__ __forceinline__ void rr_pair(int r, int k, int Np, int& p, int& q) {
  const int M = Np - 1;
  if (k == 0) {
    p = M;
    q = r % M;
  } else {
    p = (r + k) % M;
    q = (r - k + M) % M;
  }
}

__global__ void __launch_bounds__(JAC_NT) k_psd_jacobi(JacobiArgs a) {
  if (a.check_state && (a.st->done || !a.is->proceed)) return;
  const int b = a.small_blk[blockIdx.x];
  const int N = a.blk_N[b];
  const int Np = (N + 1) & ~1;  // even; a padded zero row/column never rotates
  double* G = a.mats + a.blk_mat[b];
  extern __shared__ double smem[];
  double* A = smem;               // Np x Np, column-major
  double* V = A + Np * Np;        // Np x Np
  double* alpha = V + Np * Np;    // Np
  double* beta = alpha + Np;      // Np
  double* tval = beta + Np;       // Np/2
  int* partner = (int*)(tval + Np / 2);
  __shared__ int nrot;
  __shared__ double normF;
  const int tid = threadIdx.x;

  for (int e = tid; e < Np * Np; e += JAC_NT) {
    const int i = e % Np, j = e / Np;
    A[e] = (i < N && j < N) ? G[(size_t)j * N + i] : 0.0;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    double s = 0.0;
    for (int e = tid; e < Np * Np; e += 32) s = fma(A[e], A[e], s);
    s = warp_sum(s);
    if (tid == 0) normF = sqrt(s);
  }
  __syncthreads();
  constexpr double EPS = 2.220446049250313e-16;
  // Absolute floor N EPS ||A||_F: leaving all couplings below it changes the projection by at most
  // ~N^2 EPS ||A||_F (Pi is 1-Lipschitz), far inside the 1e-9 parity bar, while rounding re-creates
  // couplings of ~EPS ||A|| every round — without the floor the relative test below (high relative
  // accuracy next to (near-)zero eigenvalues) never reports a quiet sweep and all 60 sweeps run.
  const double tiny = fmax((double)N * EPS * normF, 1e-300);
  constexpr int PER = JAC_MAXN * JAC_MAXN / JAC_NT;
  double nv[PER];
  int ei[PER], ej[PER];  // (row, column) of this thread's element slots, fixed for the whole solve
#pragma unroll
  for (int cnt = 0; cnt < PER; ++cnt) {
    const int e = tid + cnt * JAC_NT;
    ei[cnt] = e % Np;
    ej[cnt] = e / Np;
  }

  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) nrot = 0;
    __syncthreads();
    for (int r = 0; r < Np - 1; ++r) {
      // 1. rotation parameters of the Np/2 disjoint pairs (GvL sym.schur2)
      if (tid < Np / 2) {
        int p, q;
        rr_pair(r, tid, Np, p, q);
        const double apq = A[p + q * Np], app = A[p + p * Np], aqq = A[q + q * Np];
        double c = 1.0, s = 0.0, t = 0.0;
        if (fabs(apq) > EPS * sqrt(fabs(app) * fabs(aqq)) && fabs(apq) > tiny) {
          const double th = (aqq - app) / (2.0 * apq);
          t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(fma(th, th, 1.0)));
          c = 1.0 / sqrt(fma(t, t, 1.0));
          s = t * c;
          atomicAdd(&nrot, 1);
        }
        alpha[p] = c; beta[p] = -s; partner[p] = q;
        alpha[q] = c; beta[q] = s;  partner[q] = p;
        tval[tid] = t;
      }
      __syncthreads();
      // 2. A <- J^T A J elementwise from the 2x2 coupling (all reads before any write)
      // (compile-time trip counts keep nv / vv in registers)
      double vv[JAC_MAXN * JAC_MAXN / JAC_NT];
#pragma unroll
      for (int cnt = 0; cnt < JAC_MAXN * JAC_MAXN / JAC_NT; ++cnt) {
        const int e = tid + cnt * JAC_NT;
        if (e < Np * Np) {
          const int i = ei[cnt], j = ej[cnt];
          const int ip = partner[i], jp = partner[j];
          const double ai = alpha[i], bi = beta[i], aj = alpha[j], bj = beta[j];
          nv[cnt] = ai * (aj * A[i + j * Np] + bj * A[i + jp * Np]) +
                    bi * (aj * A[ip + j * Np] + bj * A[ip + jp * Np]);
          // V <- V J (column j mixes with its partner)
          vv[cnt] = aj * V[i + j * Np] + bj * V[i + jp * Np];
        }
      }
      __syncthreads();
#pragma unroll
      for (int cnt = 0; cnt < JAC_MAXN * JAC_MAXN / JAC_NT; ++cnt) {
        const int e = tid + cnt * JAC_NT;
        if (e < Np * Np) {
          A[e] = nv[cnt];
          V[e] = vv[cnt];
        }
      }
      __syncthreads();
      // exact annihilation and the standard diagonal update
      if (tid < Np / 2) {
        const double t = tval[tid];
        if (t != 0.0) {
          int p, q;
          rr_pair(r, tid, Np, p, q);
          // recompute from the pre-rotation values is not possible any more; use the rotated
          // diagonal (already c^2 a_pp - 2cs a_pq + s^2 a_qq) and zero the coupling exactly
          A[p + q * Np] = 0.0;
          A[q + p * Np] = 0.0;
        }
      }
      __syncthreads();
    }
    if (nrot == 0) {
#ifdef SOSADMM_JACOBI_DEBUG
      if (tid == 0) printf("jacobi block %d N %d sweeps %d\n", b, N, sweep + 1);
#endif
      break;
    }
    __syncthreads();
  }
  // Pi(A) = V diag(max(lambda, 0)) V^T, lambda_k = A[k, k]
  for (int k = tid; k < Np; k += JAC_NT) alpha[k] = fmax(A[k + k * Np], 0.0);
  __syncthreads();
  for (int e = tid; e < N * N; e += JAC_NT) {
    const int i = e % N, j = e / N;
    if (i < j) continue;  // lower triangle (row i >= column j) is what k_pack reads
    double acc = 0.0;
    for (int k = 0; k < Np; ++k) acc = fma(V[i + k * Np] * alpha[k], V[j + k * Np], acc);
    G[(size_t)j * N + i] = acc;
    G[(size_t)i * N + j] = acc;
  }
}

inline size_t jacobi_smem_bytes(int N) {
  const int Np = (N + 1) & ~1;
  return sizeof(double) * (2 * (size_t)Np * Np + 2 * Np + Np / 2) + sizeof(int) * Np;
}
