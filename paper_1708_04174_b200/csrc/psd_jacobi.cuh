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
  double* vp;            // warm start: per small block the N x N eigenvectors of the
  const long long* blk_vp;  //   previous solve at vp + blk_vp[b] (identity before the first)
  int warm;              // 1 = start from B = P^T A P with P the previous eigenvectors
  int blocked;           // 1 = a round updates 2 x 2 blocks per thread (one shared-memory read per output): selects the
                         //     kernel instantiation on the host (jacobi_kernel)
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

// MAXN: compile-time bound of the launch's largest block (32 or 64), sizing the per-thread element
// slots.  Per round: the elementwise update A' = J^T A J, V' = V J from the ping-pong copy (no
// read/write hazard, the annihilated couplings written as exact zeros in the same pass), the next
// round's Np/2 rotation parameters (one of the last Np/2 threads each, from its own copies of the three entries it
// needs), ONE __syncthreads.
// Warm start (iterates unchanged up to rounding): consecutive ADMM iterations
// project slowly changing matrices, so the previous solve's eigenvectors P nearly diagonalise the
// new input; Jacobi runs on B = P^T A P (measured on pop6: 8.6 -> 4.9 sweeps, tools/
// warm_jacobi_probe.py) and the eigenvectors are P V_B.  Every 64th iteration starts cold (P = I)
// so that the rounding of the accumulated product never builds up.
template <int MAXN, int NT, bool BLK>
__global__ void __launch_bounds__(NT) k_psd_jacobi(JacobiArgs a) {
  if (a.check_state && (a.st->done || !a.is->proceed)) return;
  const int b = a.small_blk[blockIdx.x];
  const int N = a.blk_N[b];
  const int Np = (N + 1) & ~1;  // even; a padded zero row/column never rotates
  const int NN = Np * Np;
  double* G = a.mats + a.blk_mat[b];
  extern __shared__ double smem[];
  // A (ping-pong: smem + c NN) and V (smem + (2 + c) NN), Np x Np column-major each
  auto Ab = [&](int c) { return smem + (size_t)c * NN; };
  auto Vb = [&](int c) { return smem + (size_t)(2 + c) * NN; };
  double* P = smem + 4 * NN;                      // previous eigenvectors / final V
  double* alpha = smem + 5 * NN;                  // 2 Np (round-parity slots)
  double* beta = alpha + 2 * Np;                  // 2 Np
  __shared__ int nrot[4];
  __shared__ double offp[2 * (NT / 32)];  // per-warp off(A')^2 of a sweep's last round, by sweep parity
  __shared__ double normF;
  const int tid = threadIdx.x;

  for (int e = tid; e < NN; e += NT) {
    const int i = e % Np, j = e / Np;
    Ab(0)[e] = (i < N && j < N) ? G[(size_t)max(i, j) * N + min(i, j)] : 0.0;  // upper triangle (k_scatter)
    Vb(0)[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    double s = 0.0;
    for (int e = tid; e < NN; e += 32) s = fma(Ab(0)[e], Ab(0)[e], s);
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
  constexpr int PER = MAXN * MAXN / NT;
  int ei[PER], ej[PER];  // (row, column) of this thread's element slots, fixed for the whole solve
#pragma unroll
  for (int cnt = 0; cnt < PER; ++cnt) {
    const int e = tid + cnt * NT;
    ei[cnt] = e % Np;
    ej[cnt] = e / Np;
  }
  // C = X Y (Np x Np, column-major) over this thread's element slots
  auto mm = [&](const double* X, bool xt, const double* Y, double* C) {
#pragma unroll
    for (int cnt = 0; cnt < PER; ++cnt) {
      const int e = tid + cnt * NT;
      if (e < NN) {
        const int i = ei[cnt], j = ej[cnt];
        double acc = 0.0;
        for (int k = 0; k < Np; ++k) acc = fma(xt ? X[k + i * Np] : X[i + k * Np], Y[k + j * Np], acc);
        C[e] = acc;
      }
    }
  };
  double* vpg = a.vp + a.blk_vp[b];
  const bool warm = a.warm && (a.st->iter & 63) != 0;
  if (warm) {
    for (int e = tid; e < NN; e += NT) {
      const int i = e % Np, j = e / Np;
      P[e] = (i < N && j < N) ? vpg[(size_t)j * N + i] : (i == j ? 1.0 : 0.0);
    }
    __syncthreads();
    mm(Ab(0), false, P, Ab(1));  // T = A P
    __syncthreads();
    mm(P, true, Ab(1), Vb(1));   // B = P^T T (V buffers as scratch)
    __syncthreads();
    for (int e = tid; e < NN; e += NT) {  // symmetrise: Jacobi reads one triangle per pair
      const int i = e % Np, j = e / Np;
      Ab(0)[e] = 0.5 * (Vb(1)[i + j * Np] + Vb(1)[j + i * Np]);
    }
    __syncthreads();
  }
  // Rotation parameters, ping-pong by round parity: round g reads slot g & 1 while its parameter
  // threads (tid < Np/2) write round g + 1's into slot (g + 1) & 1.  They compute the three entries
  // a'_pp, a'_qq, a'_pq of the next round's pair from THIS round's update (the same expression, hence
  // the same bits, as the elementwise pass writes), so a round needs ONE __syncthreads.
  // nrot[s & 3] flags a rotation in sweep s (round 0 of sweep s + 1 is decided in sweep s's last round).
  auto params = [&](double apq, double app, double aqq, int p, int q, double* al, double* be, int slot) {
    double c = 1.0, sn = 0.0;
    if (apq * apq > EPS * EPS * fabs(app * aqq) && fabs(apq) > tiny) {
      // half-angle form (GvL sym.schur2), two rsqrt and no division: with h = sqrt(d^2 + (2 a_pq)^2),
      // c^2 = (1 + |d| / h) / 2 in [1/2, 1] (no cancellation), s = sign(d) a_pq / (h c)
      const double d = aqq - app, tw = 2.0 * apq;
      const double rh = rsqrt(fma(d, d, tw * tw));
      const double cc = 0.5 * fma(fabs(d), rh, 1.0);
      const double rc = rsqrt(cc);
      c = cc * rc;
      sn = copysign(1.0, d) * (0.5 * tw) * rh * rc;
      nrot[slot] = 1;
    }
    al[p] = c; be[p] = -sn;
    al[q] = c; be[q] = sn;
  };
  const int M = Np - 1;
  // partner of i in round r of the tournament: p + q = 2 r (mod M), the fixed player M meets r
  auto partner = [&](int i, int r2) {  // r2 = 2 r mod M
    if (i == M) return r2 & 1 ? (r2 + M) >> 1 : r2 >> 1;  // r = r2 / 2 (mod M, M odd)
    int t = r2 - i;
    t += t < 0 ? M : 0;
    return t == i ? M : t;
  };
  // parameter threads: the LAST Np/2 threads of the CTA, whose second element slot is empty when
  // Np^2 <= NT (MAXN) + NT - Np/2 (e.g. pop6's Np = 28 at NT = 512), so the round's longest thread
  // carries one element update fewer
  // Blocked round update (a.blocked): work items of a round are the (Np/2)^2 blocks {p_a, q_a} x {p_b, q_b} of
  // A' = J^T A J (pairs a, b = tournament slots: four reads, four outputs) and the Np x Np/2 row-pair items
  // (i, {p_b, q_b}) of V' = V J (two reads, two outputs): one shared-memory read per output instead of four /
  // two (the elementwise pass is shared-memory-bandwidth bound: 63 KB per round at N = 28).  The slot
  // decomposition of a thread's items is fixed for the whole solve.
  const int H = Np >> 1;
  constexpr int PERI = BLK ? (MAXN / 2 * (MAXN / 2) + MAXN * (MAXN / 2) + NT - 1) / NT : 1;
  short ia[PERI], ib[PERI];  // item (ia, ib): A block of slots (ia, ib) if ia < H, else V item (row ia - H, slot ib)
#pragma unroll
  for (int cnt = 0; cnt < (BLK ? PERI : 0); ++cnt) {
    const int it = tid + cnt * NT;
    int x = -1, y = 0;
    if (it < H * H) {  // slot a fastest: consecutive lanes read consecutive rows p_a (descending q_a)
      x = it % H;
      y = it / H;
    } else if (it < H * H + Np * H) {
      const int v = it - H * H;
      x = H + v % Np;
      y = v / Np;
    }
    ia[cnt] = (short)x;
    ib[cnt] = (short)y;
  }
  // pair of slot k in round r without a division (0 <= r, k < M)
  auto slot_pair = [&](int r, int k, int& p, int& q) {
    if (k == 0) {
      p = M;
      q = r;
    } else {
      p = r + k;
      p -= p >= M ? M : 0;
      q = r - k;
      q += q < 0 ? M : 0;
    }
  };
  const int pt = tid - (NT - Np / 2);
  if (tid < 4) nrot[tid] = 0;
  __syncthreads();
  if (pt >= 0) {  // round 0 from the (warm-started) input
    int p, q;
    rr_pair(0, pt, Np, p, q);
    params(Ab(0)[p + q * Np], Ab(0)[p + p * Np], Ab(0)[q + q * Np], p, q, alpha, beta, 0);
  }
  __syncthreads();
  int cur = 0, g = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    for (int r = 0; r < M; ++r, ++g) {
      const double* A = Ab(cur);
      const double* V = Vb(cur);
      const double* al = alpha + (g & 1) * Np;
      const double* be = beta + (g & 1) * Np;
      const int r2 = (2 * r) % M;
      double* An = Ab(cur ^ 1);
      double* Vn = Vb(cur ^ 1);
      // A' = J^T A J, V' = V J elementwise from the 2 x 2 coupling of (row i, ip) x (col j, jp)
      auto elem = [&](int i, int j) {
        const int ip = partner(i, r2), jp = partner(j, r2);
        const double ai = al[i], bi = be[i], aj = al[j], bj = be[j];
        const double na = ai * (aj * A[i + j * Np] + bj * A[i + jp * Np]) +
                          bi * (aj * A[ip + j * Np] + bj * A[ip + jp * Np]);
        return (j == ip && bi != 0.0) ? 0.0 : na;  // the coupling of a rotated pair: exact zero
      };
      double off2 = 0.0;  // this thread's share of off(A')^2, summed in a sweep's last round
      if constexpr (BLK) {
        // out(i, j) of the 2 x 2 coupling: rows (i, ip) with (ai, bi), columns (j, jp) with (aj, bj); x = A[i, j],
        // y = A[i, jp], z = A[ip, j], w = A[ip, jp] -- elem()'s expression
        auto rot = [](double ai, double bi, double aj, double bj, double x, double y, double z, double w) {
          return ai * (aj * x + bj * y) + bi * (aj * z + bj * w);
        };
#pragma unroll
        for (int cnt = 0; cnt < PERI; ++cnt) {
          const int x = ia[cnt], kb = ib[cnt];
          if (x < 0) continue;
          int pb, qb;
          slot_pair(r, kb, pb, qb);
          const double cb = al[pb], sb = be[pb];  // (al, be)[qb] = (cb, -sb)
          if (x < H) {
            int pa, qa;
            slot_pair(r, x, pa, qa);
            const double ca = al[pa], sa = be[pa];
            const double a00 = A[pa + pb * Np], a01 = A[pa + qb * Np], a10 = A[qa + pb * Np], a11 = A[qa + qb * Np];
            double n00 = rot(ca, sa, cb, sb, a00, a01, a10, a11);    // (pa, pb)
            double n01 = rot(ca, sa, cb, -sb, a01, a00, a11, a10);   // (pa, qb)
            double n10 = rot(ca, -sa, cb, sb, a10, a11, a00, a01);   // (qa, pb)
            double n11 = rot(ca, -sa, cb, -sb, a11, a10, a01, a00);  // (qa, qb)
            if (x == kb) {  // the rotated pair itself: its coupling is an exact zero
              if (sa != 0.0) n01 = n10 = 0.0;
              off2 = fma(n01, n01, fma(n10, n10, off2));
            } else {
              off2 = fma(n00, n00, fma(n01, n01, fma(n10, n10, fma(n11, n11, off2))));
            }
            An[pa + pb * Np] = n00;
            An[pa + qb * Np] = n01;
            An[qa + pb * Np] = n10;
            An[qa + qb * Np] = n11;
          } else {
            const int i = x - H;
            const double v0 = V[i + pb * Np], v1 = V[i + qb * Np];
            Vn[i + pb * Np] = cb * v0 + sb * v1;
            Vn[i + qb * Np] = cb * v1 - sb * v0;
          }
        }
      } else {
#pragma unroll
      for (int cnt = 0; cnt < PER; ++cnt) {
        const int e = tid + cnt * NT;
        if (e < NN) {
          const int i = ei[cnt], j = ej[cnt];
          const int jp = partner(j, r2);
          const double v = elem(i, j);
          An[e] = v;
          Vn[e] = al[j] * V[i + j * Np] + be[j] * V[i + jp * Np];
          off2 = i != j ? fma(v, v, off2) : off2;
        }
      }
      }
      if (r == M - 1) {
        off2 = warp_sum(off2);
        if ((tid & 31) == 0) offp[(sweep & 1) * (NT / 32) + (tid >> 5)] = off2;
      }
      if (pt >= 0) {  // the next round's parameters from this round's a'_pq, a'_pp, a'_qq
        const int rn = r + 1 == M ? 0 : r + 1;
        int p, q;
        rr_pair(rn, pt, Np, p, q);
        params(elem(p, q), elem(p, p), elem(q, q), p, q, alpha + ((g + 1) & 1) * Np, beta + ((g + 1) & 1) * Np,
               (sweep + (rn == 0)) & 3);
      }
      cur ^= 1;
      __syncthreads();
    }
    // Stop after a quiet sweep, or as soon as off(A)_F <= N tiny (the bound a quiet sweep leaves: every
    // coupling <= tiny): |Pi(A) - V diag(lambda_+) V^T|_F <= off(A)_F since Pi is 1-Lipschitz
    double off2 = 0.0;
#pragma unroll 4
    for (int w = 0; w < NT / 32; ++w) off2 += offp[(sweep & 1) * (NT / 32) + w];
    if (nrot[sweep & 3] == 0 || off2 <= (double)N * N * tiny * tiny) {
#ifdef SOSADMM_JACOBI_DEBUG
      if (tid == 0) printf("jacobi block %d N %d sweeps %d\n", b, N, sweep + 1);
#endif
      break;
    }
    // slot of sweep + 3 (= sweep - 1): read by every thread at the end of sweep - 1 (a barrier ago),
    // next written in the last round of sweep + 2 (a barrier ahead), whichever thread computes parameters
    if (tid == 0) nrot[(sweep + 3) & 3] = 0;
  }
  const double* A = Ab(cur);
  const double* V = Vb(cur);
  if (warm) {
    mm(P, false, V, Ab(cur ^ 1));  // eigenvectors of the input: P V_B
    V = Ab(cur ^ 1);
  }
  // Pi(A) = V diag(max(lambda, 0)) V^T, lambda_k = A[k, k]; V is kept for the next warm start
  for (int k = tid; k < Np; k += NT) alpha[k] = fmax(A[k + k * Np], 0.0);
  __syncthreads();
  if (a.warm)
    for (int e = tid; e < N * N; e += NT) {
      const int i = e % N, j = e / N;
      vpg[(size_t)j * N + i] = V[i + j * Np];
    }
  for (int e = tid; e < N * N; e += NT) {
    const int i = e % N, j = e / N;
    if (i < j) continue;  // one entry per pair: k_pack reads the upper triangle (column i, row j <= i)
    double acc = 0.0;
    for (int k = 0; k < Np; ++k) acc = fma(V[i + k * Np] * alpha[k], V[j + k * Np], acc);
    G[(size_t)i * N + j] = acc;
  }
}

inline size_t jacobi_smem_bytes(int N) {
  const int Np = (N + 1) & ~1;
  return sizeof(double) * (5 * (size_t)Np * Np + 4 * Np);
}

typedef void (*JacobiKernel)(JacobiArgs);
constexpr int JAC_NT32 = 512;  // threads for blocks N <= 32 (measured: 64 / 128 / 256 / 512 / 1024 -> 0.27 / 0.17 / 0.14 / 0.12 / 0.13 ms on pop6)
inline JacobiKernel jacobi_kernel(int max_small_N, int blocked) {
  if (blocked) return max_small_N <= 32 ? k_psd_jacobi<32, JAC_NT32, true> : k_psd_jacobi<64, JAC_NT, true>;
  return max_small_N <= 32 ? k_psd_jacobi<32, JAC_NT32, false> : k_psd_jacobi<64, JAC_NT, false>;
}
inline int jacobi_threads(int max_small_N) { return max_small_N <= 32 ? JAC_NT32 : JAC_NT; }
