// Householder tridiagonalisation T = H^T A H of one symmetric block inside ONE thread-block cluster.
//
// First stage of the large-block PSD projection (north_star (c): "blocked
// Householder tridiagonalisation plus a tridiagonal solve and back-transform").  The reflectors
// H_k = I - tau_k v_k v_k^T (LAPACK dsytd2 conventions, lower storage) are applied one per step;
// step k needs p = tau A v (symmetric matrix-vector product over the trailing matrix),
// w = p - (tau/2)(p^T v) v and the rank-2 update A <- A - v w^T - w v^T.
//
// B200 mapping: the trailing lower triangle is distributed column-cyclically over the C CTAs of a
// cluster (C <= 16, non-portable size) and kept in shared memory (column j owned by CTA j mod C,
// stored from row j down; columns that do not fit stay in the block's global matrix, L2-resident).
// Per step the cluster synchronises three times (hardware cluster barrier, ~0.25 us measured);
// the partial symv vectors are reduced over distributed shared memory (DSMEM), in a fixed order so
// the result is bit-reproducible.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace cgx = cooperative_groups;

constexpr int TRD_NT = 512;
constexpr int TRD_MAXC = 16;
constexpr int TRD_MAXOWN = 80;  // owned columns per CTA (N <= 1280 with C = 16)

struct TridiagArgs {
  double* M;         // N x N column-major block matrix (lower triangle is the input)
  int N;
  int C;             // cluster size (CTAs)
  long long smem_cols_doubles;  // per-CTA shared-memory budget for column storage
  double* d;         // N
  double* e;         // N - 1
  double* tau;       // N - 1
  double* V;         // N x N column-major: v_k in column k, rows k+1..N-1 (v_k[k+1] = 1)
  const DevState* st;
  const IterScal* is;
  int check_state;
};

__device__ __forceinline__ double trd_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
#pragma unroll 1
  for (int i = 0; i < TRD_NT / 32; ++i) r += red[i];
  return r;  // every thread gets the same value (fixed order)
}

__global__ void __launch_bounds__(TRD_NT, 1) k_tridiag(TridiagArgs a) {
  if (a.check_state && (a.st->done || !a.is->proceed)) return;
  cgx::cluster_group cl = cgx::this_cluster();
  const int C = a.C, N = a.N;
  const int me = (int)cl.block_rank();
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) double sm[];
  // layout: v[N] w[N] pp[N] pslice[S+1] dotpart[1] red[32] | column storage
  double* v = sm;
  double* w = v + N;
  double* pp = w + N;
  const int Smax = (N + C - 1) / C + 1;
  double* pslice = pp + N;
  double* dotpart = pslice + Smax;
  double* red = dotpart + 2;
  double* colstore = red + 32;
  __shared__ double* colp[TRD_MAXOWN];  // generic pointer to A[j.., j] of owned column j
  __shared__ int ncol_own;

  // ---- distribute the owned columns: latest (shortest) columns first into shared memory ----
  if (tid == 0) {
    int cnt = 0;
    for (int j = me; j < N; j += C) ++cnt;
    ncol_own = cnt;
    long long used = 0;
    for (int q = cnt - 1; q >= 0; --q) {
      const int j = me + q * C;
      const long long len = N - j;
      if (used + len <= a.smem_cols_doubles) {
        colp[q] = colstore + used;
        used += len;
      } else {
        colp[q] = a.M + (size_t)j * N + j;  // spill: operate in place in global memory
      }
    }
  }
  __syncthreads();
  const int nown = ncol_own;
  for (int q = 0; q < nown; ++q) {
    const int j = me + q * C;
    double* dst = colp[q];
    const double* src = a.M + (size_t)j * N + j;
    if (dst != src)
      for (int i = tid; i < N - j; i += TRD_NT) dst[i] = src[i];
  }
  __syncthreads();

  for (int k = 0; k < N - 2; ++k) {
    const int owner = k % C;
    const int nk = N - k - 1;  // length of v (rows k+1 .. N-1)
    // ---- 1. the owner of column k builds the reflector (dlarfg) ----
    if (me == owner) {
      const double* col = colp[k / C];  // col[i - k] = A[i, k]
      double s2 = 0.0;
      for (int i = k + 2 + tid; i < N; i += TRD_NT) {
        const double x = col[i - k];
        s2 = fma(x, x, s2);
      }
      s2 = trd_block_sum(s2, red);
      const double alpha = col[1];
      double tk, beta, scale;
      if (s2 == 0.0) {
        tk = 0.0;
        beta = alpha;
        scale = 0.0;
      } else {
        beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
        tk = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int i = k + 1 + tid; i < N; i += TRD_NT) {
        const double vi = (i == k + 1) ? 1.0 : col[i - k] * scale;
        v[i] = vi;
        a.V[(size_t)k * N + i] = vi;
      }
      if (tid == 0) {
        a.d[k] = col[0];
        a.e[k] = beta;
        a.tau[k] = tk;
        dotpart[1] = tk;  // broadcast tau through shared memory
      }
    }
    cl.sync();  // #1: v_k ready in the owner's shared memory
    double tk;
    {
      double* ov = cl.map_shared_rank(v, owner);
      if (me != owner)
        for (int i = k + 1 + tid; i < N; i += TRD_NT) v[i] = ov[i];
      tk = *cl.map_shared_rank(dotpart + 1, owner);
    }
    __syncthreads();
    // ---- 2. partial symv over the owned trailing columns: pp = A_own v ----
    // owned trailing columns: j = me + q C >= k + 1
    const int q0 = (k + 1 - me + C - 1) / C > 0 ? (k + 1 - me + C - 1) / C : 0;
    for (int i = k + 1 + tid; i < N; i += TRD_NT) {
      double acc = 0.0;
      for (int q = q0; q < nown; ++q) {
        const int j = me + q * C;
        if (j >= i) break;
        acc = fma(colp[q][i - j], v[j], acc);
      }
      pp[i] = acc;
    }
    __syncthreads();
    {
      const int wid = tid >> 5, lane = tid & 31;
      for (int q = q0 + wid; q < nown; q += TRD_NT / 32) {
        const int j = me + q * C;
        const double* col = colp[q];
        double acc = 0.0;
        for (int i = j + lane; i < N; i += 32) acc = fma(col[i - j], v[i], acc);
        acc = warp_sum(acc);
        if (lane == 0) pp[j] += acc;
      }
    }
    cl.sync();  // #2: partial vectors ready
    // ---- 3. reduce my slice of rows over the cluster (fixed order), p = tau * sum ----
    const int S = (nk + C - 1) / C;
    const int r0 = k + 1 + me * S;
    const int r1 = min(N, r0 + S);
    double sdot = 0.0;
    for (int i = r0 + tid; i < r1; i += TRD_NT) {
      double acc = 0.0;
      for (int c = 0; c < C; ++c) acc += cl.map_shared_rank(pp, c)[i];
      const double p = tk * acc;
      pslice[i - r0] = p;
      sdot = fma(p, v[i], sdot);
    }
    sdot = trd_block_sum(sdot, red);
    if (tid == 0) dotpart[0] = sdot;
    cl.sync();  // #3: slices and slice dots ready
    // ---- 4. w = p - (tau/2)(p^T v) v, gathered from all slices; rank-2 update ----
    double pv = 0.0;
    for (int c = 0; c < C; ++c) pv += *cl.map_shared_rank(dotpart, c);
    const double K = 0.5 * tk * pv;
    for (int i = k + 1 + tid; i < N; i += TRD_NT) {
      const int c = (i - k - 1) / S;
      const double p = cl.map_shared_rank(pslice, c)[i - (k + 1 + c * S)];
      w[i] = p - K * v[i];
    }
    __syncthreads();
    for (int i = k + 1 + tid; i < N; i += TRD_NT) {
      const double vi = v[i], wi = w[i];
      for (int q = q0; q < nown; ++q) {
        const int j = me + q * C;
        if (j > i) break;
        double* cp = colp[q] + (i - j);
        *cp = *cp - vi * w[j] - wi * v[j];
      }
    }
    // slices / dotpart / pp are rewritten only after the next #2, by which time every CTA has
    // finished reading them (they passed #1 of step k+1 after this point).
    __syncthreads();
  }
  // ---- the final 2 x 2 trailing block ----
  if (N >= 2) {
    if (me == (N - 2) % C && tid == 0) {
      const double* col = colp[(N - 2) / C];
      a.d[N - 2] = col[0];
      a.e[N - 2] = col[1];
      a.tau[N - 2] = 0.0;
    }
    if (me == (N - 1) % C && tid == 0) a.d[N - 1] = colp[(N - 1) / C][0];
  } else if (me == 0 && tid == 0) {
    a.d[0] = colp[0][0];
  }
  cl.sync();
}

inline size_t tridiag_smem_bytes(int N, int C, long long col_doubles) {
  const int Smax = (N + C - 1) / C + 1;
  return sizeof(double) * ((size_t)3 * N + Smax + 2 + 32 + (size_t)col_doubles);
}
