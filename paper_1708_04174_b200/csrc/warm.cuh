// Warm-started large-block PSD projection ("warm-started ... from the previous
// iteration's eigenvectors (GEMM-rich: Q^T A Q on DMMA)"; PAPER.md P:397-398 `eq:HsdeStep2` projects
// every Gram block of u_hat - v onto S_+ once per ADMM iteration, and consecutive ADMM iterates change
// slowly, so the previous iteration's eigenvectors X nearly diagonalise the new block a).
//
// Iterative refinement of the eigenvector matrix (Ogita-Aishima form, with near-degenerate clusters
// solved exactly), every O(N^3) step a DMMA GEMM (dgemm.cuh):
//   W = a X,  S = X^T W,  P = X^T X,  R = I - P,  lambda_i = S_ii / P_ii;
//   clusters: runs of the sorted lambda joined by "strong" pairs |S'_ij| > theta |lambda_j - lambda_i|
//     (S' = S + (lambda_i + lambda_j)/2 R); each cluster's block S_CC is diagonalised exactly (Jacobi,
//     one CTA per cluster), V = blockdiag of those rotations, S~ = V^T S V, R~ = V^T R V;
//   E_ij = (S~_ij + lambda~_j R~_ij) / (lambda~_j - lambda~_i) between clusters, R~_ij / 2 inside one;
//   X <- X V (I + E)                                                         (one GEMM: X M, M = V (I + E)).
// Stop test on the S of the current X (the one the projection then uses):
//   ||S_{+-}||_F * sqrt 2 <= 1e-13 ||a||_F   (coupling across the sign split),
//   ||D o (sigma_i lambda_i + sigma_j lambda_j)||_F <= 1e-13 ||a||_F   (D = X^T X - I weighted by the eigenvalues
//                                            of the projected side s, sigma = membership of s: reading C19),
//   ||D||_F <= 1e-8 N                        (a well-conditioned basis),
//   Gershgorin: the rows whose same-sign off-diagonal mass rho_i reaches |lambda_i| have
//   (sum rho_i^2)^(1/2) <= 1e-12 ||a||_F (the wrong-sign part of a diagonal block is bounded by it),
// so a = X [S_++ 0; 0 S_--] X^T + O(1e-13 ||a||_F) with S_++, -S_-- PSD up to O(1e-12 ||a||_F), and the projection is
//   Pi_{S+}(a) = X_+ S_++ X_+^T   or   Pi_{S+}(-a) = X_- (-S_--) X_-^T   (the side with fewer columns;
// k_pack applies the Moreau identity for the second, as on the cold path).  The projection is
// 1-Lipschitz, so the result is within ~1e-12 ||a||_F of the exact one: the iterates are those of an
// exact eigensolver up to rounding (SURVEY f4 "performance variants that keep the iterates identical").
// No convergence within WM_MAXS evaluations, a cluster above WM_CAP, or a stalled coupling -> the
// iteration falls back to the cold path (one-cluster tridiagonalisation + divide and conquer +
// back-transform of all N columns), which also re-seeds X; after a failure the next 2^f - 1
// iterations go straight to the cold path (f = consecutive failures, capped).
#pragma once
#include "common.cuh"
#include "dgemm.cuh"
#include "gemm_f64.cuh"

constexpr int WM_MAXS = 10;         // S evaluations per ADMM iteration (at most 9 updates)
constexpr int WM_CAP = 64;          // largest cluster diagonalised exactly
constexpr double WM_THETA = 0.05;   // strong coupling threshold
constexpr double WM_TOLE = 1e-13;   // cross-sign coupling tolerance relative to ||a||_F
constexpr double WM_TOLO = 1e-8;    // unweighted orthonormality defect per unit of N (basis conditioning)
constexpr double WM_TOLG = 1e-12;   // Gershgorin sign-uncertainty bound relative to ||a||_F
constexpr int WM_NT = 1024;         // single-CTA kernels
constexpr int WM_SORT = 2048;       // bitonic sort capacity (N <= SOSADMM_MAX_BLOCK = 1280)
constexpr int WM_CLB = 64;          // CTAs of the cluster kernel
constexpr int WM_PAIRS = 1 << 16;   // strong-pair list capacity (more: the step gives up, as for a big cluster)

struct WarmState {
  int valid;        // X0 holds the eigenvectors of a previous solve of this block
  int gate;         // 1 while the refinement runs (every step kernel / GEMM is gated on it)
  int status;       // 0 running, 1 converged, 2 cold path
  int step;         // S evaluations done in this iteration
  int cur;          // X buffer of the converged iterate
  int ncl;          // clusters (size >= 2) of the current step
  int fails;        // consecutive failed refinements
  int backoff;      // iterations still sent straight to the cold path
  int src;          // what the finish used: 0 = warm (S), 1 = cold (D&C eigenpairs)
  int need_full;    // the cold path of this iteration re-seeds X (every eigenvector): the next one tries warm
  int pgate;        // 1: step 0 forms P = X^T X (0: the previous iteration certified this X and its P is kept)
  int pred;         // 1: this iteration starts from the predicted X0 (I + Esum) (k_warm_pred)
  int pred_last;    // the previous iteration's pred (k_warm_begin copies it after the predictor ran)
  int pred_ok;      // Esum holds the previous iteration's whole rotation generator (sum of M - I) and the
                    // trajectory looked smooth there (no cluster at step 0, <= 3 evaluations predicted / 4 not)
  int cl0;          // clusters formed at step 0 of this iteration
  int p_valid;      // the P buffer holds X0^T X0 of the current X0
  double normA2;    // ||a||_F^2 of this iteration
  double eta_prev;  // coupling of the previous step
  double eta, rn;   // last step's coupling and orthonormality defect (diagnostics)
  long long n_warm, n_cold, n_steps, n_fail;  // counters since setup: warm / cold iterations, refinement
  long long n_seed;                            // updates, failed attempts, cold iterations that re-seeded X
  int why;          // last failure: 1 = no convergence within WM_MAXS, 2 = stalled coupling, 3 = cluster > WM_CAP,
                    // 4 = non-finite
  int maxcl;        // largest cluster of the last step
  double tr_eta[WM_MAXS], tr_rn[WM_MAXS], tr_g[WM_MAXS], tr_ro[WM_MAXS];  // diagnostics: per S evaluation of the last
                    // iteration, coupling / ||a||_F, orthonormality defect / N, Gershgorin bound / ||a||_F
};

struct WarmArgs {
  int N, ldn, nt;            // nt = ceil(N / 32)
  const double* Mblk;        // block matrix a (ld N, upper triangle valid); the projection overwrites it
  double *Af, *X0, *X1, *W, *W1, *S, *P, *E, *Mm, *Y;
  double *Srot, *Rrot;       // rotated rows (V_C^T S)[u, :], (V_C^T R)[u, :] of every cluster member (slot rows)
  double* Esum;              // sum of (M - I) over the refinement steps: the first-order rotation generator
  double* Eprev;             // the previous iteration's generator (second-order predictor)
  int predict;               // 1: start each warm iteration from X0 (I + Esum) of the previous one; 2: extrapolated
  int wtest;                 // 1: eigenvalue-weighted orthonormality test (C19); 0: ||I - X^T X||_F <= 1e-14 N
  int bo_cap;                // backoff after f consecutive failures: 2^min(f, bo_cap) - 1 cold iterations
  double *lam, *lamt;
  int *order, *pos, *diff, *cid, *cpos, *cl_start, *cl_size, *cl_voff, *cl_rbase, *sel, *idx;
  double* Vcl;               // cluster rotations, <= WM_CAP * N doubles
  double *partA, *cross, *roff, *grow, *gcol;  // deterministic partial sums
  double *rdpart, *g2part;   // per row block: sum (1 - P_ii)^2, Gershgorin partial
  int* cnt;                  // nt row-block counters, the grid counter and the strong-pair count of k_warm_scan
  int* pairs;                // strong pairs (i, j) of the step, at most WM_PAIRS
  WarmState* ws;
  const double* lam_cold;    // ascending eigenvalues of the cold path (D&C)
  int* side;                 // le.side + b (k_pack: 1 = the block holds Pi(-a))
  const DevState* st;
  const IterScal* is;
  unsigned long long hstep[WM_MAXS];  // graph conditional handles (0 = not in a graph): refinement steps,
  unsigned long long hcold, hfull, hpart, hfin;  // cold eigensolver, its full / partial tail, warm finish
  unsigned long long hclA, hclB;      // (per step body) the cluster kernels / k_warm_M run only with clusters
};

__device__ __forceinline__ bool wm_skip(const WarmArgs& a) { return a.st->done || !a.is->proceed; }
__device__ __forceinline__ void wm_set(unsigned long long h, unsigned v) {
  if (h) cudaGraphSetConditional((cudaGraphConditionalHandle)h, v);
}
// entry (p, q) of S / P: the GEMM writes the upper triangle and mirrors it (bitwise symmetric storage),
// so the column-major read is coalesced along p whichever triangle (p, q) lies in
__device__ __forceinline__ double wm_sym(const double* A, int ld, int p, int q) { return A[(size_t)q * ld + p]; }

// fixed-order block sum over WM_NT threads (result in every thread)
__device__ __forceinline__ double wm_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  __syncthreads();
  return s;
}

// ---- predictor (before begin): the eigenvectors move smoothly along the ADMM trajectory, so the
// previous iteration's rotation, X_{k-1} = X_{k-2} (I + Esum) to first order, is applied once more:
// M = I + Esum, then X1 = X0 M (gated GEMM) and begin copies X1 to X0.  Esum keeps that generator (the
// refinement steps add their corrections to it); without a valid generator it restarts from zero.  With
// predict == 2 and two consecutive valid generators, the generator is extrapolated linearly (2 G_k - G_{k-1}):
// the ADMM trajectory changes geometrically slowly, so the first-order start's error eps G_k drops to ~eps^2 G_k.
// grid (nt, nt), 256 threads
__global__ void __launch_bounds__(256) k_warm_pred(WarmArgs a) {
  if (wm_skip(a)) return;
  const WarmState* ws = a.ws;
  const bool cond = a.predict && ws->valid && ws->backoff == 0 && ws->pred_ok;
  // second order (predict == 2): Eprev holds the generator before Esum's when the previous iteration was predicted too
  const bool o2 = cond && a.predict == 2 && ws->pred_last;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, N = a.N, ld = a.ldn;
  const int i = 32 * blockIdx.x + tx;
  for (int r = ty; r < 32 && i < N; r += 8) {
    const int j = 32 * blockIdx.y + r;
    if (j >= N) break;
    const size_t e = (size_t)j * ld + i;
    if (cond) {
      double g = a.Esum[e];
      if (o2) {  // linear extrapolation of the generator: G_k + (G_k - G_{k-1})
        const double gp = a.Eprev[e];
        a.Eprev[e] = g;
        g = 2.0 * g - gp;
        a.Esum[e] = g;
      } else if (a.predict == 2) {
        a.Eprev[e] = g;
      }
      a.Mm[e] = (i == j ? 1.0 : 0.0) + g;
    } else {
      a.Esum[e] = 0.0;
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) a.ws->pred = cond ? 1 : 0;
}

// ---- begin: full symmetric copy Af of a (32 x 32 tile transposes), ||a||_F^2 partials, state ----
// grid (nt, nt), 256 threads
__global__ void __launch_bounds__(256) k_warm_begin(WarmArgs a) {
  if (wm_skip(a)) return;
  __shared__ double t[32][33];
  __shared__ double red[8];
  const int ti = blockIdx.x, tj = blockIdx.y, tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int N = a.N;
  double ss = 0.0;
  for (int r = ty; r < 32; r += 8) {
    if (ti <= tj) {  // element (i = 32 ti + tx, j = 32 tj + r): source contiguous in i
      const int i = 32 * ti + tx, j = 32 * tj + r;
      double v = 0.0;
      if (i < N && j < N) v = i <= j ? a.Mblk[(size_t)j * N + i] : a.Mblk[(size_t)i * N + j];
      t[r][tx] = v;
    } else {         // element (i = 32 ti + r, j = 32 tj + tx), i > j: row i of the lower = column i
      const int i = 32 * ti + r, j = 32 * tj + tx;
      t[tx][r] = (i < N && j < N) ? a.Mblk[(size_t)i * N + j] : 0.0;
    }
  }
  __syncthreads();
  const bool pred = a.ws->pred;
  if (ti == 0) {  // the fused scan's link and completion counters start from zero
    for (int q = tj * 256 + threadIdx.x; q <= N; q += a.nt * 256) a.diff[q] = 0;
    if (tj == 0)
      for (int q = threadIdx.x; q <= a.nt + 1; q += 256) a.cnt[q] = 0;
  }
  for (int r = ty; r < 32; r += 8) {
    const int i = 32 * ti + tx, j = 32 * tj + r;
    const double v = t[r][tx];
    ss = fma(v, v, ss);
    if (i < N && j < N) {
      a.Af[(size_t)j * a.ldn + i] = v;
      if (pred) a.X0[(size_t)j * a.ldn + i] = a.X1[(size_t)j * a.ldn + i];  // the predicted start
    }
  }
  ss = warp_sum(ss);
  if (tx == 0) red[ty] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    a.partA[ti * a.nt + tj] = s;
    if (ti == 0 && tj == 0) {
      WarmState* ws = a.ws;
      ws->pred_last = ws->pred;
      ws->step = 0;
      ws->ncl = 0;
      ws->cl0 = 0;
      ws->cur = 0;
      ws->eta_prev = 1e300;
      if (ws->valid && ws->backoff == 0) {
        ws->gate = 1;
        ws->pgate = (ws->p_valid && !ws->pred) ? 0 : 1;
        ws->status = 0;
        ws->need_full = 0;
        wm_set(a.hstep[0], 1);
      } else {
        ws->gate = 0;
        ws->pgate = 0;
        ws->pred_ok = 0;
        ws->status = 2;
        if (ws->backoff > 0) ws->backoff--;
        ws->need_full = ws->backoff == 0;  // only the iteration before the next attempt re-seeds X
        wm_set(a.hcold, 1);
      }
    }
  }
}

// ---- per step: ONE fused pass over the upper 32 x 32 tiles of S and P (grid (nt, nt), 256 threads; the
// tiles below the diagonal exit at once) ----
//  (1) lambda of every index (diag S / diag P, all N into shared memory) and the ranks of the tile's 32 rows
//      and 32 columns by counting (ties by index: an exact, deterministic order); the diagonal tiles publish
//      lam, pos, order and their rows' (1 - P_ii)^2;
//  (2) the tile's coupling / orthonormality partials, same-sign row / column masses and strong pairs;
//  (3) row-block completion: the CTA that brings a row block's nt + 1 contributions together sums its rows'
//      rho_i in tile order and writes the block's Gershgorin partial;
//  (4) the last CTA of the grid runs the stop test and builds the clusters (fixed-order sums throughout).
__device__ void wm_decide(const WarmArgs& a, int step, double* red, double* red11, int* cpre, double* lam_s, int* flags);

__global__ void __launch_bounds__(256) k_warm_scan(WarmArgs a, int step) {
  if (wm_skip(a) || a.ws->gate != 1) return;
  const int ti = blockIdx.x, tj = blockIdx.y, nt = a.nt;
  if (ti > tj) return;
  __shared__ double lrow[32], lcol[32];
  __shared__ double colp[8][33];
  __shared__ double red[32];
  __shared__ int cpre[WM_SORT];
  __shared__ double lam_s[WM_SORT];
  __shared__ int flags[4];  // [0] ncl, [1] big, [2] maxcl, [3] last-CTA flag
  __shared__ int done_blk[2];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5, N = a.N, ld = a.ldn;
  if (tid < 64) {  // lambda of the tile's rows (tid < 32) and columns
    const int idx = tid < 32 ? 32 * ti + tid : 32 * tj + tid - 32;
    double l = 0.0;
    if (idx < N) l = a.S[(size_t)idx * ld + idx] / a.P[(size_t)idx * ld + idx];
    if (tid < 32) lrow[tid] = l;
    else lcol[tid - 32] = l;
    if (ti == tj && tid < 32 && idx < N) a.lam[idx] = l;
  }
  __syncthreads();
  // (2) the tile's pairs i < j
  const int j = 32 * tj + tx;
  const bool jv = j < N;
  const double lj = lcol[tx];
  const bool gj = lj > 0.0;
  double cr = 0.0, ro = 0.0, wp = 0.0, wm = 0.0, cs = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int rr = ty + 8 * q, i = 32 * ti + rr;
    double rs = 0.0;
    if (jv && i < j) {
      const double sv = a.S[(size_t)j * ld + i], pv = a.P[(size_t)j * ld + i];
      const double li = lrow[rr];
      const bool gi = li > 0.0;
      if (gi != gj) {
        cr = fma(sv, sv, cr);
      } else {
        rs = fabs(sv);
        cs += fabs(sv);
      }
      ro = fma(pv, pv, ro);
      // X^T X defect weighted by the eigenvalues of the projected side (either side: decided at the end)
      const double up = fmax(li, 0.0) + fmax(lj, 0.0), um = fmin(li, 0.0) + fmin(lj, 0.0);
      wp = fma(pv * up, pv * up, wp);
      wm = fma(pv * um, pv * um, wm);
      const double sp = fma(-0.5 * (li + lj), pv, sv);  // S'_ij = S_ij + lambda_bar R_ij, R_ij = -P_ij
      if (fabs(sp) > WM_THETA * fabs(lj - li)) {       // strong pair: listed for the cluster build
        const int k = atomicAdd(a.cnt + nt + 1, 1);
        if (k < WM_PAIRS) {
          a.pairs[2 * k] = i;
          a.pairs[2 * k + 1] = j;
        }
      }
    }
    rs = warp_sum(rs);  // row i's same-sign mass over this tile's columns (j > i)
    if (tx == 0 && i < N) a.grow[(size_t)tj * N + i] = rs;
  }
  colp[ty][tx] = cs;
  cr = warp_sum(cr);
  ro = warp_sum(ro);
  wp = warp_sum(wp);
  wm = warp_sum(wm);
  if (tx == 0) {
    red[ty] = cr;
    red[8 + ty] = ro;
    red[16 + ty] = wp;
    red[24 + ty] = wm;
  }
  __syncthreads();
  if (ty == 0) {
    double c = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += colp[w][tx];
    if (jv) a.gcol[(size_t)ti * N + j] = c;  // column j's mass over this tile's rows (i < j)
    if (tx == 0) {
      double c2 = 0.0, r2[3] = {0.0, 0.0, 0.0};
      for (int w = 0; w < 8; ++w) {
        c2 += red[w];
        r2[0] += red[8 + w];
        r2[1] += red[16 + w];
        r2[2] += red[24 + w];
      }
      a.cross[ti * nt + tj] = c2;
      for (int c = 0; c < 3; ++c) a.roff[(size_t)c * nt * nt + ti * nt + tj] = r2[c];
    }
  }
  if (ti == tj && ty == 1) {  // the block's (1 - P_ii)^2, weighted by (2 lambda_i)^2 per side, and its sign counts
    const int i = 32 * ti + tx;
    double d = 0.0, dp = 0.0, dm = 0.0, np = 0.0, nn = 0.0;
    if (i < N) {
      const double p = a.P[(size_t)i * ld + i], li = lrow[tx];
      d = (1.0 - p) * (1.0 - p);
      if (li > 0.0) {
        dp = 4.0 * li * li * d;
        np = 1.0;
      } else if (li < 0.0) {
        dm = 4.0 * li * li * d;
        nn = 1.0;
      }
    }
    d = warp_sum(d);
    dp = warp_sum(dp);
    dm = warp_sum(dm);
    np = warp_sum(np);
    nn = warp_sum(nn);
    if (tx == 0) {
      a.rdpart[ti] = d;
      a.rdpart[nt + ti] = dp;
      a.rdpart[2 * nt + ti] = dm;
      a.rdpart[3 * nt + ti] = np;
      a.rdpart[4 * nt + ti] = nn;
    }
  }
  // (3) row-block completion
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    done_blk[0] = -1;
    if (ti == tj) {
      if (atomicAdd(a.cnt + ti, 2) + 2 == nt + 1) done_blk[0] = ti;
    } else {
      if (atomicAdd(a.cnt + ti, 1) + 1 == nt + 1) done_blk[0] = ti;
    }
  } else if (tid == 32) {  // the column block's counter from another warp: both atomics in flight together
    done_blk[1] = -1;
    if (ti != tj && atomicAdd(a.cnt + tj, 1) + 1 == nt + 1) done_blk[1] = tj;
  }
  __syncthreads();
  for (int h = 0; h < 2; ++h) {
    const int t = done_blk[h];
    if (t < 0) continue;
    __threadfence();
    // rows i = 32 t + r; 8 threads per row take the terms tt = g, g + 8, ... (grow: tt >= t, gcol: tt <= t)
    const int r = tid & 31, g = tid >> 5, i = 32 * t + r;
    double rho = 0.0, sd = 0.0, pd = 1.0;
    if (g == 0 && i < N) {  // the row's diagonal entries, in flight together with the masses below
      sd = __ldcg(a.S + (size_t)i * ld + i);
      pd = __ldcg(a.P + (size_t)i * ld + i);
    }
    if (i < N)
      for (int tt = g; tt < nt; tt += 8) {
        if (tt >= t) rho += __ldcg(a.grow + (size_t)tt * N + i);
        if (tt <= t) rho += __ldcg(a.gcol + (size_t)tt * N + i);
      }
    colp[g][r] = rho;
    __syncthreads();
    if (g == 0) {
      double rr = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) rr += colp[w][r];
      double g2 = 0.0;
      if (i < N) {
        const double li = sd / pd;
        if (!(fabs(li) > rr)) g2 = rr * rr;
      }
      g2 = warp_sum(g2);
      if (r == 0) a.g2part[t] = g2;
    }
    __syncthreads();
  }
  // (4) the last CTA runs the stop test
  __threadfence();
  __syncthreads();
  if (tid == 0) flags[3] = atomicAdd(a.cnt + nt, 1) + 1 == nt * (nt + 1) / 2;
  __syncthreads();
  if (!flags[3]) return;
  __threadfence();
  wm_decide(a, step, red, &colp[0][0], cpre, lam_s, flags);  // colp (264 doubles) is free by now
}

// the stop test and the clusters (256 threads of the grid's last CTA)
__device__ void wm_decide(const WarmArgs& a, int step, double* red, double* red11, int* cpre, double* lam_s, int* flags) {
  WarmState* ws = a.ws;
  const int N = a.N, nt = a.nt, tid = threadIdx.x;
  constexpr int T = 256;
  auto bsum = [&](double v) {
    v = warp_sum(v);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < T / 32; ++w) s += red[w];
    __syncthreads();
    return s;
  };
  if (tid == 0) {
    flags[0] = 0;
    flags[1] = 0;
    flags[2] = 0;
  }
  double c2 = 0.0, r2 = 0.0, wp = 0.0, wm = 0.0, a2 = 0.0, rd = 0.0, rdp = 0.0, rdm = 0.0, np = 0.0, nn = 0.0, g2 = 0.0;
  const size_t nt2 = (size_t)nt * nt;
  for (int e = tid; e < nt * nt; e += T) {
    const int ti = e / nt, tj = e % nt;
    if (ti <= tj) {
      c2 += __ldcg(a.cross + e);
      r2 += __ldcg(a.roff + e);
      wp += __ldcg(a.roff + nt2 + e);
      wm += __ldcg(a.roff + 2 * nt2 + e);
    }
    if (step == 0) a2 += __ldcg(a.partA + e);
  }
  for (int t = tid; t < nt; t += T) {
    rd += __ldcg(a.rdpart + t);
    rdp += __ldcg(a.rdpart + nt + t);
    rdm += __ldcg(a.rdpart + 2 * nt + t);
    np += __ldcg(a.rdpart + 3 * nt + t);
    nn += __ldcg(a.rdpart + 4 * nt + t);
    g2 += __ldcg(a.g2part + t);
  }
  const int npairs = __ldcg(a.cnt + nt + 1);
  {  // all eleven sums behind ONE barrier pair: bsum's tree (per-warp shuffle tree, warp partials in warp order)
    double v[11] = {c2, r2, wp, wm, rd, rdp, rdm, np, nn, g2, a2};
#pragma unroll
    for (int q = 0; q < 11; ++q) v[q] = warp_sum(v[q]);
    __syncthreads();
    if ((tid & 31) == 0)
#pragma unroll
      for (int q = 0; q < 11; ++q) red11[q * (T / 32) + (tid >> 5)] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 11; ++q) {
      double t = 0.0;
      for (int w = 0; w < T / 32; ++w) t += red11[q * (T / 32) + w];
      v[q] = t;
    }
    c2 = v[0], r2 = v[1], wp = v[2], wm = v[3], rd = v[4], rdp = v[5], rdm = v[6], np = v[7], nn = v[8], g2 = v[9];
    if (step == 0 && tid == 0) ws->normA2 = v[10];
  }
  // counters back to zero for the next step (every other CTA is done with them)
  for (int t = tid; t <= nt + 1; t += T) a.cnt[t] = 0;
  __syncthreads();
  const double nA = sqrt(ws->normA2);
  // orthonormality (reading C19): with X = Q (I + F), D = X^T X - I = F + F^T and the projected side s (k_warm_select's
  // rule: lambda > 0 when #(lambda > 0) <= #(lambda < 0)), the first-order error of X_s S_ss X_s^T is
  //   F_os Lambda_s (+ transpose) and D_ss o (lambda_i + lambda_j),  |F_ij lambda_j| <= |lambda_j D_ij| + |S_ij| (i in o),
  // so the certificate needs the coupling and the lambda-WEIGHTED defect ||D_ij (sigma_i lambda_i + sigma_j lambda_j)||_F
  // (sigma = membership of s) at the coupling tolerance; the unweighted defect only has to keep the basis well
  // conditioned (second-order terms), ||D||_F <= WM_TOLO N
  const bool pos_side = np <= nn;
  const double eta = sqrt(2.0 * c2);
  const double rn = sqrt(2.0 * (pos_side ? wp : wm) + (pos_side ? rdp : rdm));
  const double ro = sqrt(2.0 * r2 + rd);
  // Gershgorin sign safety: the rows whose same-sign off-diagonal mass rho_i reaches |lambda_i| can hide a
  // wrong-sign eigenvalue of size <= rho_i in their diagonal block: (sum of those rho_i^2)^(1/2) must be at
  // rounding level, <= WM_TOLG ||a||_F (near-zero eigenvalues keep rho_i at the floor of the S product).
  if (tid == 0) {
    ws->tr_eta[step] = eta / nA;
    ws->tr_rn[step] = rn / nA;
    ws->tr_ro[step] = ro / N;
    ws->tr_g[step] = sqrt(g2) / nA;
  }
  const bool cross_ok = eta <= WM_TOLE * nA;
  const bool orth_ok = a.wtest ? (rn <= WM_TOLE * nA && ro <= WM_TOLO * N) : ro <= 1e-14 * N;
  const bool conv = cross_ok && orth_ok && sqrt(g2) <= WM_TOLG * nA && isfinite(eta) &&
                    isfinite(rn) && isfinite(ro);
  // a coupling that stops halving while still above the tolerance means the update is not converging
  const bool stall = !isfinite(eta) || !isfinite(rn) || !isfinite(ro) || step == WM_MAXS - 1 ||
                     (step > 0 && !cross_ok && eta > 0.5 * ws->eta_prev);
  if (conv || stall || npairs > WM_PAIRS) {
    if (tid == 0) {
      ws->gate = 0;
      ws->eta = eta;
      ws->rn = rn;
      ws->step = step + 1;  // S evaluations of this iteration
      if (conv) {
        ws->status = 1;
        ws->cur = step & 1;
        ws->n_warm++;
        ws->n_steps += step;
        ws->fails = 0;
        wm_set(a.hfin, 1);
      } else {
        ws->status = 2;
        ws->fails++;
        ws->backoff = (1 << min(ws->fails, a.bo_cap)) - 1;
        ws->need_full = 0;
        ws->n_fail++;
        ws->n_steps += step;
        ws->why = (!isfinite(eta) || !isfinite(rn)) ? 4 : (stall ? (step == WM_MAXS - 1 ? 1 : 2) : 3);
        ws->pred_ok = 0;
        wm_set(a.hcold, 1);
      }
    }
    return;
  }
  if (npairs == 0) {  // no strong pair: every index is its own cluster
    for (int t = tid; t < N; t += T) a.cid[t] = -1;
    if (tid == 0) {
      ws->ncl = 0;
      ws->maxcl = 0;
      if (step == 0) ws->cl0 = 0;
      ws->eta_prev = eta;
      ws->eta = eta;
      ws->rn = rn;
      ws->step = step + 1;
      if (step + 1 < WM_MAXS) wm_set(a.hstep[step + 1], 1);
    }
    return;
  }
  // sorted order of lambda (rank by counting; ties by index: exact and deterministic)
  for (int t = tid; t < N; t += T) lam_s[t] = __ldcg(a.lam + t);
  __syncthreads();
  for (int i = tid; i < N; i += T) {
    const double ki = lam_s[i];
    int c0 = 0, c1 = 0;
    int jj = 0;
    for (; jj + 1 < N; jj += 2) {
      const double k0 = lam_s[jj], k1 = lam_s[jj + 1];
      c0 += (k0 < ki || (k0 == ki && jj < i)) ? 1 : 0;
      c1 += (k1 < ki || (k1 == ki && jj + 1 < i)) ? 1 : 0;
    }
    if (jj < N) c0 += (lam_s[jj] < ki || (lam_s[jj] == ki && jj < i)) ? 1 : 0;
    a.pos[i] = c0 + c1;
    a.order[c0 + c1] = i;
  }
  // link counters of the strong pairs over the sorted positions, then their prefix sums
  for (int t = tid; t < WM_SORT; t += T) cpre[t] = 0;
  __syncthreads();
  for (int k = tid; k < npairs; k += T) {
    const int pi = __ldcg(a.pos + a.pairs[2 * k]), pj = __ldcg(a.pos + a.pairs[2 * k + 1]);
    atomicAdd(&cpre[min(pi, pj)], 1);
    atomicAdd(&cpre[max(pi, pj)], -1);
  }
  for (int off = 1; off < WM_SORT; off <<= 1) {  // Hillis-Steele inclusive scan
    __syncthreads();
    int v[WM_SORT / T];
#pragma unroll
    for (int q = 0; q < WM_SORT / T; ++q) {
      const int t = tid + q * T;
      v[q] = t >= off ? cpre[t - off] : 0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < WM_SORT / T; ++q) cpre[tid + q * T] += v[q];
  }
  __syncthreads();
  // cpre[t] > 0: sorted position t is linked to t + 1
  for (int t = tid; t < N; t += T) {
    a.cid[a.order[t]] = -1;
    a.cpos[a.order[t]] = 0;
  }
  __syncthreads();
  for (int t = tid; t < N - 1; t += T) {
    if (cpre[t] > 0 && (t == 0 || cpre[t - 1] <= 0)) {  // start of a run of size >= 2
      int sz = 2;
      while (t + sz - 1 < N - 1 && cpre[t + sz - 1] > 0 && sz <= WM_CAP) ++sz;
      if (sz > WM_CAP) {
        atomicOr(&flags[1], 1);
        atomicMax(&flags[2], sz);
      } else {
        const int q = atomicAdd(&flags[0], 1);
        atomicMax(&flags[2], sz);
        a.cl_start[q] = t;
        a.cl_size[q] = sz;
        for (int u = 0; u < sz; ++u) {
          a.cid[a.order[t + u]] = q;
          a.cpos[a.order[t + u]] = u;
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (flags[1]) {
      ws->why = 3;
      ws->pred_ok = 0;
      ws->gate = 0;
      ws->status = 2;
      ws->fails++;
      ws->backoff = (1 << min(ws->fails, a.bo_cap)) - 1;
      ws->need_full = 0;
      ws->n_fail++;
      ws->n_steps += step;
      wm_set(a.hcold, 1);
      return;
    }
    int off = 0, rb = 0;
    for (int q = 0; q < flags[0]; ++q) {
      a.cl_voff[q] = off;
      a.cl_rbase[q] = rb;
      off += a.cl_size[q] * a.cl_size[q];
      rb += a.cl_size[q];
    }
    ws->ncl = flags[0];
    ws->maxcl = flags[2];
    if (flags[0] > 0) {
      wm_set(a.hclA, 1);
      wm_set(a.hclB, 1);
    }
    if (step == 0) ws->cl0 = flags[0] > 0;
    ws->eta_prev = eta;
    ws->eta = eta;
    ws->rn = rn;
    ws->step = step + 1;
    if (step + 1 < WM_MAXS) wm_set(a.hstep[step + 1], 1);
  }
}

// ---- per step: exact eigendecomposition of every cluster block S_CC (parallel-order Jacobi) ----
// grid WM_CLB, 256 threads, WM_CL_SMEM dynamic shared memory: A and V ping-pong (2 x 2 x WM_CAP x
// (WM_CAP + 1)).  A round: the cp/2 rotation parameters of the round-robin pairs (one thread each), then
// A' = J^T A J and V' = V J elementwise from the other buffer (each element reads the four entries of its
// two pairs): two barriers per round.  A sweep ends the solve once off(A)^2 <= (4 eps)^2 ||A||_F^2.
constexpr int WM_CLT = 1024;  // threads of the cluster kernel
constexpr size_t WM_CL_SMEM = 5 * sizeof(double) * WM_CAP * (WM_CAP + 1);
__global__ void __launch_bounds__(WM_CLT) k_warm_cluster(WarmArgs a) {
  if (wm_skip(a) || a.ws->gate != 1) return;
  extern __shared__ double wm_dyn[];
  typedef double Row[WM_CAP + 1];
  Row* Ab[2] = {reinterpret_cast<Row*>(wm_dyn), reinterpret_cast<Row*>(wm_dyn + WM_CAP * (WM_CAP + 1))};
  Row* Vb[2] = {reinterpret_cast<Row*>(wm_dyn + 2 * WM_CAP * (WM_CAP + 1)),
                reinterpret_cast<Row*>(wm_dyn + 3 * WM_CAP * (WM_CAP + 1))};
  __shared__ double cs[WM_CAP], sn[WM_CAP];  // per index: the rotation of its pair, signed for its role
  __shared__ int mate[WM_CAP];
  __shared__ int mem[WM_CAP];
  __shared__ double red[WM_CLT / 32];
  Row* Rc = reinterpret_cast<Row*>(wm_dyn + 4 * WM_CAP * (WM_CAP + 1));  // R_CC, then R_CC V
  const int tid = threadIdx.x, ncl = a.ws->ncl, ld = a.ldn;
  for (int q = blockIdx.x; q < ncl; q += gridDim.x) {
    const int c = a.cl_size[q], t0 = a.cl_start[q], voff = a.cl_voff[q];
    const int cp = (c + 1) & ~1;  // even player count (a dummy index never rotates)
    __syncthreads();
    for (int u = tid; u < c; u += WM_CLT) mem[u] = a.order[t0 + u];
    __syncthreads();
    double f2 = 0.0;
    for (int e = tid; e < cp * cp; e += WM_CLT) {
      const int u = e % cp, v = e / cp;
      const bool in = u < c && v < c;
      const double x = in ? wm_sym(a.S, ld, mem[u], mem[v]) : 0.0;
      Ab[0][u][v] = x;
      Vb[0][u][v] = u == v ? 1.0 : 0.0;
      Rc[u][v] = in ? (u == v ? 1.0 : 0.0) - wm_sym(a.P, ld, mem[u], mem[v]) : 0.0;
      f2 = fma(x, x, f2);
    }
    f2 = warp_sum(f2);
    if ((tid & 31) == 0) red[tid >> 5] = f2;
    __syncthreads();
    double fro2 = 0.0;
    for (int w = 0; w < WM_CLT / 32; ++w) fro2 += red[w];
    int cur = 0;
    for (int sweep = 0; sweep < 30; ++sweep) {
      Row* A = Ab[cur];
      double o2 = 0.0;
      for (int e = tid; e < cp * cp; e += WM_CLT) {
        const int u = e % cp, v = e / cp;
        if (u != v) o2 = fma(A[u][v], A[u][v], o2);
      }
      o2 = warp_sum(o2);
      __syncthreads();
      if ((tid & 31) == 0) red[tid >> 5] = o2;
      __syncthreads();
      double off2 = 0.0;
      for (int w = 0; w < WM_CLT / 32; ++w) off2 += red[w];
      if (off2 <= 2e-30 * fro2) break;
      for (int r = 0; r < cp - 1; ++r) {
        Row* Ao = Ab[cur];
        Row* Vo = Vb[cur];
        Row* An = Ab[cur ^ 1];
        Row* Vn = Vb[cur ^ 1];
        if (tid < cp / 2) {  // round-robin pair of round r
          const int M = cp - 1, k = tid;
          int p, qv;
          if (k == 0) {
            p = M;
            qv = r % M;
          } else {
            p = (r + k) % M;
            qv = (r - k + M) % M;
          }
          if (p > qv) {
            const int tmp = p;
            p = qv;
            qv = tmp;
          }
          const double apq = Ao[p][qv], app = Ao[p][p], aqq = Ao[qv][qv];
          double cc = 1.0, ss = 0.0;
          if (fabs(apq) > 1e-300) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            cc = 1.0 / sqrt(1.0 + t * t);
            ss = t * cc;
          }
          // column p' = c col_p - s col_q, column q' = s col_p + c col_q
          cs[p] = cc;
          sn[p] = -ss;
          mate[p] = qv;
          cs[qv] = cc;
          sn[qv] = ss;
          mate[qv] = p;
        }
        __syncthreads();
        // A' = J^T A J, V' = V J: entry (u, v) from the 2 x 2 blocks of u's and v's pairs
        for (int e = tid; e < cp * cp; e += WM_CLT) {
          const int u = e % cp, v = e / cp;
          const int uu = mate[u], vv = mate[v];
          const double cu = cs[u], su = sn[u], cv = cs[v], sv = sn[v];
          // (J^T A)_{u, .} = c_u A_{u, .} + s_u A_{uu, .} ; then (.. J)_{., v} = c_v (.)_{., v} + s_v (.)_{., vv}
          const double r0 = fma(cu, Ao[u][v], su * Ao[uu][v]);
          const double r1 = fma(cu, Ao[u][vv], su * Ao[uu][vv]);
          An[u][v] = fma(cv, r0, sv * r1);
          Vn[u][v] = fma(cv, Vo[u][v], sv * Vo[u][vv]);
        }
        cur ^= 1;
        __syncthreads();
      }
    }
    Row* A = Ab[cur];
    Row* V = Vb[cur];
    // rotated eigenvalue estimates lambda~_u = mu_u / (1 - R~_uu), R~ = V^T R V, R = I - P:
    // RV = R_CC V into the free ping-pong buffer, then R~_uu = sum_t V[t][u] RV[t][u]
    Row* RV = Ab[cur ^ 1];
    __syncthreads();
    for (int e = tid; e < c * c; e += WM_CLT) {
      const int t = e % c, u = e / c;
      double x = 0.0;
      for (int t2 = 0; t2 < c; ++t2) x = fma(Rc[t][t2], V[t2][u], x);
      RV[t][u] = x;
    }
    __syncthreads();
    for (int u = tid; u < c; u += WM_CLT) {
      double ruu = 0.0;
      for (int t = 0; t < c; ++t) ruu = fma(V[t][u], RV[t][u], ruu);
      a.lamt[mem[u]] = A[u][u] / (1.0 - ruu);
    }
    for (int e = tid; e < c * c; e += WM_CLT) {
      const int t = e % c, u = e / c;
      a.Vcl[voff + e] = V[t][u];  // column u: eigenvector u over the members t
    }
  }
}

// ---- per step: rotated rows of the cluster members, (V_C^T S)[u, j] and (V_C^T R)[u, j] for every j ----
// grid (nt, ncl capped), 256 threads = 32 columns x 8 row groups; S and P are stored full (mirrored), so
// row m of S is column m: coalesced along j.
__global__ void __launch_bounds__(256) k_warm_rot(WarmArgs a) {
  if (wm_skip(a) || a.ws->gate != 1) return;
  __shared__ double Vs[WM_CAP * WM_CAP];
  __shared__ int mem[WM_CAP];
  const int ncl = a.ws->ncl, N = a.N, ld = a.ldn;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = 32 * blockIdx.x + tx;
  for (int q = blockIdx.y; q < ncl; q += gridDim.y) {
    const int c = a.cl_size[q], rb = a.cl_rbase[q];
    __syncthreads();
    for (int e = threadIdx.x; e < c * c; e += 256) Vs[e] = a.Vcl[a.cl_voff[q] + e];
    for (int u = threadIdx.x; u < c; u += 256) mem[u] = a.order[a.cl_start[q] + u];
    __syncthreads();
    if (j >= N) continue;
    double sr[WM_CAP / 8], rr[WM_CAP / 8];
#pragma unroll
    for (int k = 0; k < WM_CAP / 8; ++k) sr[k] = rr[k] = 0.0;
    for (int t = 0; t < c; ++t) {
      const int m = mem[t];
      const double sv = a.S[(size_t)m * ld + j];
      const double rv = (m == j ? 1.0 : 0.0) - a.P[(size_t)m * ld + j];
#pragma unroll
      for (int k = 0; k < WM_CAP / 8; ++k) {
        const int u = ty + 8 * k;
        if (u < c) {
          const double v = Vs[t + u * c];
          sr[k] = fma(v, sv, sr[k]);
          rr[k] = fma(v, rv, rr[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < WM_CAP / 8; ++k) {
      const int u = ty + 8 * k;
      if (u < c) {
        a.Srot[(size_t)(rb + u) * ld + j] = sr[k];
        a.Rrot[(size_t)(rb + u) * ld + j] = rr[k];
      }
    }
  }
}

// coefficient list of rotated index i over the old basis: (members, V column) or the unit vector
struct WmCo {
  int n;
  const int* mem;  // order + cl_start (members in sorted order)
  const double* v; // V column (n entries), null = 1
  int self;
};
__device__ __forceinline__ WmCo wm_coef(const WarmArgs& a, int i) {
  WmCo r;
  const int q = a.cid[i];
  if (q < 0) {
    r.n = 1;
    r.mem = nullptr;
    r.v = nullptr;
    r.self = i;
  } else {
    const int c = a.cl_size[q];
    r.n = c;
    r.mem = a.order + a.cl_start[q];
    r.v = a.Vcl + a.cl_voff[q] + (size_t)a.cpos[i] * c;
    r.self = i;
  }
  return r;
}

// ---- per step: E (rotated basis), full N x N; grid (nt, nt), 256 threads ----
// The 32 x 32 tile of S and P a CTA needs is staged through shared memory; pairs involving a cluster
// member take the general path (global reads along the cluster's member columns).
__global__ void __launch_bounds__(256) k_warm_E(WarmArgs a) {
  if (wm_skip(a) || a.ws->gate != 1) return;
  __shared__ double St[32][33], Pt[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, N = a.N, ld = a.ldn;
  const int ti = blockIdx.x, tj = blockIdx.y;
  // stage: St[r][c] = S(32 ti + c, 32 tj + r) (full symmetric storage: straight column reads)
  for (int r = ty; r < 32; r += 8) {
    const int i = 32 * ti + tx, j = 32 * tj + r;
    double sv = 0.0, pv = 0.0;
    if (i < N && j < N) {
      sv = a.S[(size_t)j * ld + i];
      pv = a.P[(size_t)j * ld + i];
    }
    St[r][tx] = sv;
    Pt[r][tx] = pv;
  }
  __syncthreads();
  const int i = 32 * ti + tx;
  if (i >= N) return;
  const int qi = a.cid[i];
  const double li = qi >= 0 ? a.lamt[i] : a.lam[i];
  // no clusters this step: V = I, so M = I + E is written here and k_warm_M has nothing to do
  const bool direct = a.ws->ncl == 0;
  double* out = direct ? a.Mm : a.E;
  for (int r = ty; r < 32; r += 8) {
    const int j = 32 * tj + r;
    if (j >= N) break;
    const int qj = a.cid[j];
    double e;
    if (qi < 0 && qj < 0) {  // both singletons: S~ = S, R~ = R
      const double rt = (i == j ? 1.0 : 0.0) - Pt[r][tx];
      if (i == j) {
        e = 0.5 * rt;
      } else {
        const double lj = a.lam[j];
        const double d = lj - li;
        e = d != 0.0 ? fma(lj, rt, St[r][tx]) / d : 0.5 * rt;
      }
    } else {
      // rotated rows: slot of a cluster member = its cluster's row base + its position in the cluster
      const bool same = (i == j) || (qi >= 0 && qi == qj);
      double st = 0.0, rt = 0.0;
      if (qi >= 0 && qj < 0) {         // S~_ij = (V^T S)[i, j]
        const size_t si = (size_t)(a.cl_rbase[qi] + a.cpos[i]) * ld;
        st = a.Srot[si + j];
        rt = a.Rrot[si + j];
      } else if (qi < 0 && qj >= 0) {  // S~_ij = S~_ji = (V^T S)[j, i]
        const size_t sj = (size_t)(a.cl_rbase[qj] + a.cpos[j]) * ld;
        st = a.Srot[sj + i];
        rt = a.Rrot[sj + i];
      } else {                         // both in clusters: S~_ij = sum_t (V^T S)[i, m_t] V_C(j)[t, u_j]
        const size_t si = (size_t)(a.cl_rbase[qi] + a.cpos[i]) * ld;
        const int c = a.cl_size[qj];
        const int* mem = a.order + a.cl_start[qj];
        const double* vj = a.Vcl + a.cl_voff[qj] + (size_t)a.cpos[j] * c;
        for (int t = 0; t < c; ++t) {
          const int m = mem[t];
          if (!same) st = fma(a.Srot[si + m], vj[t], st);
          rt = fma(a.Rrot[si + m], vj[t], rt);
        }
      }
      if (same) {
        e = 0.5 * rt;
      } else {
        const double lj = qj >= 0 ? a.lamt[j] : a.lam[j];
        const double d = lj - li;
        e = d != 0.0 ? fma(lj, rt, st) / d : 0.5 * rt;
      }
    }
    out[(size_t)j * ld + i] = direct ? (i == j ? 1.0 : 0.0) + e : e;
    if (direct && a.predict) a.Esum[(size_t)j * ld + i] += e;
  }
}

// ---- per step: M = V (I + E); grid (nt, nt), 256 threads ----
__global__ void __launch_bounds__(256) k_warm_M(WarmArgs a) {
  if (wm_skip(a) || a.ws->gate != 1 || a.ws->ncl == 0) return;  // (ncl == 0: k_warm_E wrote M)
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, N = a.N, ld = a.ldn;
  const int ai = 32 * blockIdx.x + tx;
  if (ai >= N) return;
  const int q = a.cid[ai];
  for (int r = ty; r < 32; r += 8) {
    const int j = 32 * blockIdx.y + r;
    if (j >= N) break;
    double m;
    if (q < 0) {
      m = (ai == j ? 1.0 : 0.0) + a.E[(size_t)j * ld + ai];
    } else {
      const int c = a.cl_size[q];
      const int* mem = a.order + a.cl_start[q];
      const double* vr = a.Vcl + a.cl_voff[q] + a.cpos[ai];  // row cpos(ai) of V_C: stride c
      m = 0.0;
      for (int u = 0; u < c; ++u) {
        const int mu = mem[u];
        m = fma(vr[(size_t)u * c], (mu == j ? 1.0 : 0.0) + a.E[(size_t)j * ld + mu], m);
      }
    }
    a.Mm[(size_t)j * ld + ai] = m;
    if (a.predict) a.Esum[(size_t)j * ld + ai] += m - (ai == j ? 1.0 : 0.0);
  }
}

// ---- end of the cold path: which tail runs (full re-seed + finish, or the partial-spectrum recon) ----
__global__ void k_warm_cold_switch(WarmArgs a) {
  if (wm_skip(a)) return;
  a.ws->n_cold++;
  if (a.ws->need_full) wm_set(a.hfull, 1);
  else wm_set(a.hpart, 1);
}

// ---- finish: side selection (warm S or cold eigenpairs), compact index list ----
__global__ void __launch_bounds__(WM_NT) k_warm_select(WarmArgs a, int block_id) {
  if (wm_skip(a)) return;
  __shared__ int cnt[WM_NT / 32 + 1];
  __shared__ int np_s, nn_s;
  WarmState* ws = a.ws;
  const int N = a.N, tid = threadIdx.x;
  const int src = ws->status == 1 ? 0 : 1;
  const double* lam = src == 0 ? a.lam : a.lam_cold;
  if (tid == 0) {
    np_s = 0;
    nn_s = 0;
  }
  __syncthreads();
  int p = 0, n = 0;
  for (int i = tid; i < N; i += WM_NT) {
    p += lam[i] > 0.0;
    n += lam[i] < 0.0;
  }
  atomicAdd(&np_s, p);
  atomicAdd(&nn_s, n);
  __syncthreads();
  const int side = np_s <= nn_s ? 0 : 1;
  // compact list of the chosen side's indices, ascending (block scan over chunks of WM_NT)
  int base = 0;
  for (int c0 = 0; c0 < N; c0 += WM_NT) {
    const int i = c0 + tid;
    const bool f = i < N && (side == 0 ? lam[i] > 0.0 : lam[i] < 0.0);
    const unsigned b = __ballot_sync(0xffffffffu, f);
    const int w = tid >> 5, l = tid & 31;
    __syncthreads();
    if (l == 0) cnt[w] = __popc(b);
    __syncthreads();
    if (tid == 0) {
      int s = 0;
      for (int q = 0; q < WM_NT / 32; ++q) {
        const int x = cnt[q];
        cnt[q] = s;
        s += x;
      }
      cnt[WM_NT / 32] = s;
    }
    __syncthreads();
    if (f) a.idx[base + cnt[w] + __popc(b & ((1u << l) - 1u))] = i;
    base += cnt[WM_NT / 32];
  }
  if (tid == 0) {
    a.sel[0] = base;
    a.sel[1] = 0;
    a.sel[2] = side;
    a.side[block_id] = side;
    ws->src = src;
    ws->p_valid = src == 0;  // a certified warm X keeps its P (X1 is copied to X0 bit for bit)
    // its rotation generator (Esum) predicts the next iteration's start -- only while the trajectory is
    // smooth: a cluster at step 0 (near-degenerate eigenvalues moving) or more evaluations than the
    // unpredicted steady state switch the predictor off until an iteration converges quickly again
    ws->pred_ok = src == 0 && !ws->cl0 && ws->step <= (ws->pred ? 3 : 4);
    if (src == 1) {
      ws->valid = 1;  // X0 = the cold path's eigenvectors
      ws->cur = 0;
      ws->n_seed++;
    }
  }
}

// ---- finish: Xs = X[:, idx] (into Mm), Ss = +-S[idx, idx] or +-diag(lambda) (into E), X1 -> X0 ----
// grid >= 148, 256 threads
__global__ void __launch_bounds__(256) k_warm_gather(WarmArgs a) {
  if (wm_skip(a)) return;
  const WarmState* ws = a.ws;
  const int N = a.N, ld = a.ldn, r = a.sel[0], side = a.sel[2], src = ws->src;
  const double sg = side ? -1.0 : 1.0;
  const double* X = (src == 0 && ws->cur == 1) ? a.X1 : a.X0;
  const long long n1 = (long long)N * r, n2 = (long long)r * r;
  const long long n3 = (src == 0 && ws->cur == 1) ? (long long)N * N : 0;
  const long long tot = n1 + n2 + n3;
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < tot; e += (long long)gridDim.x * 256) {
    if (e < n1) {
      const int row = (int)(e % N), t = (int)(e / N);
      a.Mm[(size_t)t * ld + row] = X[(size_t)a.idx[t] * ld + row];
    } else if (e < n1 + n2) {
      const long long f = e - n1;
      const int t = (int)(f % r), u = (int)(f / r);
      double v;
      if (src == 0) v = sg * wm_sym(a.S, ld, a.idx[t], a.idx[u]);
      else v = t == u ? sg * a.lam_cold[a.idx[t]] : 0.0;
      a.E[(size_t)u * ld + t] = v;
    } else {
      const long long f = e - n1 - n2;
      const int row = (int)(f % N), col = (int)(f / N);
      a.X0[(size_t)col * ld + row] = a.X1[(size_t)col * ld + row];
    }
  }
}
