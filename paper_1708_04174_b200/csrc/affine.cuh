// Affine-projection kernels: u_hat = (I + Q)^{-1}(u + v) with partial orthogonality.
//
// PAPER.md P:426-446 (tau elimination + rank-one SMW with cached h = M^{-1} zeta)
// (sigma_1 elimination: (I + A A^T) sigma_2 = w2 - A w1), P:469-480 (Woodbury with P = I + D
// diagonal, D = A_orth A_orth^T, Proposition 1) and the Appendix op list P:870-877.
//
// Elimination order (reading C15): the linear system is solved as
//   q = M^{-1} w_12 (partial orthogonality + Woodbury, with r = w_12),
//   u_hat_3 = (w3 + zeta^T q) / (1 + zeta^T h),   u_hat_12 = q - u_hat_3 h,   h = M^{-1} zeta cached,
// which is E:MatrixInverse / E:MatrixInverseResult reassociated: rows 1-2 of (I+Q)u = w
// read M u_12 + zeta u_3 = w_12 and row 3 reads u_3 - zeta^T u_12 = w3.  It avoids subtracting two
// vectors ~1/tau larger than the result (p - coef h) when tau << 1.
//
// Data flow per iteration:
//   k_gather   (rows)     : g = A w1, x = P^{-1}(w2 - g), partial b^T x; residual partials of u^k
//   k_lowT     (t' cols)  : y_t = A_low^T x, A_low^T y
//   k_kinv     (t' rows)  : z_t = K^{-1} y_t         (K = I + A_low^T P^{-1} A_low)
//   k_tphase   (1 CTA)    : residuals/termination of u^k (reading C9); coef, u_hat_low, u_hat_3,
//                           tau/kappa update, free columns (A_low^T sigma_2 = z_t by the Woodbury
//                           identity, b^T sigma_2 = b^T x - (A_low^T P^{-1} b)^T z_t)
//   k_rowupdate(rows)     : sigma_2 = x - P^{-1} A_low z_t, u_hat_2 = sigma_2 - coef h_2, y, s update
//   k_scatter  (svec pos) : a = u_hat_xi - z (= xi + A_orth^T u_hat_2 on orthogonal columns), into the
//                           per-block symmetric matrices (input of the PSD projection)
//   k_pack     (svec pos) : xi = svec(Pi(a)), z = xi - a (Moreau); commit tau, kappa, k
#pragma once
#include "common.cuh"

struct AffineArgs {
  int m, n, t_free, tl, npsd;
  // orthogonal columns, grouped by row (CSR of A_orth)
  const int* seg_ptr;
  const int* seg_col;
  const double* seg_val;
  // alpha-ordered copies of xi and z on the orthogonal columns (entry e of the CSR = column seg_col[e]),
  // maintained by k_pack so the gather streams its segments contiguously; segpos[col] = e (-1: none)
  double* xis;
  double* zs;
  const int* segpos;
  // A_low: columns low_col[j]; CSR (rows) and CSC (low columns)
  const int* low_col;
  const int* lr_ptr;
  const int* lr_idx;
  const int* lr_col;   // low_col[lr_idx[e]] (the gather's direct column index)
  int row_lanes;       // k_rowupdate lanes per row: 8 when some row has >= 16 low-rank entries, else 1
  int fuse_low;        // 1: k_tphase forms A_low^T x and K^{-1} y_t itself (t' <= FUSE_LOW_TL, few entries): two launches less
  const double* lr_val;
  const int* lc_ptr;
  const int* lc_row;
  const double* lc_val;
  const double* c_low;
  const double* h1_low;
  const double* beta_low;
  const double* Kinv;  // tl x tl, symmetric, row i at Kinv + i * ldk (ldk = tl rounded up to even:
  int ldk;             //   16-byte aligned column pairs for the tile apply)
  const int* empty_cols;
  int n_empty;
  // row data
  const double* b;
  const double* Pinv;
  const double* h2;
  double denom, bh2, nb, nc;
  // per-column data (size n): code >= 0 orth row, -1 empty orth column, <= -2 low index (-2 - j)
  const int* code;
  const double* aval;
  // state
  double* xi;
  double* z;
  double* y;
  double* s;
  DevState* st;
  IterScal* is;
  // scratch
  double* x;
  double* uhat2;
  double* yt;
  double* zt;
  double* ulow;
  double* aty;
  double* part;
  int gather_blocks;
  double* kpart;  // symmetric K^{-1} apply (tl >= KINV_SYM_MIN): nt x nt x KT per-tile partials
  double* hist;   // residual history: slot k mod SOS_HIST = (k, pres, dres, gap, pobj) of u^k (k_tphase)
  double* asvec;  // PSD part of u_hat_xi - z (size npsd)
  // PSD blocks
  int nblk;
  const long long* blk_col;   // first column of block b
  const int* blk_N;
  const long long* blk_mat;   // offset of block b's N x N matrix in mats
  double* mats;
  const int* cta_blk;         // position-parallel kernels: CTA -> (block, first local svec index)
  const long long* cta_q0;
  int pos_ctas;
  const int* side;            // per block: 1 = matrix holds Pi(-a) = Pi(a) - a (large-block path)
  const double* shard_scal;   // sharded mode (shard.cuh): all-reduced [orth dual, low dual, low dual0]
};

constexpr int GATHER_NT = 256;
constexpr int SOS_HIST = 1024;  // residual history ring (sosadmm_residual_history)
constexpr int POS_NT = 256;
constexpr int POS_PER_CTA = 1024;

// ---------------------------------------------------------------------------------------------
// k_gather: one thread per row alpha.
//   g_alpha  = sum_{orth j in seg(alpha)} A_{alpha j}(xi_j + z_j) + sum_{low j} A_{alpha j} r1_j
//              (r1 = w1 - c w3 with w1 = xi + z; c vanishes on orthogonal columns)
//   x_alpha  = (y_alpha + s_alpha + b_alpha w3 - g_alpha) / P_alpha
// and, for the residuals of u^k (reading C9), (A xi)_alpha and sum_{j in seg(alpha)} (A^T y + z)_j^2.
__global__ void __launch_bounds__(GATHER_NT) k_gather(AffineArgs a) {
  __shared__ double sh[6 * (GATHER_NT / 32)];
  if (a.st->done) return;
  const double tau = a.st->tau;
  const int r = blockIdx.x * GATHER_NT + threadIdx.x;
  double p_pres = 0, p_axi = 0, p_dres = 0, p_by = 0;
  dd bxd{0.0, 0.0};
  if (r < a.m) {
    // the row's scalars first (independent loads in flight together with the segment's)
    const double yr = a.y[r], sr = a.s[r], br = a.b[r], pinv = a.Pinv[r];
    double gx = 0.0, gz = 0.0, dres = 0.0;
    const int e0 = a.seg_ptr[r], e1 = a.seg_ptr[r + 1];
    for (int e = e0; e < e1; ++e) {  // alpha-ordered copies: row r's segment is contiguous
      const double v = a.seg_val[e];
      const double xj = a.xis[e], zj = a.zs[e];
      gx = fma(v, xj, gx);
      gz = fma(v, zj, gz);
      const double d = fma(v, yr, zj);
      dres = fma(d, d, dres);
    }
    double gl = 0.0, axl = 0.0;
    const int l0 = a.lr_ptr[r], l1 = a.lr_ptr[r + 1];
#pragma unroll 4
    for (int e = l0; e < l1; ++e) {
      const int j = a.lr_col[e];
      const double v = a.lr_val[e];
      const double xj = a.xi[j];
      const double r1 = xj + a.z[j];  // w1 on the low columns (q = M^{-1} w_12, reading C15)
      gl = fma(v, r1, gl);
      axl = fma(v, xj, axl);
    }
    const double g = (gx + gz) + gl;
    const double r2 = yr + sr;  // w2
    const double xr = (r2 - g) * pinv;
    a.x[r] = xr;
    const double axi = gx + axl;
    const double pr = axi - br * tau;
    bxd = dd_prod(br, xr);
    p_pres = pr * pr;
    p_axi = axi * axi;
    p_dres = dres;
    p_by = br * yr;
  }
  gather_part_sums<GATHER_NT>(bxd, p_pres, p_axi, p_dres, p_by, sh, a.part, a.gather_blocks, blockIdx.x, false, 0.0);
}

// One warp, low column j:  y_t[j] = (A_low^T x)_j,  aty[j] = (A_low^T y)_j.
__device__ __forceinline__ void lowT_column(const AffineArgs& a, int j, int lane) {
  double sx = 0.0, sy = 0.0;
  for (int e = a.lc_ptr[j] + lane; e < a.lc_ptr[j + 1]; e += 32) {
    const int r = a.lc_row[e];
    const double v = a.lc_val[e];
    sx = fma(v, a.x[r], sx);
    sy = fma(v, a.y[r], sy);
  }
  sx = warp_sum(sx);
  sy = warp_sum(sy);
  if (lane == 0) {
    a.yt[j] = sx;
    a.aty[j] = sy;
  }
}

// One warp, row i:  z_t[i] = sum_j Kinv[i, j] y_t[j]  (P:874 with the cached factor applied as an
// explicit SPD inverse; K symmetric so row i = column i).
__device__ __forceinline__ void kinv_row(const AffineArgs& a, int i, int lane) {
  const double* row = a.Kinv + (size_t)i * a.ldk;
  double acc = 0.0;
  for (int j = lane; j < a.tl; j += 32) acc = fma(row[j], a.yt[j], acc);
  acc = warp_sum(acc);
  if (lane == 0) a.zt[i] = acc;
}

// k_lowT: one warp per low column.
__global__ void __launch_bounds__(256) k_lowT(AffineArgs a) {
  if (a.st->done) return;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= a.tl) return;
  lowT_column(a, wid, lane);
}

// k_kinv: one warp per row.
__global__ void __launch_bounds__(256) k_kinv(AffineArgs a) {
  if (a.st->done) return;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= a.tl) return;
  kinv_row(a, wid, lane);
}

// Symmetric K^{-1} apply for large t' (config 3: t' = 7,801, K^{-1} = 487 MB, HBM-bound): read only
// the tiles on and below the diagonal (half the bytes).  Tile (I, J), I >= J, of KT x KT contributes
// K_IJ y_J to block I and, when I > J, K_IJ^T y_I = K_JI y_I to block J; the first is stored at
// kpart[I][J], the second at kpart[J][I], so z_I = sum_J kpart[I][J] in fixed J order (k_kinv_sum):
// deterministic, no atomics.
constexpr int KT = 64;
constexpr int KINV_SYM_MIN = 2048;  // below it K^{-1} (<= 32 MB) is L2-resident: one warp per row
__global__ void __launch_bounds__(256) k_kinv_tiles(AffineArgs a) {
  if (a.st->done) return;
  __shared__ double rsum[KT];      // row partials (each warp owns whole rows)
  __shared__ double csum[8][KT];   // column partials of the eight warps
  const int nt = (a.tl + KT - 1) / KT;
  const int bidx = blockIdx.x;
  int I = (int)((sqrt(8.0 * bidx + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= bidx) ++I;
  while (I * (I + 1) / 2 > bidx) --I;
  const int J = bidx - I * (I + 1) / 2;
  // lane l owns the column pair (2l, 2l + 1) of the tile (one 16-byte load per row), warp w the rows
  // w, w + 8, ..., w + 56
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int jc = J * KT + 2 * lane;
  const bool c0 = jc < a.tl, c1 = jc + 1 < a.tl;
  const double yj0 = c0 ? a.yt[jc] : 0.0, yj1 = c1 ? a.yt[jc + 1] : 0.0;
  double2 kv[KT / 8];
#pragma unroll
  for (int u = 0; u < KT / 8; ++u) {  // all loads first: 8 independent 16-byte loads in flight
    const int i = I * KT + w + 8 * u;
    kv[u] = (c0 && i < a.tl) ? __ldcs(reinterpret_cast<const double2*>(a.Kinv + (size_t)i * a.ldk + jc))
                             : make_double2(0.0, 0.0);
    if (!c1) kv[u].y = 0.0;  // the padding column of an odd t'
  }
  double ca0 = 0.0, ca1 = 0.0, v[KT / 8];
#pragma unroll
  for (int u = 0; u < KT / 8; ++u) {
    const int i = I * KT + w + 8 * u;
    const double yi = i < a.tl ? a.yt[i] : 0.0;
    ca0 = fma(kv[u].x, yi, ca0);
    ca1 = fma(kv[u].y, yi, ca1);
    v[u] = fma(kv[u].x, yj0, kv[u].y * yj1);
  }
  // the 8 row sums over the warp's 32 lanes by a halving butterfly: at offset o the lanes with bit o
  // set keep the upper half of their values and receive the partner's upper half, so lane L ends
  // with row u(L) = bits (16, 8, 4) of L, then the last two xor steps complete the sums
#pragma unroll
  for (int n = KT / 8, o = 16; n > 1; n >>= 1, o >>= 1) {
    const bool hi = lane & o;
#pragma unroll
    for (int u = 0; u < n / 2; ++u) {
      const double send = hi ? v[u] : v[u + n / 2];
      const double keep = hi ? v[u + n / 2] : v[u];
      v[u] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  if ((lane & 3) == 0) {
    const int u = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    rsum[w + 8 * u] = v[0];
  }
  csum[w][2 * lane] = ca0;
  csum[w][2 * lane + 1] = ca1;
  __syncthreads();
  if (tid < KT) {
    a.kpart[((size_t)I * nt + J) * KT + tid] = rsum[tid];
  } else if (tid < 2 * KT && I != J) {
    const int cc = tid - KT;
    a.kpart[((size_t)J * nt + I) * KT + cc] = ((csum[0][cc] + csum[1][cc]) + (csum[2][cc] + csum[3][cc])) +
                                              ((csum[4][cc] + csum[5][cc]) + (csum[6][cc] + csum[7][cc]));
  }
}

// one CTA per output block I: thread (r, q) sums the partials J = q, q + 4, ... of row r (loads
// issued 8 at a time), the four chains combined in a fixed order
__global__ void __launch_bounds__(256) k_kinv_sum(AffineArgs a) {
  if (a.st->done) return;
  __shared__ double ps[4][KT];
  const int nt = (a.tl + KT - 1) / KT, I = blockIdx.x, r = threadIdx.x & (KT - 1), q = threadIdx.x >> 6;
  const double* p = a.kpart + (size_t)I * nt * KT + r;
  double acc = 0.0;
  int J = q;
  for (; J + 28 < nt; J += 32) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = p[(size_t)(J + 4 * u) * KT];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += t[u];
  }
  for (; J < nt; J += 4) acc += p[(size_t)J * KT];
  ps[q][r] = acc;
  __syncthreads();
  const int i = I * KT + threadIdx.x;
  if (threadIdx.x < KT && i < a.tl) a.zt[i] = (ps[0][threadIdx.x] + ps[1][threadIdx.x]) + (ps[2][threadIdx.x] + ps[3][threadIdx.x]);
}

// k_tphase: single CTA.  mode 0 = full iteration, 1 = check-only (residuals of u^k, no update),
// 2 = affine-only (unit entry point: no termination logic, no writes to xi/z).
constexpr int TP_NT = 512;
constexpr int FUSE_LOW_TL = 16;     // a.fuse_low: t' <= 16 and nnz(A_low) <= 4096 (configs 0, 1, 4: t' = 1), so
constexpr int FUSE_LOW_NNZ = 4096;  //   this CTA's 16 warps do k_lowT's and k_kinv's work (the same warp sums: same bits)
__global__ void __launch_bounds__(TP_NT) k_tphase(AffineArgs a, int mode) {
  __shared__ double bc[10];
  DevState* st = a.st;
  if (st->done) return;
  const int tid = threadIdx.x;
  if (a.fuse_low) {
    const int w = tid >> 5, lane = tid & 31;
    if (w < a.tl) lowT_column(a, w, lane);
    __syncthreads();  // y_t (global) written by this CTA's warps, read by them below
    if (w < a.tl) kinv_row(a, w, lane);
    __syncthreads();
  }
  // 1. fixed-order reductions of the gather partials (b^T x in double-double) and of the low-column
  //    sums: the trees of block_sum / dd_block_sum (per-warp shuffle tree, then the warp partials in
  //    warp order — the same bits), all values at once behind ONE barrier (the loads issued together)
  constexpr int NW = TP_NT / 32;
  __shared__ double shp[7][NW], shd[2][NW];
  const int gb = a.gather_blocks;
  double vals[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // PRES, AXI, DRES, BY, c^T xi, dl, dl0
  dd bxv{0.0, 0.0};
  for (int i = tid; i < gb; i += TP_NT) {
#pragma unroll
    for (int q = 0; q < 4; ++q) vals[q] += a.part[(PART_PRES + q) * gb + i];
    bxv = dd_add(bxv, dd{a.part[PART_BX * gb + i], a.part[PART_BXLO * gb + i]});
  }
  // low / free columns: c^T xi, dual residual of low columns, (A_low xi part already in gather)
  const double tau = st->tau, kappa = st->kappa, w3 = tau + kappa;
  const bool sharded = a.shard_scal != nullptr;  // low-column dual sums arrive all-reduced
  for (int j = tid; j < a.tl; j += TP_NT) {
    const int col = a.low_col[j];
    const double cj = a.c_low[j];
    vals[4] = fma(cj, a.xi[col], vals[4]);  // c vanishes off the (replicated) free columns
    if (!sharded) {
      const double d0 = a.aty[j] + a.z[col];
      const double d = d0 - cj * tau;
      vals[5] = fma(d, d, vals[5]);
      vals[6] = fma(d0, d0, vals[6]);
    }
  }
  if (!sharded)
    for (int j = tid; j < a.n_empty; j += TP_NT) {
      const double zj = a.z[a.empty_cols[j]];
      vals[5] = fma(zj, zj, vals[5]);
      vals[6] = fma(zj, zj, vals[6]);
    }
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vals[q] += __shfl_down_sync(0xffffffffu, vals[q], o);
  bxv = dd_warp_sum(bxv);
  {
    const int w = tid >> 5, l = tid & 31;
    if (l == 0) {
#pragma unroll
      for (int q = 0; q < 7; ++q) shp[q][w] = vals[q];
      shd[0][w] = bxv.hi;
      shd[1][w] = bxv.lo;
    }
  }
  __syncthreads();
  if (tid < 7) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < NW; ++i) r += shp[tid][i];
    const int slot = tid < 4 ? PART_PRES + tid : 3 + tid;  // bc[1..4] parts, bc[7..9] low sums
    bc[slot] = (sharded && tid >= 5) ? a.shard_scal[tid - 4] : r;
  } else if (tid == 32) {
    dd r{0.0, 0.0};
    for (int i = 0; i < NW; ++i) r = dd_add(r, dd{shd[0][i], shd[1][i]});
    bc[PART_BX] = r.hi;
    bc[PART_BXLO] = r.lo;
  }
  __syncthreads();
  double sums[NPART];
  for (int k = 0; k < NPART; ++k) sums[k] = bc[k];
  const double cx = bc[7], dl = bc[8], dl0 = bc[9];

  // 2. residuals of u^k and the termination rule (reading C9)
  if (mode != 2 && tid == 0) {
    const double by = sums[PART_BY];
    const double nATyz = sqrt(sums[PART_DRES] + dl0);  // ||A^T y + z|| (certificate test)
    const double nAxi = sqrt(sums[PART_AXI]);
    const double pinf = (by > 0.0) ? nATyz / by : INFINITY;
    const double dinf = (cx < 0.0) ? nAxi / (-cx) : INFINITY;
    double pres = INFINITY, dres = INFINITY, gap = INFINITY, pobj = NAN, dobj = NAN;
    if (tau > 0.0) {
      pres = sqrt(sums[PART_PRES]) / tau / (1.0 + a.nb);
      pobj = cx / tau;
      dobj = by / tau;
      gap = fabs(pobj - dobj) / (1.0 + fabs(pobj) + fabs(dobj));
    }
    // ||A^T y + z - c tau||: c vanishes on orthogonal columns, dl holds the low columns
    if (tau > 0.0) dres = sqrt(sums[PART_DRES] + dl) / tau / (1.0 + a.nc);
    st->res_pri = pres;
    st->res_dual = dres;
    st->res_gap = gap;
    st->pobj = pobj;
    if (a.hist && mode == 0) {  // the residuals of u^k, k = st->iter, in the history ring
      double* hq = a.hist + 5 * (size_t)(st->iter % SOS_HIST);
      hq[0] = (double)st->iter;
      hq[1] = pres;
      hq[2] = dres;
      hq[3] = gap;
      hq[4] = pobj;
    }
    st->dobj = dobj;
    st->pinf = pinf;
    st->dinf = dinf;
    int status = 0;
    const bool bad = !(isfinite(sums[PART_PRES]) && isfinite(sums[PART_DRES]) && isfinite(dl) &&
                       isfinite(tau) && isfinite(kappa));
    if (bad) {
      st->nonfinite = 1;
      st->nonfinite_iter = st->iter;
      st->done = 1;
      status = 5;  // INCONCLUSIVE
    } else if (st->iter >= 1) {
      if (fmax(pres, fmax(dres, gap)) <= st->tol) status = 1;
      else if (pinf <= st->tol) status = 2;
      else if (dinf <= st->tol) status = 3;
      if (status == 0 && st->iter >= st->max_iters) status = 4;
    }
    st->status = status;
    if (status != 0) st->done = 1;
    a.is->proceed = (mode == 0 && status == 0) ? 1 : 0;
  }
  if (mode == 2 && tid == 0) a.is->proceed = 1;
  __syncthreads();
  if (mode == 1) return;
  if (!a.is->proceed) return;

  // 3. tau elimination by the Schur complement on u_hat_3 (reading C15):
  //    q_low = w1_low + A_low^T sigma_2 = w1_low + z_t;  b^T q_2 = b^T x - beta_low^T z_t
  //    u_hat_3 = (w3 + c^T q_1 - b^T q_2) / (1 + zeta^T h);  u_hat_12 = q - u_hat_3 h
  dd bz{0.0, 0.0}, cq{0.0, 0.0};
  for (int j = tid; j < a.tl; j += TP_NT) {
    const int col = a.low_col[j];
    const double q1 = (a.xi[col] + a.z[col]) + a.zt[j];
    a.ulow[j] = q1;  // temporarily q_low
    bz = dd_add(bz, dd_prod(a.beta_low[j], a.zt[j]));
    cq = dd_add(cq, dd_prod(a.c_low[j], q1));
  }
  bz = dd_warp_sum(bz);
  cq = dd_warp_sum(cq);
  {
    const int w = tid >> 5, l = tid & 31;
    __syncthreads();  // shp is reused
    if (l == 0) {
      shp[0][w] = bz.hi;
      shp[1][w] = bz.lo;
      shp[2][w] = cq.hi;
      shp[3][w] = cq.lo;
    }
    __syncthreads();
  }
  if (tid == 0) {
    bz = dd{0.0, 0.0};
    cq = dd{0.0, 0.0};
    for (int i = 0; i < NW; ++i) bz = dd_add(bz, dd{shp[0][i], shp[1][i]});
    for (int i = 0; i < NW; ++i) cq = dd_add(cq, dd{shp[2][i], shp[3][i]});
    bc[0] = bz.hi;
    bc[1] = bz.lo;
    // zeta^T q = c^T q_1 - b^T q_2 = cq - (bx - bz), all in double-double
    dd bq2 = dd_add(dd{sums[PART_BX], sums[PART_BXLO]}, dd{-bc[0], -bc[1]});
    dd zq = dd_add(cq, dd{-bq2.hi, -bq2.lo});
    dd num = dd_add(dd{w3, 0.0}, zq);
    const double u3 = (num.hi + num.lo) / a.denom;
    a.is->omega3 = w3;
    a.is->coef = u3;
    a.is->u3 = u3;
    a.is->bsig2 = bq2.hi;
    const double tn = fmax(0.0, u3 - kappa);  // P_{R+}
    a.is->tau_new = tn;
    a.is->kappa_new = kappa - u3 + tn;
  }
  __syncthreads();
  const double u3 = a.is->u3;
  for (int j = tid; j < a.tl; j += TP_NT) a.ulow[j] = a.ulow[j] - u3 * a.h1_low[j];
  __syncthreads();
  if (mode == 2) return;
  // 4. free columns: cone R^t -> identity; xi = u_hat - z, z = z - u_hat + xi
  for (int j = tid; j < a.tl; j += TP_NT) {
    const int col = a.low_col[j];
    if (col < a.t_free) {
      const double u = a.ulow[j];
      const double zo = a.z[col];
      const double xn = u - zo;
      a.xi[col] = xn;
      a.z[col] = (zo - u) + xn;
    }
  }
}

// k_rowupdate: sigma_2 = q_2 = x - P^{-1} A_low z_t; u_hat_2 = q_2 - u_hat_3 h_2;
// y = u_hat_2 - s (R^m cone: identity); s = s - u_hat_2 + y.
__global__ void __launch_bounds__(256) k_rowupdate(AffineArgs a, int write_state) {
  if (a.st->done || !a.is->proceed) return;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.m) return;
  double v = 0.0;
  for (int e = a.lr_ptr[r]; e < a.lr_ptr[r + 1]; ++e) v = fma(a.lr_val[e], a.zt[a.lr_idx[e]], v);
  const double sig2 = a.x[r] - a.Pinv[r] * v;
  const double u2 = sig2 - a.is->coef * a.h2[r];
  a.uhat2[r] = u2;
  if (write_state) {
    const double so = a.s[r];
    const double yn = u2 - so;
    a.y[r] = yn;
    a.s[r] = (so - u2) + yn;
  }
}

// k_rowupdate with 8 lanes per row (rows with many low-rank entries, e.g. config 2's ~66): the
// lanes take entries l, l + 8, ... and combine by a fixed xor-shuffle tree
__global__ void __launch_bounds__(256) k_rowupdate8(AffineArgs a, int write_state) {
  if (a.st->done || !a.is->proceed) return;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = g >> 3, l = g & 7;
  double v = 0.0;
  if (r < a.m)
    for (int e = a.lr_ptr[r] + l; e < a.lr_ptr[r + 1]; e += 8) v = fma(a.lr_val[e], a.zt[a.lr_idx[e]], v);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  if (r >= a.m || l != 0) return;
  const double sig2 = a.x[r] - a.Pinv[r] * v;
  const double u2 = sig2 - a.is->coef * a.h2[r];
  a.uhat2[r] = u2;
  if (write_state) {
    const double so = a.s[r];
    const double yn = u2 - so;
    a.y[r] = yn;
    a.s[r] = (so - u2) + yn;
  }
}

// k_scatter: projection input a = u_hat_xi - z for every PSD svec position, written to
// asvec and unpacked (÷sqrt 2 off the diagonal) into the upper triangle of the block's matrix.
__global__ void __launch_bounds__(POS_NT) k_scatter(AffineArgs a, int zero_z) {
  if (a.st->done || !a.is->proceed) return;
  const int b = a.cta_blk[blockIdx.x];
  const long long q0 = a.cta_q0[blockIdx.x];
  const int N = a.blk_N[b];
  const long long L = (long long)N * (N + 1) / 2;
  const long long col0 = a.blk_col[b];
  double* M = a.mats + a.blk_mat[b];
  constexpr int PT = POS_PER_CTA / POS_NT;  // positions per thread, q = q0 + tid + t POS_NT
  // all loads of the thread's positions first (independent: memory-level parallelism), then the writes
  double v[PT];
  int ii[PT], jj[PT];
  {
    int i, j;
    svec_ij(q0 + threadIdx.x, i, j);
#pragma unroll
    for (int t = 0; t < PT; ++t) {  // advance (i, j) by POS_NT positions without another sqrt
      ii[t] = i;
      jj[t] = j;
      i += POS_NT;
      while (i > j && j < N) {
        i -= j + 1;
        ++j;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < PT; ++t) {
    const long long q = q0 + threadIdx.x + t * POS_NT;
    v[t] = 0.0;
    if (q >= L) continue;
    const long long col = col0 + q;
    const int code = a.code[col];
    if (code >= 0) v[t] = fma(a.aval[col], a.uhat2[code], a.xi[col]);
    else if (code == -1) v[t] = a.xi[col];
    else v[t] = a.ulow[-2 - code] - (zero_z ? 0.0 : a.z[col]);
  }
#pragma unroll
  for (int t = 0; t < PT; ++t) {
    const long long q = q0 + threadIdx.x + t * POS_NT;
    if (q >= L) continue;
    a.asvec[col0 + q - a.t_free] = v[t];
    // upper triangle only (column j, row i <= j: consecutive q are consecutive addresses); every
    // projection kernel reads the upper triangle (the Jacobi kernel symmetrically, the cluster
    // tridiagonalisation as "row i of the lower triangle")
    M[(size_t)jj[t] * N + ii[t]] = (ii[t] == jj[t]) ? v[t] : v[t] * SOS_IRT2;
  }
}

// k_pack: xi = svec(Pi(a)) (x sqrt 2 off the diagonal), z = xi - a (P:399-400 with the Moreau
// decomposition); CTA 0 commits tau, kappa and the iteration counter.
__global__ void __launch_bounds__(POS_NT) k_pack(AffineArgs a, double* out_xi, int commit) {
  if (a.st->done || !a.is->proceed) return;
  const int b = a.cta_blk[blockIdx.x];
  const long long q0 = a.cta_q0[blockIdx.x];
  const int N = a.blk_N[b];
  const long long L = (long long)N * (N + 1) / 2;
  const long long col0 = a.blk_col[b];
  const double* M = a.mats + a.blk_mat[b];
  const int neg = a.side ? a.side[b] : 0;
  constexpr int PT = POS_PER_CTA / POS_NT;
  double mv[PT], av[PT];
  int sp[PT];
  {
    int i, j;
    svec_ij(q0 + threadIdx.x, i, j);
#pragma unroll
    for (int t = 0; t < PT; ++t) {
      const long long q = q0 + threadIdx.x + t * POS_NT;
      const bool ok = q < L;
      // the projection kernels leave their result in the upper triangle (column j, row i <= j)
      mv[t] = ok ? M[(size_t)j * N + i] * (i == j ? 1.0 : SOS_RT2) : 0.0;
      av[t] = ok ? a.asvec[col0 + q - a.t_free] : 0.0;
      sp[t] = (ok && !out_xi) ? a.segpos[col0 + q] : -1;
      i += POS_NT;
      while (i > j && j < N) {
        i -= j + 1;
        ++j;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < PT; ++t) {
    const long long q = q0 + threadIdx.x + t * POS_NT;
    if (q >= L) continue;
    const long long col = col0 + q;
    double xn, zn;
    if (neg) {  // M = Pi(-a): z = M, xi = a + M (Moreau decomposition a = Pi(a) - Pi(-a))
      zn = mv[t];
      xn = av[t] + mv[t];
    } else {    // M = Pi(a): xi = M, z = xi - a
      xn = mv[t];
      zn = mv[t] - av[t];
    }
    if (out_xi) {
      out_xi[col - a.t_free] = xn;
    } else {
      a.xi[col] = xn;
      a.z[col] = zn;
      if (sp[t] >= 0) {  // the gather's alpha-ordered copies
        a.xis[sp[t]] = xn;
        a.zs[sp[t]] = zn;
      }
    }
  }
  if (commit && blockIdx.x == 0 && threadIdx.x == 0) {
    DevState* st = a.st;
    st->tau = a.is->tau_new;
    st->kappa = a.is->kappa_new;
    st->iter += 1;
  }
}

// Refresh the alpha-ordered copies from xi, z (after set_iterate / a restore).
__global__ void k_seg_copy(AffineArgs a) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.seg_ptr[a.m]) return;
  const int j = a.seg_col[e];
  a.xis[e] = a.xi[j];
  a.zs[e] = a.z[j];
}

// For configurations without PSD positions the commit happens here.
__global__ void k_commit(AffineArgs a) {
  if (a.st->done || !a.is->proceed) return;
  a.st->tau = a.is->tau_new;
  a.st->kappa = a.is->kappa_new;
  a.st->iter += 1;
}

// Unit entry point helper: unpack one block's svec vector src into its matrix (and asvec).
__global__ void k_unpack_block(AffineArgs a, int b, const double* src) {
  const int N = a.blk_N[b];
  const long long L = (long long)N * (N + 1) / 2;
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= L) return;
  double* M = a.mats + a.blk_mat[b];
  const double v = src[q];
  a.asvec[a.blk_col[b] - a.t_free + q] = v;
  int i, j;
  svec_ij(q, i, j);
  if (i == j) {
    M[(size_t)i * N + i] = v;
  } else {
    const double h = v * SOS_IRT2;
    M[(size_t)j * N + i] = h;
    M[(size_t)i * N + j] = h;
  }
}
