// Blocked Householder tridiagonalisation (LAPACK dsytrd / dlatrd organisation) inside one cluster,
// with the trailing rank-2nb update on the FP64 tensor cores (DMMA) — north_star (c): "blocked
// Householder tridiagonalisation ... with FP64 tensor-core (DMMA) trailing updates".
//
// Same distribution and exchanges as k_tridiag (tridiag.cuh): the lower triangle lives in the
// distributed shared memory of a C-CTA cluster, row i on CTA i mod C; every step has two push-only
// exchanges (st.async + mbarrier).  The difference is the update: within a panel of NB reflectors
// the trailing matrix is NOT updated; step k works on the stale matrix A_s (as of the panel start)
// and corrects with the panel's V = [v_k0 .. v_k-1], W = [w_k0 .. w_k-1] (dlatrd):
//     p   = tau (A_s v - V (W^T v) - W (V^T v))
//     x~  = column k+1 of A_s - V W[k+1, :]^T - W V[k+1, :]^T      (defines the next reflector)
// so the per-step pass over the trailing matrix is a READ-ONLY symmetric matrix-vector product
// (half the shared-memory traffic of the fused update+symv, and no update arithmetic), and once per
// panel every CTA applies A_s -= V W^T + W V^T to its rows with mma.sync.m8n8k4.f64 (K = 2 NB).
// The dot products V^T v, W^T v are sums over all rows: each CTA pushes its partials with the
// reduce-scatter of the symv (the same exchange).  Rows k0+1..k0+NB of W (needed by every CTA for x~)
// are pushed by their owners with the x~ allgather.  Every reduction is a fixed-order tree.
#pragma once
#include "tridiag.cuh"

constexpr int TRB_NB = 8;  // reflectors per panel

// Shared-memory layout (doubles): xt[2][N] | per own slot (S): ws[S] xs[S] qr[C][S] rp[NW][S]
// Vo[S][NB] Wo[S][NB] | Vd[NB][NB] Wd[NB][NB] pab[C][2NB] ab[2NB] | sd[C] se[C] ss[C] red[32] | rows
__host__ __device__ inline long long trb_fixed_doubles(int N, int C, int S, int NB) {
  return 2LL * N + 2LL * S + (long long)C * S + (long long)TRD_NW * S + 2LL * S * NB + 2LL * NB * NB +
         2LL * C * NB + 2LL * NB + 3LL * C + 32;
}

template <int MAXB, int CC, int NB>
__global__ void __launch_bounds__(TRD_NT, 1) k_tridiag_blk(TridiagArgs a) {
  if (a.check_state && (a.st->done || !a.is->proceed)) return;
  constexpr int C = CC;
  constexpr int logC = CC >= 16 ? 4 : (CC >= 8 ? 3 : (CC >= 4 ? 2 : (CC >= 2 ? 1 : 0)));
  const int N = a.N;
  const int me = (int)trd_cluster_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 3, cc = lane & 7;
  const int nown = (N - me + C - 1) >> logC;  // own rows i = me + q C
  auto first_slot = [&](int m) { return m > me ? (m - me + C - 1) >> logC : 0; };  // first q with i >= m
  const int S = (N + C - 1) >> logC;          // identical in every CTA (remote addresses use it)
  extern __shared__ __align__(16) double sm[];
  double* xt = sm;                // [2][N] x~_k by step parity (allgathered)
  double* ws = xt + 2 * N;        // w_k on own rows
  double* xs = ws + S;            // x~_{k+1} on own rows
  double* qr = xs + S;            // [C][S] reduce-scatter receive
  double* rp = qr + C * S;        // [NW][S] per-warp row partials
  double* Vo = rp + TRD_NW * S;   // [S][NB] panel V on own rows
  double* Wo = Vo + S * NB;       // [S][NB] panel W on own rows
  double* Vd = Wo + S * NB;       // [NB][NB] V on the panel's rows k0+1 .. k0+NB
  double* Wd = Vd + NB * NB;      // [NB][NB] W on the panel's rows k0+1 .. k0+NB
  double* pab = Wd + NB * NB;     // [C][2NB] partial (V^T v, W^T v) from each CTA
  double* ab = pab + 2 * C * NB;  // [2NB] their sums: a = V^T v, b = W^T v
  double* sd = ab + 2 * NB;       // [C] partial v^T A_s v
  double* se = sd + C;            // [C] partial (A_s v)[k+1]
  double* ss = se + C;            // [C] partial ||x~||^2
  double* red = ss + C;           // [32]
  double* rows = red + 32;
  __shared__ int roff[TRD_MAXOWN];  // smem offset of own row slot q, -1 = spilled to global
  __shared__ int nspill_s;
  __shared__ double qk1_s, scal_s[2];
  __shared__ __align__(8) uint64_t barQ, barY;
  double* Vg = a.Vg;  // [N][NB] panel V, every CTA writes its own rows (read back for the update)
  double* Wg = a.Wg;

  if (tid == 0) {
    long long need = 0;
    for (int q = 0; q < nown; ++q) need += me + q * C + 1;
    int ns = 0;
    while (need > a.smem_rows_doubles && ns < nown) {
      need -= me + ns * C + 1;
      ++ns;
    }
    long long off = 0;
    for (int q = 0; q < nown; ++q) {
      if (q < ns) {
        roff[q] = -1;
      } else {
        roff[q] = (int)off;
        off += me + q * C + 1;
      }
    }
    nspill_s = ns;
    trd_bar_init(&barQ);
    trd_bar_init(&barY);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nspill = nspill_s;
  auto rowptr_g = [&](int q) -> double* { return a.M + (size_t)(me + q * C) * N; };
  auto rowptr_s = [&](int q) -> double* { return rows + roff[q]; };
  auto rowptr = [&](int q) -> double* { return q < nspill ? rowptr_g(q) : rowptr_s(q); };
  for (int q = nspill; q < nown; ++q) {
    const int i = me + q * C;
    const double* src = a.M + (size_t)i * N;  // upper triangle of column i = row i of the lower
    double* dst = rowptr_s(q);
    for (int j = tid; j <= i; j += TRD_NT) dst[j] = src[j];
  }
  trd_cluster_sync();  // barriers initialised and every CTA running before the first remote store
  auto push = [&](double* dst, int peer, double v, uint64_t* bar) {
    trd_push(trd_mapa(dst, peer), v, trd_mapa(bar, peer));
  };

  // ---- column 0 defines v_0: push x~_0 = A[1:, 0], ||A[2:, 0]||^2 partials; d[0] ----
  if (tid == 0) trd_bar_expect(&barY, (unsigned)(8 * ((N - 1) + C)));
  {
    double s2 = 0.0;
    for (int q = tid; q < nown; q += TRD_NT) {
      const int i = me + q * C;
      const double x = rowptr(q)[0];
      xs[q] = x;
      if (i >= 2) s2 = fma(x, x, s2);
      if (i == 0) a.d[0] = x;
    }
    s2 = trd_block_sum(s2, red);
    for (int e = tid; e < nown * C; e += TRD_NT) {
      const int q = e >> logC, peer = e & (C - 1), i = me + q * C;
      if (i >= 1) push(xt + i, peer, xs[q], &barY);
    }
    if (tid < C) push(ss + me, tid, s2, &barY);
  }
  trd_bar_wait(&barY, 0);

  const bool prof = a.prof != nullptr && me == 0 && tid == 0;
#define TRB_STAMP(ph) \
  if (prof) a.prof[(size_t)k * 16 + (ph)] = clock64();
  for (int k = 0; k < N - 2; ++k) {
    const int par = k & 1;
    const int k0 = k - k % NB, t = k - k0;  // panel start, position in the panel
    TRB_STAMP(0)
    const double* xk = xt + par * N;  // x~_k
    const int qs1 = first_slot(k + 1), qs2 = first_slot(k + 2);
    const int nb = (N - k - 1 + 7) >> 3;
    auto nwarps_of_row = [&](int i) { return min(min(TRD_NW, nb), (i - k - 1) / 8 + 1); };
    // ---- Phase A: the reflector of column k (warp 0) ----
    if (warp == 0) {
      if (lane == 0)
        trd_bar_expect(&barQ, (unsigned)(8 * (C * (nown - qs2) + 2 * C + 2 * t * C)));
      const double sig = trd_sumc<CC>(ss);
      const double alpha = xk[k + 1];
      double tk = 0.0, beta = alpha, scale = 0.0;
      if (sig != 0.0) {  // one rsqrt + one division (see k_tridiag)
        const double n2 = fma(alpha, alpha, sig);
        const double rs = rsqrt(n2);
        const double nrm = n2 * rs;
        beta = -copysign(nrm, alpha);
        tk = fma(fabs(alpha), rs, 1.0);
        scale = copysign(1.0, alpha) / (fabs(alpha) + nrm);
      }
      TRB_STAMP(8)
      if (lane == 0) {
        scal_s[0] = tk;
        scal_s[1] = scale;
        if (me == (k & (C - 1))) {
          a.e[k] = beta;
          a.tau[k] = tk;
        }
      }
    }
    __syncthreads();
    TRB_STAMP(9)
    const double tk = scal_s[0], scale = scal_s[1];
    auto vof = [&](int i) { return i == k + 1 ? 1.0 : (i > k + 1 ? xk[i] * scale : 0.0); };  // v_k[i]
    if (me == (k & (C - 1)))
      for (int j = k + 1 + tid; j < N; j += TRD_NT) a.V[(size_t)k * N + j] = vof(j);
    if (tid < NB) Vd[tid * NB + t] = vof(k0 + 1 + tid);  // v_k on the panel's rows
    int nbt = 0;
#pragma unroll
    for (int tt = 0; tt < MAXB; ++tt) nbt += trd_block(warp, tt) < nb ? 1 : 0;
    double vn[MAXB], qa[MAXB];
#pragma unroll
    for (int tt = 0; tt < MAXB; ++tt) {
      const int j = k + 1 + 8 * trd_block(warp, tt) + cc;
      vn[tt] = (tt < nbt && j < N) ? vof(j) : 0.0;
      qa[tt] = 0.0;
    }
    TRB_STAMP(1)

    // ---- Phase X: read-only symv with the stale matrix over own rows i >= k+1 ----
    double dpart = 0.0;
    const int qw = first_slot(k + 1 + 8 * warp);
    auto row_group = [&](int g, int qe, auto rp_of, auto FULL) {
      constexpr bool full = decltype(FULL)::value;
      const int q = full ? g + lr : min(g + lr, qe - 1);
      const bool valid = full || g + lr < qe;
      const int ic = me + q * C;
      const int i = valid ? ic : -1;
      const int imin = me + g * C;
      const int imax = me + (full ? g + 3 : min(g + 3, qe - 1)) * C;
      const double* R = rp_of(q);
      const double vin = vof(ic);
      double racc = 0.0;
#pragma unroll
      for (int tt = 0; tt < MAXB; ++tt) {
        const int jf = k + 1 + 8 * trd_block(warp, tt);
        if (tt >= nbt || jf > imax) break;
        const int j = jf + cc;
        if (jf + 7 < imin) {
          if (full || valid) {
            const double x = R[j];
            racc = fma(x, vn[tt], racc);
            qa[tt] = fma(x, vin, qa[tt]);
          }
        } else if (j <= i) {
          const double x = R[j];
          racc = fma(x, vn[tt], racc);
          qa[tt] = fma(x, (j < i) ? vin : 0.0, qa[tt]);
        }
      }
      racc += __shfl_xor_sync(0xffffffffu, racc, 1);
      racc += __shfl_xor_sync(0xffffffffu, racc, 2);
      racc += __shfl_xor_sync(0xffffffffu, racc, 4);
      if (valid && cc == 0) {
        rp[warp * S + q] = racc;
        dpart = fma(racc, vin, dpart);
      }
    };
    // two full groups per iteration: independent load / FMA chains for latency hiding
    auto row_group2 = [&](int g, auto rp_of) {
      const int qA = g + lr, qB = g + 4 + lr;
      const int iA = me + qA * C, iB = me + qB * C;
      const int iminA = me + g * C, iminB = me + (g + 4) * C, imax = me + (g + 7) * C;
      const double* RA = rp_of(qA);
      const double* RB = rp_of(qB);
      const double vA = vof(iA), vB = vof(iB);
      double ra = 0.0, rb = 0.0;
#pragma unroll
      for (int tt = 0; tt < MAXB; ++tt) {
        const int jf = k + 1 + 8 * trd_block(warp, tt);
        if (tt >= nbt || jf > imax) break;
        const int j = jf + cc;
        if (jf + 7 < iminA) {  // both groups strictly below the diagonal
          const double xa = RA[j], xb = RB[j];
          ra = fma(xa, vn[tt], ra);
          rb = fma(xb, vn[tt], rb);
          qa[tt] = fma(xb, vB, fma(xa, vA, qa[tt]));
        } else {
          if (j <= iA) {
            const double xa = RA[j];
            ra = fma(xa, vn[tt], ra);
            qa[tt] = fma(xa, (j < iA) ? vA : 0.0, qa[tt]);
          }
          if (j <= iB) {
            const double xb = RB[j];
            rb = fma(xb, vn[tt], rb);
            qa[tt] = fma(xb, (j < iB) ? vB : 0.0, qa[tt]);
          }
        }
      }
      ra += __shfl_xor_sync(0xffffffffu, ra, 1);
      rb += __shfl_xor_sync(0xffffffffu, rb, 1);
      ra += __shfl_xor_sync(0xffffffffu, ra, 2);
      rb += __shfl_xor_sync(0xffffffffu, rb, 2);
      ra += __shfl_xor_sync(0xffffffffu, ra, 4);
      rb += __shfl_xor_sync(0xffffffffu, rb, 4);
      if (cc == 0) {
        rp[warp * S + qA] = ra;
        rp[warp * S + qB] = rb;
        dpart = fma(ra, vA, fma(rb, vB, dpart));
      }
    };
    auto row_groups = [&](int qb, int qe, auto rp_of) {
      if (nbt == 0) return;
      int g = max(qb, qw);
      for (; g + 8 <= qe; g += 8) row_group2(g, rp_of);
      for (; g + 4 <= qe; g += 4) row_group(g, qe, rp_of, std::true_type());
      if (g < qe) row_group(g, qe, rp_of, std::false_type());
    };
    if (qs1 < nspill) row_groups(qs1, nspill, rowptr_g);
    row_groups(max(qs1, nspill), nown, rowptr_s);
    TRB_STAMP(2)
#pragma unroll
    for (int tt = 0; tt < MAXB; ++tt) {
      if (tt >= nbt) break;
      double v = qa[tt];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      qa[tt] = v;
      if (lr == 0) dpart = fma(v, vn[tt], dpart);
    }
    if (warp == 0 && lane == 0) qk1_s = qa[0];
    if (lr == 0) {
#pragma unroll
      for (int tt = 0; tt < MAXB; ++tt) {
        if (tt >= nbt) break;
        const int j = k + 1 + 8 * trd_block(warp, tt) + cc;
        if (j >= k + 2 && j < N) push(qr + me * S + (j >> logC), j & (C - 1), qa[tt], &barQ);
      }
    }
    dpart = warp_sum(dpart);
    if (lane == 0) red[warp] = dpart;
    __syncthreads();
    TRB_STAMP(3)
    // panel dot products over own rows: warp u < t -> a_u = sum V[i][u] v_i, warp t + u -> b_u
    if (warp < 2 * t) {
      const int u = warp < t ? warp : warp - t;
      const double* P = warp < t ? Vo : Wo;
      double acc = 0.0;
      for (int q = qs1 + lane; q < nown; q += 32) acc = fma(P[q * NB + u], vof(me + q * C), acc);
      acc = warp_sum(acc);
      if (lane < C) push(pab + me * 2 * NB + (warp < t ? u : NB + u), lane, acc, &barQ);
    }
    if (tid < C) {
      const double dsum = trd_sumc<TRD_NW>(red);
      double e1 = qk1_s;
      if (((k + 1) & (C - 1)) == me) e1 += trd_sum16(rp + ((k + 1) >> logC), nwarps_of_row(k + 1), S);
      push(sd + me, tid, dsum, &barQ);
      push(se + me, tid, e1, &barQ);
    }
    TRB_STAMP(4)
    const bool last = (k == N - 3);
    const int nslot = nown - qs1;
    const int nslotw = (nslot + 31) >> 5;
    double prow_own = 0.0;
    if (tid < nslot) {
      const int i = me + (qs1 + tid) * C;
      if (i > k + 1) prow_own = trd_sum16(rp + qs1 + tid, nwarps_of_row(i), S);
    }
    // rows of the panel's W this exchange delivers: w_k on rows k+2 .. min(k0+NB, N-1)
    const int npw = max(0, min(k0 + NB, N - 1) - (k + 1));
    if (tid == 0 && !last) trd_bar_expect(&barY, (unsigned)(8 * ((N - k - 2) + C + npw)));
    trd_bar_wait(&barQ, par);
    TRB_STAMP(5)

    // ---- Phase Y: corrected w_k on own rows, x~_{k+1}, its norm partial ----
    if (tid < 2 * t) ab[tid < t ? tid : NB + tid - t] = trd_sum16(pab + (tid < t ? tid : NB + tid - t), C, 2 * NB);
    __syncthreads();
    double Kc = 0.0, wk1 = 0.0;
    if (tid < max(nslot, 1)) {  // only the own-row threads (and thread 0) need the scalars
      double sab = 0.0;  // a . b
      for (int u = 0; u < t; ++u) sab = fma(ab[u], ab[NB + u], sab);
      const double sdv = trd_sumc<CC>(sd) - 2.0 * sab;  // v^T A v with the panel correction
      Kc = 0.5 * tk * tk * sdv;
      // p_{k+1} and w_k[k+1] (row k+1 is the panel row rr = t): every CTA, same order
      double corr1 = 0.0;
      for (int u = 0; u < t; ++u) corr1 = fma(Vd[t * NB + u], ab[NB + u], fma(Wd[t * NB + u], ab[u], corr1));
      wk1 = tk * (trd_sumc<CC>(se) - corr1) - Kc;
      if (tid == 0) Wd[t * NB + t] = wk1;
    }
    TRB_STAMP(10)
    double s2 = 0.0;
    if (tid < nslot) {
      const int q = qs1 + tid, i = me + q * C;
      double* R = rowptr(q);
      double* vo = Vo + q * NB;
      double* wo = Wo + q * NB;
      if (i == k + 1) {
        vo[t] = 1.0;
        wo[t] = wk1;
        Vg[(size_t)i * NB + t] = 1.0;
        Wg[(size_t)i * NB + t] = wk1;
        double dd = 0.0;  // d_{k+1} = A_s[k+1][k+1] - 2 V[k+1, :] . W[k+1, :]
        for (int u = 0; u <= t; ++u) dd = fma(Vd[t * NB + u], u == t ? wk1 : Wd[t * NB + u], dd);
        a.d[k + 1] = R[k + 1] - 2.0 * dd;
      } else {
        const double vin = xk[i] * scale;
        double corr = 0.0;
        for (int u = 0; u < t; ++u) corr = fma(vo[u], ab[NB + u], fma(wo[u], ab[u], corr));
        const double pq = prow_own + trd_sum16(qr + q, C, S) - corr;
        const double wi = fma(-Kc, vin, tk * pq);
        vo[t] = vin;
        wo[t] = wi;
        ws[q] = wi;
        Vg[(size_t)i * NB + t] = vin;
        Wg[(size_t)i * NB + t] = wi;
        // x~_{k+1}[i] = A_s[i][k+1] - sum_{u <= t} (V[i][u] W[k+1][u] + W[i][u] V[k+1][u])
        double cx = 0.0;
        for (int u = 0; u < t; ++u) cx = fma(vo[u], Wd[t * NB + u], fma(wo[u], Vd[t * NB + u], cx));
        cx = fma(vin, wk1, fma(wi, 1.0, cx));
        const double x = R[k + 1] - cx;
        xs[q] = x;
        if (i >= k + 3) s2 = x * x;
        if (last) {  // i == N - 1: the trailing 2 x 2 block
          a.e[N - 2] = x;
          double dd = 0.0;
          for (int u = 0; u <= t; ++u) dd = fma(vo[u], wo[u], dd);
          a.d[N - 1] = R[N - 1] - 2.0 * dd;
          a.tau[N - 2] = 0.0;
        }
      }
    }
    if (last) break;
    if (warp < nslotw) {
      s2 = warp_sum(s2);
      if (lane == 0) red[16 + warp] = s2;
    }
    TRB_STAMP(6)
    __syncthreads();  // xs / ws of every own row written
    if (tid < C) push(ss + me, tid, trd_sum16(red + 16, nslotw, 1), &barY);
    {
      double* xnext = xt + (par ^ 1) * N;
      const int nact = nown - qs2;
      for (int e = tid; e < nact * C; e += TRD_NT) {
        const int q = qs2 + (e >> logC), peer = e & (C - 1), i = me + q * C;
        push(xnext + i, peer, xs[q], &barY);
        if (i <= k0 + NB) push(Wd + (i - k0 - 1) * NB + t, peer, ws[q], &barY);  // panel rows of W
      }
    }
    TRB_STAMP(7)
    trd_bar_wait(&barY, par ^ 1);
    if (t == NB - 1) {
      // ---- panel end: A_s -= V W^T + W V^T on own rows i, columns k+2 <= j <= i (DMMA, K = 2 NB) ----
      trd_cluster_sync();  // every CTA's rows of Vg / Wg are written and visible
      const int jlo = k + 2;
      const int qlo2 = first_slot(jlo);
      const int nrt = (nown - qlo2 + 7) >> 3;  // row tiles of 8 own slots
      const int ncol = N - jlo;
      const int nct = (ncol + 7) >> 3;         // column tiles of 8
      // column tile outer (its B fragments loaded once from L2), row tiles inner
      for (int ct = warp; ct < nct; ct += TRD_NW) {
        const int j0 = jlo + 8 * ct;
        double bfr[2 * NB / 4];  // B[kk][n]: kk < NB from W rows, kk >= NB from V rows (n = column)
#pragma unroll
        for (int s4 = 0; s4 < 2 * NB / 4; ++s4) {
          const int kk = 4 * s4 + (lane & 3);
          const int jn = j0 + (lane >> 2);
          bfr[s4] = (jn < N) ? (kk < NB ? Wg[(size_t)jn * NB + kk] : Vg[(size_t)jn * NB + kk - NB]) : 0.0;
        }
        for (int rt = 0; rt < nrt; ++rt) {
          const int qb = qlo2 + 8 * rt;
          const int imax_t = me + min(qb + 7, nown - 1) * C;
          if (imax_t < j0) continue;  // tile entirely above the diagonal
          double c0 = 0.0, c1 = 0.0;
          const int qa_ = min(qb + (lane >> 2), nown - 1);
#pragma unroll
          for (int s4 = 0; s4 < 2 * NB / 4; ++s4) {
            const int kk = 4 * s4 + (lane & 3);
            const double af = kk < NB ? Vo[qa_ * NB + kk] : Wo[qa_ * NB + kk - NB];
            dmma_8x8x4(c0, c1, af, bfr[s4]);
          }
          const int q = qb + (lane >> 2);
          if (q < nown) {
            const int i = me + q * C;
            double* R = rowptr(q);
            const int jj = j0 + 2 * (lane & 3);
            if (jj <= i) R[jj] -= c0;
            if (jj + 1 <= i) R[jj + 1] -= c1;
          }
        }
      }
      __syncthreads();  // updated rows before the next step's symv
    }
  }
#undef TRB_STAMP
  trd_cluster_sync();
}

typedef void (*TridiagBlkKernel)(TridiagArgs);
#define TRB_KERNELS(X) X(2, 4) X(2, 8) X(4, 8) X(4, 16) X(7, 16) X(10, 16)
inline TridiagBlkKernel tridiag_blk_kernel_mc(int maxb, int C) {
#define TRB_CASE(MB, CCX) \
  if (maxb == MB && C == CCX) return k_tridiag_blk<MB, CCX, TRB_NB>;
  TRB_KERNELS(TRB_CASE)
#undef TRB_CASE
  return nullptr;
}
