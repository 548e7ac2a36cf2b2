// Blocked (compact-WY) back-transform of the selected tridiagonal eigenvectors, third stage of the
// large-block PSD projection (north_star (c) "back-transform ... on FP64 tensor
// cores"; PAPER.md P:397-398 needs Pi(a) = H Z_r diag(lambda_r) Z_r^T H^T).
//
//   H = H_0 H_1 ... H_{N-3},  H_k = I - tau_k v_k v_k^T  (from k_tridiag, LAPACK dsytrd 'L').
//   Reflectors are grouped in blocks of BTW_NB: H_{k0} ... H_{k0+nb-1} = I - V_b T_b V_b^T with T_b
//   upper triangular (LAPACK dlarft, forward / columnwise), so W = H Z_r is
//   for b = last .. 0:   Y = V_b^T W;  Y = T_b Y;  W -= V_b Y
// — two thin DMMA GEMMs per block instead of 32 rank-1 BLAS-1 updates.  One cluster of BTC_P CTAs
// owns BTW_NC columns of W; the rows are split over the cluster, so each CTA holds its row slice of
// W and of V_b in shared memory (V_b's slice is loaded once per block, with a cp.async double
// buffer prefetching block b-1 while block b computes), and the 32 x 8 partial products V_b^T W are
// all-reduced over distributed shared memory (push to every peer, one cluster barrier per block,
// fixed summation order).  Column tiles are independent clusters.
//
// T_b: k_bt_gram forms partial Gram matrices G = V_b^T V_b per (block, row chunk) in parallel;
// k_bt_larft sums them in a fixed order and builds T_b by the recursive dlarft formula
//   T = [T11  -T11 G12 T22; 0  T22]   (halves of sizes 1, 2, 4, 8, 16), diag(T) = tau.
#pragma once
#include "common.cuh"
#include "gemm_f64.cuh"

constexpr int BTW_NB = 32;   // reflectors per WY block
constexpr int BTW_NC = 8;    // W columns per CTA (one DMMA n-tile)
constexpr int BTW_NT = 256;  // 8 warps
constexpr int BTW_RC = 128;  // V rows per streamed chunk
constexpr int BTW_LD = BTW_RC + 4;  // padded chunk row stride (conflict-free DMMA fragment reads)
constexpr int BTG_RC = 128;  // rows per Gram partial

// v_k[row] as stored by k_tridiag: 0 above row k+1, 1 at row k+1, V[k N + row] below; reflectors
// k >= nref do not exist (zero).
__device__ __forceinline__ double btw_v(const double* __restrict__ V, int N, int nref, int k, int row) {
  return (k < nref && row > k && row < N) ? __ldg(V + (size_t)k * N + row) : 0.0;
}

inline int bt_gram_chunks(int N) { return (N + BTG_RC - 1) / BTG_RC; }

// grid (nblk, chunks): Gp[b][chunk] = V_b[rows of chunk]^T V_b[rows of chunk] (32 x 32).
__global__ void __launch_bounds__(BTW_NT) k_bt_gram(const double* __restrict__ V, double* __restrict__ Gp, int N,
                                                    int nref, const DevState* st, const IterScal* is,
                                                    int check_state) {
  if (check_state && (st->done || !is->proceed)) return;
  const int b = blockIdx.x, ch = blockIdx.y, k0 = b * BTW_NB;
  const int r0 = ch * BTG_RC;
  double* out = Gp + ((size_t)b * gridDim.y + ch) * BTW_NB * BTW_NB;
  const int tid = threadIdx.x;
  if (r0 + BTG_RC <= k0 + 1) {  // chunk entirely above the block's reflectors
    for (int e = tid; e < BTW_NB * BTW_NB; e += BTW_NT) out[e] = 0.0;
    return;
  }
  __shared__ double vs[BTW_NB][BTG_RC + 1];
  for (int e = tid; e < BTW_NB * BTG_RC; e += BTW_NT) {
    const int rr = e % BTG_RC, c = e / BTG_RC;
    vs[c][rr] = btw_v(V, N, nref, k0 + c, r0 + rr);
  }
  __syncthreads();
  const int gi = tid >> 3, gj0 = (tid & 7) * 4;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int rr = 0; rr < BTG_RC; ++rr) {
    const double vi = vs[gi][rr];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = fma(vi, vs[gj0 + q][rr], acc[q]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) out[gi * BTW_NB + gj0 + q] = acc[q];
}

// grid nblk: G = sum of the chunk partials (fixed order); T_b by the recursive dlarft formula.
__global__ void __launch_bounds__(BTW_NT) k_bt_larft(const double* __restrict__ Gp, int nchunks,
                                                     const double* __restrict__ tau, double* __restrict__ Tall,
                                                     int nref, const DevState* st, const IterScal* is,
                                                     int check_state) {
  if (check_state && (st->done || !is->proceed)) return;
  const int b = blockIdx.x, k0 = b * BTW_NB;
  const int nb = min(BTW_NB, nref - k0);
  __shared__ double G[BTW_NB][BTW_NB + 1];
  __shared__ double T[BTW_NB][BTW_NB + 1];
  __shared__ double X[BTW_NB][BTW_NB + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < BTW_NB * BTW_NB; e += BTW_NT) {
    const int i = e / BTW_NB, j = e % BTW_NB;
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += Gp[((size_t)b * nchunks + c) * BTW_NB * BTW_NB + e];
    G[i][j] = s;
    T[i][j] = (i == j && i < nb) ? tau[k0 + i] : 0.0;
  }
  __syncthreads();
  for (int s = 1; s < BTW_NB; s *= 2) {
    // pairs of diagonal blocks (p, p + s), p = 0, 2s, 4s, ...: T12 = -T11 G12 T22
    const int npairs = BTW_NB / (2 * s), per = s * s;
    for (int e = tid; e < npairs * per; e += BTW_NT) {  // X = G12 T22
      const int pr = e / per, i = (e % per) / s, j = e % s;
      const int p = pr * 2 * s;
      double acc = 0.0;
      for (int l = 0; l <= j; ++l) acc = fma(G[p + i][p + s + l], T[p + s + l][p + s + j], acc);
      X[p + i][p + s + j] = acc;
    }
    __syncthreads();
    for (int e = tid; e < npairs * per; e += BTW_NT) {  // T12 = -T11 X
      const int pr = e / per, i = (e % per) / s, j = e % s;
      const int p = pr * 2 * s;
      double acc = 0.0;
      for (int l = i; l < s; ++l) acc = fma(T[p + i][p + l], X[p + l][p + s + j], acc);
      T[p + i][p + s + j] = -acc;
    }
    __syncthreads();
  }
  double* To = Tall + (size_t)b * BTW_NB * BTW_NB;
  for (int e = tid; e < BTW_NB * BTW_NB; e += BTW_NT) To[e] = T[e / BTW_NB][e % BTW_NB];  // row-major
}

// ---------------------------------------------------------------------------------------------
constexpr int BTC_P = 8;      // CTAs per cluster (row split)
constexpr int BTC_NT = 128;   // 4 warps
constexpr int BTC_NW = BTC_NT / 32;

__device__ __forceinline__ void btc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned btc_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void btc_push(const double* local, int peer, double v) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(local);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(peer));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

__host__ __device__ inline int btc_rows(int N) { return (((N + BTC_P - 1) / BTC_P) + 7) / 8 * 8; }
__host__ __device__ inline int btc_ldv(int RS) { return RS + 4; }
inline size_t bt_apply_smem_bytes(int N) {
  const int RS = btc_rows(N), LDV = btc_ldv(RS);
  return sizeof(double) * ((size_t)RS * BTW_NC + 2 * BTW_NB * LDV + 2 * BTC_P * BTW_NB * BTW_NC +
                           BTC_NW * BTW_NB * BTW_NC + BTW_NB * BTW_NC + 2 * BTW_NB * BTW_NB);
}

// W[:, c] = H Z[:, c0 + c] sqrt|lambda_{c0+c}|, c < r (r, c0 from k_select's sel[]); W has pitch ldw;
// scale = 0 writes H Z[:, c0 + c] itself (the warm mode's cold path: every eigenvector, warm.cuh).
// grid: BTC_P x (number of 8-column tiles), cluster (BTC_P, 1, 1).
__global__ void __launch_bounds__(BTC_NT) k_bt_apply(const double* __restrict__ Qf, const double* __restrict__ lamf,
                                                     const double* __restrict__ V, const double* __restrict__ Tall,
                                                     const int* __restrict__ sel, double* __restrict__ W, int N,
                                                     int nref, const DevState* st, const IterScal* is,
                                                     int check_state, int ldw, int scale) {
  if (check_state && (st->done || !is->proceed)) return;
  const int r = sel[0], c0 = sel[1];
  const int q = (int)btc_rank();
  const int cbase = (blockIdx.x / BTC_P) * BTW_NC;
  if (cbase >= r) return;  // uniform over the cluster
  const int RS = btc_rows(N), LDV = btc_ldv(RS);
  const int rlo = q * RS, rhi = min(N, rlo + RS);
  extern __shared__ __align__(16) double smem[];
  double* Ws = smem;                               // [RS][8] row slice of W
  double* Vs = Ws + (size_t)RS * BTW_NC;           // [2][32][LDV]  V_b row slice
  double* Yr = Vs + 2 * BTW_NB * LDV;              // [2][P][32*8]  partials received from peers
  double* Yp = Yr + 2 * BTC_P * BTW_NB * BTW_NC;   // [NW][32*8]    warp partials
  double* Ys = Yp + BTC_NW * BTW_NB * BTW_NC;      // [32*8]
  double* Ts = Ys + BTW_NB * BTW_NC;               // [2][32*32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int nblk = (nref + BTW_NB - 1) / BTW_NB;

  for (int e = tid; e < RS * BTW_NC; e += BTC_NT) {
    const int rr = e / BTW_NC, c = e % BTW_NC, row = rlo + rr;
    Ws[e] = (row < rhi && cbase + c < r) ? Qf[(size_t)(c0 + cbase + c) * N + row] : 0.0;
  }
  auto issue = [&](int b, int buf) {
    const int k0 = b * BTW_NB, lo = max(rlo, k0 + 1);
    double* dst = Vs + (size_t)buf * BTW_NB * LDV;
    for (int refl = warp; refl < BTW_NB && k0 + refl < nref; refl += BTC_NW) {
      const double* src = V + (size_t)(k0 + refl) * N;
      for (int row = lo + lane; row < rhi; row += 32) cp_async8(dst + refl * LDV + (row - rlo), src + row);
    }
    double* tdst = Ts + buf * BTW_NB * BTW_NB;
    for (int e = 2 * tid; e < BTW_NB * BTW_NB; e += 2 * BTC_NT) cp_async16(tdst + e, Tall + (size_t)b * BTW_NB * BTW_NB + e);
    cp_async_commit();
  };
  issue(nblk - 1, 0);
  btc_cluster_sync();  // every CTA of the cluster runs before the first remote store
  int buf = 0;
  for (int b = nblk - 1; b >= 0; --b, buf ^= 1) {
    const int k0 = b * BTW_NB, lo = max(rlo, k0 + 1);
    const bool active = lo < rhi;
    if (b > 0) {
      issue(b - 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* Vc = Vs + (size_t)buf * BTW_NB * LDV;
    double* Yrb = Yr + (size_t)(b & 1) * BTC_P * BTW_NB * BTW_NC;
    if (active) {
      // ---- partial Y = V_b[slice]^T W[slice]: 4-row k-steps over [lo, rhi) ----
      double acc[4][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
      for (int rs = lo + 4 * warp; rs < rhi; rs += 4 * BTC_NW) {
        const int row = rs + lc;
        const bool ok = row < rhi;
        const double bf = ok ? Ws[(row - rlo) * BTW_NC + lr] : 0.0;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const int refl = mt * 8 + lr;
          const double af = (ok && row > k0 + refl && k0 + refl < nref) ? Vc[refl * LDV + (row - rlo)] : 0.0;
          dmma_8x8x4(acc[mt][0], acc[mt][1], af, bf);
        }
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) Yp[(warp * BTW_NB + mt * 8 + lr) * BTW_NC + 2 * lc + h] = acc[mt][h];
      __syncthreads();
      for (int e = tid; e < BTW_NB * BTW_NC; e += BTC_NT) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < BTC_NW; ++w) s += Yp[w * BTW_NB * BTW_NC + e];
        for (int p = 0; p < BTC_P; ++p) {
          const int phi = min(N, (p + 1) * RS);
          if (phi > k0 + 1) btc_push(Yrb + q * BTW_NB * BTW_NC + e, p, s);  // peers with work in block b
        }
      }
    }
    btc_cluster_sync();
    if (active) {
      // ---- Y = sum of the active slices' partials (fixed order); Y <- T_b Y ----
      const double* Tb = Ts + buf * BTW_NB * BTW_NB;
      for (int e = tid; e < BTW_NB * BTW_NC; e += BTC_NT) {
        double s = 0.0;
        for (int p = 0; p < BTC_P; ++p) {
          const int plo = max(p * RS, k0 + 1), phi = min(N, (p + 1) * RS);
          if (plo < phi) s += Yrb[p * BTW_NB * BTW_NC + e];
        }
        Ys[e] = s;
      }
      __syncthreads();
      double t[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = tid + h * BTC_NT, i = e / BTW_NC, c = e % BTW_NC;
        double acc = 0.0;
        for (int j = i; j < BTW_NB; ++j) acc = fma(Tb[i * BTW_NB + j], Ys[j * BTW_NC + c], acc);
        t[h] = acc;
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; ++h) Ys[tid + h * BTC_NT] = t[h];
      __syncthreads();
      // ---- W[slice] -= V_b[slice] Y over 8-row m-tiles from lo ----
      for (int rt = lo + 8 * warp; rt < rhi; rt += 8 * BTC_NW) {
        const int arow = rt + lr;
        const bool ok = arow < rhi;
        double c0v = 0.0, c1v = 0.0;
#pragma unroll
        for (int ks = 0; ks < BTW_NB / 4; ++ks) {
          const int refl = ks * 4 + lc;
          const double af = (ok && arow > k0 + refl && k0 + refl < nref) ? Vc[refl * LDV + (arow - rlo)] : 0.0;
          const double bf = Ys[(ks * 4 + lc) * BTW_NC + lr];
          dmma_8x8x4(c0v, c1v, af, bf);
        }
        if (ok) {
          double2* wp = reinterpret_cast<double2*>(Ws + (arow - rlo) * BTW_NC + 2 * lc);
          double2 wv = *wp;
          wv.x -= c0v;
          wv.y -= c1v;
          *wp = wv;
        }
      }
    }
    __syncthreads();  // Vs[buf], Ts[buf] free for the prefetch two blocks ahead
  }
  for (int e = tid; e < RS * BTW_NC; e += BTC_NT) {
    const int rr = e / BTW_NC, c = e % BTW_NC, row = rlo + rr;
    if (row < rhi && cbase + c < r)
      W[(size_t)(cbase + c) * ldw + row] = scale ? Ws[e] * sqrt(fabs(lamf[c0 + cbase + c])) : Ws[e];
  }
}
