// Householder tridiagonalisation T = H^T A H of one symmetric block inside ONE thread-block cluster.
//
// First stage of the large-block PSD projection (north_star (c): "blocked
// Householder tridiagonalisation plus a tridiagonal solve and back-transform").  The reflectors
// H_k = I - tau_k v_k v_k^T follow LAPACK dsytd2 ('L'): v_k[k+1] = 1, v_k[0..k] = 0,
//   p = tau A v,  w = p - (tau/2)(p^T v) v,  A <- A - v w^T - w v^T.
//
// B200 mapping (one cluster of C <= 16 CTAs, everything in distributed shared memory):
//   * the lower triangle is distributed by ROWS, row i on CTA i mod C, so every column (and with
//     it every reflector) is spread evenly over the cluster: no CTA ever broadcasts a whole vector
//     (DSMEM is ~20 B/cycle per SM, so a one-to-all broadcast would serialise on one port);
//   * communication is push-only: st.async into the consumers' shared memory, each store completing
//     transaction bytes on the consumer's mbarrier, which waits for the byte count it expects — no
//     cluster-wide barrier (and none of its memory fences) inside the loop; every reduction is
//     summed in a fixed order, so the factorisation is bit-reproducible;
//   * the rank-2 update of step k-1 is fused with the symmetric matrix-vector product of step k
//     (one read + one write of the trailing matrix per step), and the column that defines the next
//     reflector is updated eagerly, so each step has only TWO exchange phases:
//       [fused update(k-1) + symv(k)] -> push row-sum partials (reduce-scatter) + 2 scalars -> barQ
//       [w_k for own rows, column k+1, its norm partial] -> push x, w (allgather) + 1 scalar -> barY
// Rows that do not fit in shared memory (smallest first) stay in the block matrix in global memory
// (upper triangle of column i = row i of the lower triangle), L2-resident.
#pragma once
#include "common.cuh"

constexpr int TRD_NT = 512;
constexpr int TRD_NW = TRD_NT / 32;
constexpr int TRD_MAXC = 16;
constexpr int TRD_MAXOWN = 96;  // own rows per CTA
// Phase X thread mapping: lane = (lr, cc), lr = lane / 8 picks one of 4 rows of a row group, cc one
// of 8 consecutive columns of a column block; warp w owns column blocks w, w + 16, w + 32, ...
// (MAXB of them), so row sums reduce over 8 lanes and column sums over 4 lanes only.
inline int tridiag_maxb(int N) {
  const int nb = ((N - 1) + 7) / 8;
  const int m = (nb + TRD_NW - 1) / TRD_NW;
  return m <= 2 ? 2 : (m <= 4 ? 4 : (m <= 7 ? 7 : 10));
}

struct TridiagArgs {
  double* M;         // N x N column-major block matrix (both triangles valid on input)
  int N;
  int C;             // cluster size (CTAs)
  long long smem_rows_doubles;  // per-CTA shared-memory budget for row storage
  double* d;         // N
  double* e;         // N - 1
  double* tau;       // N - 1
  double* V;         // N x N column-major: v_k in column k, rows k+1..N-1 (v_k[k+1] = 1)
  const DevState* st;
  const IterScal* is;
  int check_state;
  long long* prof;   // optional (debug): clock64 stamps of CTA 0 per step and phase, 8 per step
};

__device__ __forceinline__ void trd_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned trd_mapa(const void* p, int rank) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void trd_push(unsigned raddr, double v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void trd_bar_init(uint64_t* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
}
__device__ __forceinline__ void trd_bar_expect(uint64_t* bar, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void trd_bar_wait(uint64_t* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  unsigned ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(b), "r"(parity)
                 : "memory");
}
__device__ __forceinline__ unsigned trd_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// fixed-order sum of p[c * stride], c < n (n <= 16), as a balanced tree (same order everywhere)
__device__ __forceinline__ double trd_sum16(const double* p, int n, int stride) {
  double v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) v[c] = (c < n) ? p[c * stride] : 0.0;
#pragma unroll
  for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
    for (int c = 0; c < h; ++c) v[c] += v[c + h];
  return v[0];
}

// fixed-order block sum over TRD_NT threads; result valid in every thread
__device__ __forceinline__ double trd_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  return trd_sum16(red, TRD_NW, 1);
}

// Shared-memory layout (doubles): xt[2][N] wb[N] | per own slot (S = ceil(N/C)): vown[2][S] wown[S]
// pown[S] xs[S] qr[C][S] rp[NW][S] | scalars sd[C] se[C] ss[C] red[32] | rows.
__host__ __device__ inline long long trd_fixed_doubles(int N, int C) {
  const int S = (N + C - 1) / C;
  return 3LL * N + 5LL * S + (long long)C * S + (long long)TRD_NW * S + 3LL * C + 32;
}

template <int MAXB>
__global__ void __launch_bounds__(TRD_NT, 1) k_tridiag(TridiagArgs a) {
  if (a.check_state && (a.st->done || !a.is->proceed)) return;
  const int C = a.C, N = a.N;
  const int me = (int)trd_cluster_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 3, cc = lane & 7;
  const int S = (N + C - 1) / C;
  extern __shared__ __align__(16) double sm[];
  double* xt = sm;                 // [2][N] x~_k: the column that defines v_k (allgathered), by parity
  double* wb = xt + 2 * N;         // w_{k-1} (allgathered)
  double* vown = wb + N;           // [2][S] v_k on own rows, by step parity
  double* wown = vown + 2 * S;     // w on own rows
  double* pown = wown + S;         // own row dots
  double* xs = pown + S;           // updated column on own rows (Phase Y)
  double* qr = xs + S;             // [C][S] reduce-scatter receive
  double* rp = qr + C * S;         // [NW][S] per-warp row partials
  double* sd = rp + TRD_NW * S;    // [C] partial v^T A v
  double* se = sd + C;             // [C] partial (A v)[k+1]
  double* ss = se + C;             // [C] partial ||x~||^2
  double* red = ss + C;            // [32]: warp partials (two independent halves)
  double* rows = red + 32;
  __shared__ int roff[TRD_MAXOWN];  // smem offset of own row slot q, -1 = spilled to global
  __shared__ int nspill_s;
  __shared__ double qk1_s;
  __shared__ __align__(8) uint64_t barQ, barY;

  const int nown = (N - me + C - 1) / C;  // own rows i = me + q C
  auto first_slot = [&](int m) { return (m - me + C - 1) / C > 0 ? (m - me + C - 1) / C : 0; };  // i >= m
  if (tid == 0) {
    // smallest rows spill first; rows are stored whole (entries 0..i)
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
  for (int q = nspill; q < nown; ++q) {
    const int i = me + q * C;
    const double* src = a.M + (size_t)i * N;  // upper triangle of column i = row i of the lower
    double* dst = rows + roff[q];
    for (int j = tid; j <= i; j += TRD_NT) dst[j] = src[j];
  }
  for (int j = tid; j < N; j += TRD_NT) wb[j] = 0.0;
  for (int q = tid; q < 2 * S; q += TRD_NT) vown[q] = 0.0;
  for (int q = tid; q < S; q += TRD_NT) wown[q] = 0.0;
  trd_cluster_sync();  // barriers initialised and every CTA running before the first remote store

  auto rowptr_g = [&](int q) -> double* { return a.M + (size_t)(me + q * C) * N; };
  auto rowptr_s = [&](int q) -> double* { return rows + roff[q]; };
  auto rowval = [&](int q, int j) -> double {  // entry (i, j) of own row slot q
    return q < nspill ? rowptr_g(q)[j] : rowptr_s(q)[j];
  };

  // ---- column 0 defines v_0: push x~_0 = A[1:, 0], ||A[2:, 0]||^2 partials; d[0] ----
  if (tid == 0) trd_bar_expect(&barY, (unsigned)(8 * ((N - 1) + C)));
  {
    double s2 = 0.0;
    for (int q = tid; q < nown; q += TRD_NT) {
      const int i = me + q * C;
      const double x = rowval(q, 0);
      xs[q] = x;
      if (i >= 2) s2 = fma(x, x, s2);
      if (i == 0) a.d[0] = x;
    }
    s2 = trd_block_sum(s2, red);
    for (int e = tid; e < nown * C; e += TRD_NT) {
      const int q = e / C, peer = e % C, i = me + q * C;
      if (i >= 1) trd_push(trd_mapa(xt + i, peer), xs[q], trd_mapa(&barY, peer));
    }
    if (tid < C) trd_push(trd_mapa(ss + me, tid), s2, trd_mapa(&barY, tid));
  }
  trd_bar_wait(&barY, 0);

  double scale_prev = 0.0;
  const bool prof = a.prof != nullptr && me == 0 && tid == 0;
#define TRD_STAMP(ph) \
  if (prof) a.prof[(size_t)k * 8 + (ph)] = clock64();
  for (int k = 0; k < N - 2; ++k) {
    const int par = k & 1;
    TRD_STAMP(0)
    const double* xk = xt + par * N;          // x~_k
    const double* xkm = xt + (par ^ 1) * N;   // x~_{k-1}
    const int qs1 = first_slot(k + 1), qs2 = first_slot(k + 2);
    if (tid == 0) trd_bar_expect(&barQ, (unsigned)(8 * (C * (nown - qs2) + 2 * C)));
    // ---- Phase A: the reflector of column k (every CTA computes it redundantly, same order) ----
    const double sig = trd_sum16(ss, C, 1);
    const double alpha = xk[k + 1];
    double tk, beta, scale;
    if (sig == 0.0) {
      tk = 0.0;
      beta = alpha;
      scale = 0.0;
    } else {
      beta = -copysign(sqrt(fma(alpha, alpha, sig)), alpha);
      tk = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (me == k % C) {
      for (int j = k + 1 + tid; j < N; j += TRD_NT) a.V[(size_t)k * N + j] = (j == k + 1) ? 1.0 : xk[j] * scale;
      if (tid == 0) {
        a.e[k] = beta;
        a.tau[k] = tk;
      }
    }
    double* vcur = vown + par * S;
    const double* vprev = vown + (par ^ 1) * S;
    for (int q = qs1 + tid; q < nown; q += TRD_NT) {
      const int i = me + q * C;
      vcur[q] = (i == k + 1) ? 1.0 : xk[i] * scale;
    }
    // this lane's columns: blocks bb = warp + 16 t of 8 columns starting at k + 1
    const int nb = (N - k - 1 + 7) / 8;
    const int nbt = nb > warp ? (nb - warp + TRD_NW - 1) / TRD_NW : 0;  // blocks of this warp
    double vn[MAXB], vo[MAXB], wo[MAXB], qa[MAXB];
#pragma unroll
    for (int t = 0; t < MAXB; ++t) {
      const int j = k + 1 + 8 * (warp + TRD_NW * t) + cc;
      const bool ok = t < nbt && j < N;
      vn[t] = !ok ? 0.0 : (j == k + 1 ? 1.0 : xk[j] * scale);
      vo[t] = ok ? xkm[j] * scale_prev : 0.0;  // scale_prev = 0 at k = 0: no pending update
      wo[t] = ok ? wb[j] : 0.0;
      qa[t] = 0.0;
    }
    __syncthreads();
    TRD_STAMP(1)

    // ---- Phase X: fused rank-2 update of step k-1 and symv with v_k over own rows i >= k+1 ----
    // rows in groups of 4 (lane row lr), processed from slot qb to qe with row pointers from rp_of
    auto row_groups = [&](int qb, int qe, auto rp_of) {
      for (int g = qb; g < qe; g += 4) {
        const int q = min(g + lr, qe - 1);
        const bool valid = g + lr < qe;
        const int i = valid ? me + q * C : -1;
        const int imin = me + g * C;                   // smallest row of the group (uniform)
        const int imax = me + min(g + 3, qe - 1) * C;  // largest row of the group (uniform)
        double* R = rp_of(q);
        const double vio = vprev[q], wio = wown[q], vin = vcur[q];
        double racc = 0.0;
#pragma unroll
        for (int t = 0; t < MAXB; ++t) {
          const int jf = k + 1 + 8 * (warp + TRD_NW * t);
          if (t >= nbt || jf > imax) break;  // this and all later blocks lie right of the group's diagonal
          const int j = jf + cc;
          if (jf + 7 < imin) {  // strictly below every row's diagonal: no masking
            double x = R[j];
            x = fma(-vio, wo[t], fma(-wio, vo[t], x));
            R[j] = x;
            racc = fma(x, vn[t], racc);
            qa[t] = fma(x, vin, qa[t]);
          } else if (j <= i) {
            double x = R[j];
            x = fma(-vio, wo[t], fma(-wio, vo[t], x));
            R[j] = x;
            racc = fma(x, vn[t], racc);
            qa[t] = fma(x, (j < i) ? vin : 0.0, qa[t]);
          }
        }
        racc += __shfl_xor_sync(0xffffffffu, racc, 1);
        racc += __shfl_xor_sync(0xffffffffu, racc, 2);
        racc += __shfl_xor_sync(0xffffffffu, racc, 4);
        if (valid && cc == 0) rp[warp * S + q] = racc;
      }
    };
    if (qs1 < nspill) row_groups(qs1, nspill, rowptr_g);
    row_groups(max(qs1, nspill), nown, rowptr_s);
    TRD_STAMP(2)
    // column sums over the 4 row lanes; lanes with lr == 0 hold q[j] for their 8-column blocks
    double dpart = 0.0;
#pragma unroll
    for (int t = 0; t < MAXB; ++t) {
      if (t >= nbt) break;
      double v = qa[t];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      qa[t] = v;
      if (lr == 0) dpart = fma(v, vn[t], dpart);
    }
    if (warp == 0 && lane == 0) qk1_s = qa[0];  // column k+1 (block 0, cc 0)
    // reduce-scatter of the transposed partials: column j's partial goes to the owner of row j
    if (lr == 0) {
#pragma unroll
      for (int t = 0; t < MAXB; ++t) {
        if (t >= nbt) break;
        const int j = k + 1 + 8 * (warp + TRD_NW * t) + cc;
        if (j >= k + 2 && j < N) {
          const int peer = j % C;
          trd_push(trd_mapa(qr + me * S + j / C, peer), qa[t], trd_mapa(&barQ, peer));
        }
      }
    }
    __syncthreads();
    TRD_STAMP(3)
    for (int q = qs1 + tid; q < nown; q += TRD_NT) {
      const double s = trd_sum16(rp + q, TRD_NW, S);
      pown[q] = s;
      dpart = fma(s, vcur[q], dpart);
    }
    dpart = warp_sum(dpart);
    if (lane == 0) red[warp] = dpart;
    __syncthreads();
    TRD_STAMP(4)
    if (tid < C) {
      const double dsum = trd_sum16(red, TRD_NW, 1);
      double e1 = qk1_s;
      if ((k + 1) % C == me) e1 += pown[(k + 1) / C];
      const unsigned rb = trd_mapa(&barQ, tid);
      trd_push(trd_mapa(sd + me, tid), dsum, rb);
      trd_push(trd_mapa(se + me, tid), e1, rb);
    }
    const bool last = (k == N - 3);
    if (tid == 0 && !last) trd_bar_expect(&barY, (unsigned)(8 * (2 * (N - k - 2) + C)));
    trd_bar_wait(&barQ, par);
    TRD_STAMP(5)

    // ---- Phase Y: w_k on own rows, eager update of column k+1, its norm partial ----
    const double sdv = trd_sum16(sd, C, 1), sev = trd_sum16(se, C, 1);
    const double Kc = 0.5 * tk * tk * sdv;   // (tau/2) p^T v with p = tau A v
    const double wk1 = tk * sev - Kc;       // w_k[k+1] (v_k[k+1] = 1)
    double s2 = 0.0;
    for (int q = qs1 + tid; q < nown; q += TRD_NT) {
      const int i = me + q * C;
      if (i == k + 1) {
        a.d[k + 1] = rowval(q, k + 1) - 2.0 * wk1;
        wown[q] = wk1;
        continue;
      }
      const double pq = pown[q] + trd_sum16(qr + q, C, S);
      const double wi = fma(-Kc, vcur[q], tk * pq);
      wown[q] = wi;
      double* R = q < nspill ? rowptr_g(q) : rowptr_s(q);
      const double x = fma(-vcur[q], wk1, R[k + 1] - wi);
      R[k + 1] = x;
      xs[q] = x;
      if (i >= k + 3) s2 = fma(x, x, s2);
      if (last) {  // i == N - 1: the trailing 2 x 2 block
        a.e[N - 2] = x;
        a.d[N - 1] = R[N - 1] - 2.0 * vcur[q] * wi;
        a.tau[N - 2] = 0.0;
      }
    }
    if (last) break;
    TRD_STAMP(6)
    s2 = warp_sum(s2);
    if (lane == 0) red[16 + warp] = s2;  // second half of red: no conflict with the dsum partials
    {
      double* xnext = xt + (par ^ 1) * N;
      const int nact = nown - qs2;  // own rows >= k+2
      for (int e = tid; e < nact * C; e += TRD_NT) {
        const int q = qs2 + e / C, peer = e % C, i = me + q * C;
        const unsigned rb = trd_mapa(&barY, peer);
        trd_push(trd_mapa(xnext + i, peer), xs[q], rb);
        trd_push(trd_mapa(wb + i, peer), wown[q], rb);
      }
    }
    __syncthreads();
    if (tid < C) trd_push(trd_mapa(ss + me, tid), trd_sum16(red + 16, TRD_NW, 1), trd_mapa(&barY, tid));
    scale_prev = scale;
    TRD_STAMP(7)
    trd_bar_wait(&barY, par ^ 1);
  }
#undef TRD_STAMP
  trd_cluster_sync();  // no CTA leaves while a peer may still address its shared memory
}

inline size_t tridiag_smem_bytes(int N, int C, long long row_doubles) {
  return sizeof(double) * (size_t)(trd_fixed_doubles(N, C) + row_doubles);
}

typedef void (*TridiagKernel)(TridiagArgs);
inline TridiagKernel tridiag_kernel(int N) {
  switch (tridiag_maxb(N)) {
    case 2: return k_tridiag<2>;
    case 4: return k_tridiag<4>;
    case 7: return k_tridiag<7>;
    default: return k_tridiag<10>;
  }
}
