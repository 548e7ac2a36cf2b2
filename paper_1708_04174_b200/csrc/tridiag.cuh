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
#include <type_traits>

#include "common.cuh"

constexpr int TRD_NT = 512;
constexpr int TRD_NW = TRD_NT / 32;
constexpr int TRD_MAXC = 16;
constexpr int TRD_MAXOWN = 256;  // own rows per CTA (the single-CTA tail owns every trailing row)
// Phase X thread mapping: lane = (lr, cc), lr = lane / 8 picks one of 4 rows of a row group, cc one
// of 8 consecutive columns of a column block; warp w owns column blocks w, w + 16, w + 32, ...
// (MAXB of them), so row sums reduce over 8 lanes and column sums over 4 lanes only.
inline int tridiag_maxb(int N) {
  const int nb = ((N - 1) + 7) / 8;
  const int m = (nb + TRD_NW - 1) / TRD_NW;
  return m <= 2 ? 2 : (m <= 4 ? 4 : (m <= 7 ? 7 : 10));
}

struct TridiagArgs {
  double* M;         // N x N column-major block matrix (upper triangle valid on input)
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
  int kb, ke;        // Householder steps [kb, ke) done by this launch
  double* hand;      // 3 N + 2 doubles: head -> tail hand-over state
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
__device__ __forceinline__ void trd_push2(unsigned raddr, double v0, double v1, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(v0), "d"(v1), "r"(rbar)
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
  unsigned ok = 0, spins = 0;
  unsigned long long t0 = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(b), "r"(parity)
                 : "memory");
    // a lost exchange is a bug: fail loudly instead of hanging the GPU — but only after 20 s of wall
    // clock (%globaltimer), so time-slicing / MPS contention can never trip it on a correct exchange
    if (!ok && (++spins & 0xFFFFu) == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > 20000000000ull) __trap();
    }
  }
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

// Column block of warp w's t-th slot: a "snake" order (w, 31 - w, 32 + w, 63 - w, ...) so that the
// triangular work (block bb covers rows >= 8 bb) is balanced over the warps; increasing in t.
__device__ __forceinline__ int trd_block(int w, int t) { return TRD_NW * t + ((t & 1) ? TRD_NW - 1 - w : w); }

// fixed-order sum of p[0..n), n <= 16, over the lanes of a warp (xor tree within each half-warp;
// every lane gets the result, the same value in every warp and CTA)
__device__ __forceinline__ double trd_lane_sum16(const double* p, int n) {
  const int l = threadIdx.x & 15;  // both half-warps compute the same sum
  double v = (l < n) ? p[l] : 0.0;
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

// fixed-order sum of p[0..CC) (compile-time count: unrolled, unpredicated loads and a balanced tree)
template <int CC>
__device__ __forceinline__ double trd_sumc(const double* p) {
  double v[CC];
#pragma unroll
  for (int c = 0; c < CC; ++c) v[c] = p[c];
#pragma unroll
  for (int h = CC / 2; h >= 1; h >>= 1)
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

// Shared-memory layout (doubles): xw[2][N] (double2: x~_k[j], scale_{k-1} w_{k-1}[j], by step
// parity) | per own slot (S slots): xs[S] qr[C][S] rp[NW][S] | scalars sd[C] se[C] sc[C] red[32] | rows.
__host__ __device__ inline long long trd_fixed_doubles(int N, int C, int S) {
  return 4LL * N + 2LL * C + (long long)S + (long long)C * S + (long long)TRD_NW * S + 32;
}
__host__ __device__ inline int trd_log2(int C) { return C >= 16 ? 4 : (C >= 8 ? 3 : (C >= 4 ? 2 : (C >= 2 ? 1 : 0))); }

// k_tridiag<MAXB, CC> runs Householder steps [kb, ke) of one block; CC is the cluster size (compile
// time, so every fixed-order C-term sum is an unrolled tree), CC = 1 the single-CTA variant (SOLO).
//   cluster head (SOLO = false, C in {4,8,16}, kb = 0): if ke < N - 2 it stops after step ke - 1 and
//     hands its state over through global memory: the unfinished trailing rows i >= ke (entries
//     ke..i, still owing the lazy rank-2 update of step ke - 1) go back to the block matrix, and
//     hand[] = [x~_ke (N), x~_{ke-1} (N), scale_{ke-1} w_{ke-1} (N)];
//   single-CTA tail (SOLO = true, C = 1, kb = ke of the head): resumes from that state with local
//     stores and __syncthreads in place of the DSMEM exchanges.
// Scalar work is done by one warp (reflector) or by the own-row threads (Phase Y) only; the other
// warps only run the fused pass and the exchanges (redundant FP64 div/sqrt in 16 warps cost issue
// slots, measured).  v_k on a row is recomputed as x~_k[i] * scale_k (1 at row k+1).
template <int MAXB, int CC>
__global__ void __launch_bounds__(TRD_NT, 1) k_tridiag(TridiagArgs a) {
  if (a.check_state && (a.st->done || !a.is->proceed)) return;
  constexpr bool SOLO = CC == 1;
  constexpr int C = CC;
  constexpr int logC = CC >= 16 ? 4 : (CC >= 8 ? 3 : (CC >= 4 ? 2 : (CC >= 2 ? 1 : 0)));
  const int N = a.N;
  const int kb = a.kb, ke = min(a.ke, N - 2);
  const int me = SOLO ? 0 : (int)trd_cluster_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 3, cc = lane & 7;
  const int nown = (N - me + C - 1) >> logC;  // own rows i = me + q C
  auto first_slot = [&](int m) { return m > me ? (m - me + C - 1) >> logC : 0; };  // first q with i >= m
  const int qlo = first_slot(kb);             // rows below kb are finished before this launch
  // per-slot arrays are indexed q - qlo; S must be the same in every CTA of the cluster (the DSMEM
  // exchange addresses are computed from the local layout)
  const int S = SOLO ? N - kb : (N + C - 1) >> logC;
  const int jb = kb;                          // row storage starts at column kb
  extern __shared__ __align__(16) double sm[];
  // xw[par][j] = (x~_k[j], w_{k-1}[j]) for k of parity par: x~_k is the column that defines v_k,
  // w_{k-1} the pending update; both allgathered in ONE 16-byte st.async per (row, peer)
  double2* xw = reinterpret_cast<double2*>(sm);
  // [C] per-CTA partials of (v^T A v, (A v)[k+1]), already scaled (one 16-byte push per peer)
  double2* sde = reinterpret_cast<double2*>(sm + 4 * (size_t)N);
  double* xs = sm + 4 * (size_t)N + 2 * C;  // column 0 on own rows (first push)
  double* qr = xs + S;             // [C][S] reduce-scatter receive
  double* rp = qr + C * S;         // [NW][S] per-warp row partials
  double* red = rp + TRD_NW * S;   // [32]: warp partials (two independent halves)
  double* rows = red + 32;
  __shared__ int roff[TRD_MAXOWN];  // smem offset of own row slot q - qlo, -1 = spilled to global
  __shared__ int nspill_s;
  __shared__ double qk1_s, scal_s[2][2];  // (tau_k, scale_k) by step parity
  __shared__ __align__(8) uint64_t barQ, barY;

  if (tid == 0) {
    // smallest rows spill first; rows are stored from column jb to the diagonal.  Consecutive rows
    // start 8 doubles apart modulo 16 (<= 15 doubles of padding each), so the two rows a half-warp
    // touches in one 8-column block (lanes lr = 0, 1 or 2, 3) fall in disjoint bank halves.
    long long need = 0;
    for (int q = qlo; q < nown; ++q) need += me + q * C + 1 - jb + 15;
    int ns = qlo;
    while (need > a.smem_rows_doubles && ns < nown) {
      need -= me + ns * C + 1 - jb + 15;
      ++ns;
    }
    long long off = 0, prev = -1;
    for (int q = qlo; q < nown; ++q) {
      if (q < ns) {
        roff[q - qlo] = -1;
      } else {
        if (prev >= 0) off += (((prev + 8 - off) % 16) + 16) % 16;
        roff[q - qlo] = (int)off;
        prev = off;
        off += me + q * C + 1 - jb;
      }
    }
    nspill_s = ns;
    if (!SOLO) {
      trd_bar_init(&barQ);
      trd_bar_init(&barY);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const int nspill = nspill_s;
  // Phase Y maps YP threads to every own row slot: S * YP <= TRD_NT holds for every supported size
  // (N <= SOSADMM_MAX_BLOCK = 1280: S <= 80 with C = 16, YP = 4); fail loudly otherwise
  if (S * (CC >= 16 ? 4 : (CC >= 4 ? 2 : 1)) > TRD_NT) __trap();
  auto rowptr_g = [&](int q) -> double* { return a.M + (size_t)(me + q * C) * N; };
  auto rowptr_s = [&](int q) -> double* { return rows + roff[q - qlo] - jb; };
  auto rowval = [&](int q, int j) -> double {  // entry (i, j) of own row slot q
    return q < nspill ? rowptr_g(q)[j] : rowptr_s(q)[j];
  };
  for (int q = nspill; q < nown; ++q) {
    const int i = me + q * C;
    const double* src = a.M + (size_t)i * N;  // upper triangle of column i = row i of the lower
    double* dst = rowptr_s(q);
    for (int j = jb + tid; j <= i; j += TRD_NT) dst[j] = src[j];
  }
  if (kb == 0) {
    for (int j = tid; j < 2 * N; j += TRD_NT) xw[j] = make_double2(0.0, 0.0);  // x~_{-1}, w_{-1} = 0
  } else {  // resume from the head's hand-over state
    const int pk = kb & 1;
    for (int j = tid; j < N; j += TRD_NT) {
      xw[pk * N + j] = make_double2(a.hand[j], a.hand[2 * N + j]);
      xw[(pk ^ 1) * N + j] = make_double2(a.hand[N + j], 0.0);
    }
  }
  if (!SOLO) trd_cluster_sync();  // barriers initialised and every CTA running before the first remote store
  else __syncthreads();

  // exchange primitives: SOLO = plain local stores (the waits are __syncthreads)
  auto push = [&](double* dst, int peer, double v, uint64_t* bar) {
    if (SOLO) *dst = v;
    else trd_push(trd_mapa(dst, peer), v, trd_mapa(bar, peer));
  };
  auto push2 = [&](double2* dst, int peer, double v0, double v1, uint64_t* bar) {
    if (SOLO) *dst = make_double2(v0, v1);
    else trd_push2(trd_mapa(dst, peer), v0, v1, trd_mapa(bar, peer));
  };

  if (kb == 0) {
    // ---- column 0 defines v_0: push x~_0 = A[1:, 0] (allgather); d[0] ----
    if (!SOLO && tid == 0) trd_bar_expect(&barY, (unsigned)(16 * (N - 1)));  // (x, 0) pairs
    for (int q = tid; q < nown; q += TRD_NT) {
      const int i = me + q * C;
      const double x = rowval(q, 0);
      xs[q] = x;
      if (i == 0) a.d[0] = x;
    }
    __syncthreads();
    for (int e = tid; e < nown * C; e += TRD_NT) {
      const int q = e >> logC, peer = e & (C - 1), i = me + q * C;
      if (i >= 1) push2(xw + i, peer, xs[q], 0.0, &barY);
    }
    if (!SOLO) trd_bar_wait(&barY, 0);
    else __syncthreads();
  }

  const bool prof = a.prof != nullptr && me == 0 && tid == 0;
#define TRD_STAMP(ph) \
  if (prof) a.prof[(size_t)k * 16 + (ph)] = clock64();
  // Steps run through the smallest column-block variant that covers the trailing matrix: MB blocks
  // per warp while nb > 16 * (next smaller MB), so late steps carry fewer register arrays and
  // shorter unrolled loops (the variants share all state; k advances inside).
  int k = kb;
  auto run = [&](auto MBc, int nb_min) -> bool {
    constexpr int MB = decltype(MBc)::value;
    for (; k < ke; ++k) {
      if (((N - k - 1 + 7) >> 3) <= nb_min) return false;
      const int par = k & 1;
      TRD_STAMP(0)
      const double2* xwk = xw + par * N;         // (x~_k, w_{k-1})
      const double2* xwm = xw + (par ^ 1) * N;   // (x~_{k-1}, .)
      auto xk = [&](int j) { return xwk[j].x; };
      auto xkm = [&](int j) { return xwm[j].x; };
      const int qs1 = first_slot(k + 1), qs2 = first_slot(k + 2);
      const int nb = (N - k - 1 + 7) >> 3;      // 8-column blocks of the trailing matrix
      auto nwarps_of_row = [&](int i) { return min(min(TRD_NW, nb), (i - k - 1) / 8 + 1); };  // warps reaching row i
      // Deferred scaling: the reflector v_k = e_{k+1} + scale_k y with y = x~_k[k+2:] (the pivot entry
      // zeroed), so the fused pass computes z = A_k y with the UNSCALED column and needs none of the
      // reflector scalars; p = A_k v_k = A_k[:, k+1] + scale_k z and v^T A v = A_k[k+1,k+1]
      // + 2 scale z[k+1] + scale^2 y^T z are formed per own row in Phase Y, and the sqrt / division
      // chain of the reflector is off the critical path.
      // The chain runs on the LAST warp at the top of the step: its column blocks start furthest right,
      // so it has the least fused-pass work (none once fewer than 16 blocks remain).  It sums
      // ||x~_k[k+2:]||^2 itself from the allgathered column (same order in every CTA: no norm
      // exchange).  scal_s is double-buffered by step parity (read after the next __syncthreads).
      if (warp == TRD_NW - 1) {
        // beta = -sign(alpha) sqrt(n2), tau = 1 + |alpha| / sqrt(n2), scale = 1 / (alpha - beta)
        // = sign(alpha) / (|alpha| + sqrt(n2)): one rsqrt + one division
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int j = k + 2 + lane;
        for (; j + 96 < N; j += 128) {
          const double x0 = xk(j), x1 = xk(j + 32), x2 = xk(j + 64), x3 = xk(j + 96);
          s0 = fma(x0, x0, s0);
          s1 = fma(x1, x1, s1);
          s2 = fma(x2, x2, s2);
          s3 = fma(x3, x3, s3);
        }
        for (; j < N; j += 32) {
          const double x0 = xk(j);
          s0 = fma(x0, x0, s0);
        }
        const double sig = warp_sum((s0 + s1) + (s2 + s3));
        const double alpha = xk(k + 1);
        double tk = 0.0, beta = alpha, scale = 0.0;
        if (sig != 0.0) {
          const double n2 = fma(alpha, alpha, sig);
          const double rs = rsqrt(n2);
          const double nrm = n2 * rs;
          beta = -copysign(nrm, alpha);
          tk = fma(fabs(alpha), rs, 1.0);
          scale = copysign(1.0, alpha) / (fabs(alpha) + nrm);
        }
        if (lane == 0) {
          scal_s[par][0] = tk;
          scal_s[par][1] = scale;
          if (me == (k & (C - 1))) {
            a.e[k] = beta;
            a.tau[k] = tk;
          }
        }
      }
      // this lane's columns: blocks bb = warp + 16 t of 8 columns starting at k + 1
      int nbt = 0;  // blocks of this warp (trd_block is increasing in t)
    #pragma unroll
      for (int t = 0; t < MB; ++t) nbt += trd_block(warp, t) < nb ? 1 : 0;
      double vn[MB], vo[MB], wo[MB], qa[MB];
    #pragma unroll
      for (int t = 0; t < MB; ++t) {
        const int j = k + 1 + 8 * trd_block(warp, t) + cc;
        const bool ok = t < nbt && j < N;
        const double2 cw = ok ? xwk[j] : make_double2(0.0, 0.0);
        vn[t] = (j == k + 1) ? 0.0 : cw.x;       // y[j]
        vo[t] = ok ? xkm(j) : 0.0;               // x~_{k-1}[j] (v_{k-1} = scale_{k-1} x~_{k-1} below row k)
        wo[t] = cw.y;                            // scale_{k-1} w_{k-1}[j] (0 at k = 0: no pending update)
        qa[t] = 0.0;
      }
      if (tid == 32 && !SOLO) trd_bar_expect(&barQ, (unsigned)(8 * (C * (nown - qs2) + 2 * C)));
      TRD_STAMP(1)

      // ---- Phase X: fused rank-2 update of step k-1 and symv with v_k over own rows i >= k+1 ----
      double dpart = 0.0;  // this thread's share of v^T A v (row part: racc v_i; column part: q_j v_j)
      const int qw = first_slot(k + 1 + 8 * warp);  // a warp only visits rows reaching its first block
      // one group of 4 rows (lane row lr); FULL = all four rows exist (every group but possibly the
      // last), which removes every per-lane validity test from the unmasked path
      auto row_group = [&](int g, int qe, auto rp_of, auto FULL) {
        constexpr bool full = decltype(FULL)::value;
        const int q = full ? g + lr : min(g + lr, qe - 1);
        const bool valid = full || g + lr < qe;
        const int ic = me + q * C;                     // row (clamped on the padding lanes)
        const int i = valid ? ic : -1;
        const int imin = me + g * C;                   // smallest row of the group (uniform)
        const int imax = me + (full ? g + 3 : min(g + 3, qe - 1)) * C;  // largest row of the group (uniform)
        double* R = rp_of(q);
        const double vio = xkm(ic);                    // x~_{k-1}[i], i >= k + 1
        const double vin = (ic == k + 1) ? 0.0 : xk(ic);  // y[i]
        const double wio = xwk[ic].y;                  // scale_{k-1} w_{k-1}[i]
        double racc = 0.0;
    #pragma unroll
        for (int t = 0; t < MB; ++t) {
          const int jf = k + 1 + 8 * trd_block(warp, t);
          if (t >= nbt || jf > imax) break;  // this and all later blocks lie right of the group's diagonal
          const int j = jf + cc;
          if (jf + 7 < imin) {  // strictly below every row's diagonal: no column masking
            if (full || valid) {
              double x = R[j];
              x = fma(-vio, wo[t], fma(-wio, vo[t], x));
              R[j] = x;
              racc = fma(x, vn[t], racc);
              qa[t] = fma(x, vin, qa[t]);
            }
          } else if (j <= i) {  // i = -1 on the padding lanes of the last group
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
        if (valid && cc == 0) {
          rp[warp * S + q - qlo] = racc;
          dpart = fma(racc, vin, dpart);
        }
      };
      auto row_groups = [&](int qb, int qe, auto rp_of) {
        if (nbt == 0) return;
        int g = max(qb, qw);
    #pragma unroll 2
        for (; g + 4 <= qe; g += 4) row_group(g, qe, rp_of, std::true_type());
        if (g < qe) row_group(g, qe, rp_of, std::false_type());
      };
      if (qs1 < nspill) row_groups(qs1, nspill, rowptr_g);
      row_groups(max(qs1, nspill), nown, rowptr_s);
      TRD_STAMP(2)
      // column sums over the 4 row lanes; lanes with lr == 0 hold q[j] for their 8-column blocks
    #pragma unroll
      for (int t = 0; t < MB; ++t) {
        if (t >= nbt) break;
        double v = qa[t];
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        qa[t] = v;
        if (lr == 0) dpart = fma(v, vn[t], dpart);
      }
      if (warp == 0 && lane == 0) qk1_s = qa[0];  // column k+1 (block 0, cc 0)
      // reduce-scatter of the transposed partials: column j's partial goes to the owner of row j.
      // After the column sums every row lane holds all of its blocks' sums, so the 4 row lanes
      // split the blocks (lane row lr sends block 4 g + lr): one 32-lane push per 4 blocks
    #pragma unroll
      for (int g = 0; g < (MB + 3) / 4; ++g) {
        if (4 * g >= nbt) break;
        double v = 0.0;
        int t = 4 * g;
    #pragma unroll
        for (int u = 1; u < 4; ++u)
          if (4 * g + u < MB && lr == u) t = 4 * g + u;
    #pragma unroll
        for (int u = 0; u < 4; ++u)
          if (4 * g + u < MB && lr == u) v = qa[4 * g + u];
        const int j = k + 1 + 8 * trd_block(warp, t) + cc;
        if (4 * g + lr < MB && t < nbt && j >= k + 2 && j < N)  // row lanes past the last block stay idle
          push(qr + me * S + (j >> logC) - qlo, j & (C - 1), v, &barQ);
      }
      dpart = warp_sum(dpart);
      if (lane == 0) red[warp] = dpart;
      __syncthreads();
      TRD_STAMP(3)
      const bool own1 = ((k + 1) & (C - 1)) == me;  // this CTA owns row k + 1
      if (tid < C) {
        // scale_k is known here (scal_s, before the last __syncthreads), so each CTA pushes its share
        // of v^T A v = c1 + 2 scale z1 + scale^2 y^T z and of p[k+1] = c1 + scale z1 directly, the
        // owner of row k + 1 adding c1 = A_k[k+1, k+1]: one st.async per peer
        const double scl = scal_s[par][1];
        const double yzp = trd_sumc<TRD_NW>(red), z1p = qk1_s;
        const double c1p = own1 ? rowval((k + 1) >> logC, k + 1) : 0.0;
        push2(sde + me, tid, fma(scl, fma(scl, yzp, 2.0 * z1p), c1p), fma(scl, z1p, c1p), &barQ);
      }
      TRD_STAMP(4)
      const bool last = (k == N - 3);
      const int nslot = nown - qs1;
      // Phase Y runs YP threads per own row (each pushes to C / YP of the peers)
      constexpr int YP = CC >= 16 ? 4 : (CC >= 4 ? 2 : 1);  // measured: 1 / 2 / 4 -> 4.59 / 4.58 / 4.55 ms
      const int yq = tid / YP, yh = tid % YP;
      double prow_own = 0.0;  // this CTA's row dot of its own row (sum over the warps), before the wait
      if (yq < nslot) {
        const int i = me + (qs1 + yq) * C;
        if (i > k + 1) prow_own = trd_sum16(rp + qs1 + yq - qlo, nwarps_of_row(i), S);
      }
      const double tk = scal_s[par][0], scale = scal_s[par][1];  // written before the last __syncthreads
      TRD_STAMP(8)
      if (!SOLO) {
        if (tid == 0 && !last) trd_bar_expect(&barY, (unsigned)(16 * (N - k - 2)));
        trd_bar_wait(&barQ, par);
      } else {
        __syncthreads();
      }
      TRD_STAMP(5)

      // ---- Phase Y (own-row threads): w_k, eager update of column k+1, its norm partial ----
      double Kc = 0.0, wk1 = 0.0;
      if (yq < nslot) {
        double vv[CC], pp[CC];  // fixed-order sums of the C partials
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          const double2 t = sde[c];
          vv[c] = t.x;
          pp[c] = t.y;
        }
#pragma unroll
        for (int h = CC / 2; h >= 1; h >>= 1)
#pragma unroll
          for (int c = 0; c < h; ++c) {
            vv[c] += vv[c + h];
            pp[c] += pp[c + h];
          }
        Kc = 0.5 * tk * tk * vv[0];             // (tau/2) p^T v with p = tau A v; vv[0] = v^T A v
        wk1 = fma(tk, pp[0], -Kc);               // w_k[k+1] (v_k[k+1] = 1); pp[0] = (A v)[k+1]
      }
      TRD_STAMP(10)
      // each own-row thread pushes its (x~_{k+1}[i], scale_k w_k[i]) straight to every CTA (allgather;
      // peers staggered so the 16 stores of a warp hit 16 different CTAs)
      double2* xnext = xw + (par ^ 1) * N;  // (x~_{k+1}, scale_k w_k)
      auto phase_y = [&](int q, double* R, double prow) {
        const int i = me + q * C;
        if (i == k + 1) {
          if (yh == 0) a.d[k + 1] = R[k + 1] - 2.0 * wk1;
        } else {
          const double vin = xk(i) * scale;
          const double pq = fma(scale, prow + trd_sum16(qr + q - qlo, C, S), R[k + 1]);  // (A v)[i]
          const double wi = fma(-Kc, vin, tk * pq);
          const double x = fma(-vin, wk1, R[k + 1] - wi);
          if (last) {  // i == N - 1: the trailing 2 x 2 block
            if (yh == 0) {
              R[k + 1] = x;
              a.e[N - 2] = x;
              a.d[N - 1] = R[N - 1] - 2.0 * vin * wi;
              a.tau[N - 2] = 0.0;
            }
          } else {
            const double ws = wi * scale;
    #pragma unroll
            for (int c = 0; c < C / YP; ++c) push2(xnext + i, (c * YP + yh + yq) & (C - 1), x, ws, &barY);
          }
        }
      };
      if (yq < nslot) {
        const int q = qs1 + yq;
        if (q < nspill) phase_y(q, rowptr_g(q), prow_own);
        else phase_y(q, rowptr_s(q), prow_own);
      }
      TRD_STAMP(11)
      if (me == (k & (C - 1)))  // v_k for the back-transform (global, read by later kernels only)
        for (int j = k + 1 + tid; j < N; j += TRD_NT) a.V[(size_t)k * N + j] = (j == k + 1) ? 1.0 : xk(j) * scale;
      if (last) return true;
      TRD_STAMP(7)
      if (!SOLO) trd_bar_wait(&barY, par ^ 1);
      else __syncthreads();
      if (k + 1 == ke && ke < N - 2) {
        // ---- hand over to the single-CTA tail: rows i >= ke back to global, lazy state to hand[] ----
        for (int q = max(first_slot(ke), nspill); q < nown; ++q) {
          const int i = me + q * C;
          const double* src = rowptr_s(q);
          double* dst = a.M + (size_t)i * N;
          for (int j = ke + tid; j <= i; j += TRD_NT) dst[j] = src[j];
        }
        if (me == 0) {
          const int pk = ke & 1;
          for (int j = tid; j < N; j += TRD_NT) {
            a.hand[j] = xw[pk * N + j].x;
            a.hand[N + j] = xw[(pk ^ 1) * N + j].x;
            a.hand[2 * N + j] = xw[pk * N + j].y;
          }
        }
        return true;
      }
    }
    return true;
  };
  using std::integral_constant;
  bool done = false;
  if constexpr (MAXB >= 10) done = run(integral_constant<int, 10>(), TRD_NW * 7);
  if constexpr (MAXB >= 7) if (!done) done = run(integral_constant<int, 7>(), TRD_NW * 4);
  if constexpr (MAXB >= 4) if (!done) done = run(integral_constant<int, 4>(), TRD_NW * 2);
  if (!done) done = run(integral_constant<int, 2>(), TRD_NW);
  if (!done) run(integral_constant<int, 1>(), 0);
#undef TRD_STAMP
  if (!SOLO) trd_cluster_sync();  // no CTA leaves while a peer may still address its shared memory
}

inline size_t tridiag_smem_bytes(int N, int C, int S, long long row_doubles) {
  return sizeof(double) * (size_t)(trd_fixed_doubles(N, C, S) + row_doubles);
}

typedef void (*TridiagKernel)(TridiagArgs);
// (MAXB, C) pairs reachable from tridiag_maxb / tridiag_cluster_size, plus the single-CTA tails.
#define TRD_KERNELS(X) X(2, 4) X(4, 4) X(2, 8) X(4, 8) X(7, 8) X(2, 16) X(4, 16) X(7, 16) X(10, 16) X(2, 1) X(4, 1) X(7, 1) X(10, 1)
inline TridiagKernel tridiag_kernel_mc(int maxb, int C) {
#define TRD_CASE(MB, CCX) \
  if (maxb == MB && C == CCX) return k_tridiag<MB, CCX>;
  TRD_KERNELS(TRD_CASE)
#undef TRD_CASE
  return nullptr;
}
