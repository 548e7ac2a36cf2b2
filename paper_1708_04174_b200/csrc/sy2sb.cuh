// Two-stage tridiagonalisation, stage 1: dense symmetric -> band of half-bandwidth BW (blocked
// Householder with DMMA trailing updates), north_star (c) "blocked Householder
// tridiagonalisation ... with FP64 tensor-core (DMMA) trailing updates".
//
// Panel p (columns c0 = p BW .. c0 + BW - 1, rows below r0 = c0 + BW, n = N - r0 rows):
//   QR of the n x BW sub-panel:  H_1 ... H_BW = Q = I - V T V^T  (dlarfg / dlarft forward-columnwise),
//   trailing update  A22 <- Q^T A22 Q = A22 - Y V^T - V Y^T + V S V^T,  Y = A22 V T,  S = T^T V^T Y.
// B = Q1^T A Q1 is banded (Q1 = Q_0 Q_1 ...); T = Q2^T B Q2 follows by bulge chasing (sb2st.cuh).
//
// B200 mapping: ONE persistent cooperative grid.  CTA NW (the "panel CTA") factors the panels; CTAs
// 0..NW-1 ("workers") own 8-row blocks (row block rb on worker rb mod NW) and keep their FULL rows
// (both triangles, row i = column i) in shared memory for the whole reduction, so the trailing matrix
// never travels through HBM.  Per panel the data that moves is n x BW (V, Y, the panel slice).
// Hand-offs are monotone counters in global memory (release: __threadfence + atomicAdd; acquire:
// ld.acquire spin + __threadfence, which also invalidates L1):
//   workers --(panel slice, cnt_panel)--> panel CTA: QR --(V_p, T_p, v_ready)--> workers: Y rows
//   --(Y_p, V^T Y partials, cnt_y)--> workers: first chunk (the next panel's columns) --(slice,
//   cnt_panel)--> panel CTA, which meanwhile reduces S_p (fixed order) --(s_ready)--> workers: bulk.
// The first chunk omits the V S V^T term (S_p is not known yet); the panel CTA adds it to the gathered
// slice (V_p S_p V_p[panel]^T, from the V_p it still holds), so S_p is off the critical path.
// The Y and bulk-update contractions run on the FP64 tensor cores (mma.sync m8n8k4 -> DMMA) from
// shared memory, with V / Y streamed in 128-column chunks by 16-byte cp.async (L2-resident).
// Every reduction has a fixed order: the band and reflectors are bit-reproducible.
#pragma once
#include "common.cuh"
#include "gemm_f64.cuh"

constexpr int SB_NT = 512;
constexpr int SB_NWARP = SB_NT / 32;
constexpr int SB_R = 8;      // rows per row block
constexpr int SB_KC = 128;   // streamed chunk width (columns)
constexpr int SB_LDC = SB_KC + 4;

struct Sy2sbArgs {
  const double* M;   // N x N column-major block matrix, upper triangle valid (input, not modified)
  int N, BW;         // BW = 16 or 8 (template parameter copy)
  int NW;            // worker CTAs (grid = NW + 1)
  int maxrb;         // row blocks per worker
  int ldr;           // shared-memory row stride (>= N, = 4 mod 16)
  int P;             // panels with a QR (r0 = (p + 1) BW <= N - 1)
  double* Bg;        // band: Bg[c * 2BW + (r - c)] for 0 <= r - c <= BW
  double* V1;        // N x N: reflector of column k in column k, zeros in rows k+1..k+BW-1, 1 at k+BW
  double* tau1;      // N
  double* Pg;        // panel slice: row-major [row - c0][BW]
  double* Vg;        // 2 x BW x ldv: V_p by parity, column-major (ld ldv), rows from r0(p)
  double* Yg;        // 2 x BW x ldv: Y_p by parity
  int ldv;           // even >= N
  double* Tg;        // 2 x BW x BW: T_p by parity (row-major)
  double* Sg;        // BW x BW: S_p (row-major)
  double* Pt;        // NW x BW x BW: per-worker V^T Y partials
  unsigned* cnt;     // [0] cnt_panel, [1] cnt_y, [2] v_ready, [3] s_ready (zeroed before the launch)
  long long* prof;   // optional (debug): 16 clock64 stamps per panel (panel CTA 0..7, worker 0 8..15)
  const DevState* st;
  const IterScal* is;
  int check_state;
};

__device__ __forceinline__ unsigned sb_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// thread 0 spins until *p >= target (wall-clock bounded: a lost hand-off traps after 20 s instead of
// hanging the GPU), then the whole CTA proceeds with L1 invalidated
__device__ __forceinline__ void sb_wait(const unsigned* p, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned long long t0 = 0;
    unsigned spins = 0;
    while (sb_ld_acquire(p) < target) {
      __nanosleep(32);
      if ((++spins & 0xFFu) == 0) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > 20000000000ull) __trap();
      }
    }
    __threadfence();
  }
  __syncthreads();
}
// all threads' global stores so far -> visible, then one increment
__device__ __forceinline__ void sb_arrive(unsigned* p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1u);
  }
}

inline int sy2sb_panels(int N, int BW) { return N >= 2 ? (N - 1) / BW : 0; }
inline int sy2sb_ldr(int N) { return (N + 8 + 15) / 16 * 16 + 4; }  // >= N + 8, = 4 mod 16
inline int sy2sb_ldv(int N) { return (N + 1) / 2 * 2; }                // even: 16-byte rows of V_p / Y_p
inline size_t sy2sb_worker_smem(int N, int BW, int maxrb) {
  const size_t own = (size_t)maxrb * SB_R * sy2sb_ldr(N);
  const size_t chunks = 2 * 2 * (size_t)BW * SB_LDC;                     // V, Y double buffers
  const size_t small = (size_t)maxrb * SB_R * BW * 3 + 2 * (size_t)BW * BW + (size_t)SB_NWARP * maxrb * SB_R * BW;
  return 8 * (own + chunks + small) + 64;
}
inline size_t sy2sb_panel_smem(int N, int BW) {
  return 8 * ((size_t)N * BW + SB_NWARP + 2 + SB_NT + 3 * (size_t)BW * BW + BW + 8) + 64;
}

// ----------------------------------------------------------------------------------------------
// panel CTA: QR of rows [BW, nP) of the slice held in Ps (row stride BW + 1), see the header.
// Panel QR, thread per row: thread t keeps sub-panel rows r = t + k SB_NT (k < RPT) -- all BW columns --
// in registers (BW = 16: m <= 848 rows, RPT = 2; BW = 8: m <= 1272, RPT = 3).  Per column j: the
// column-j norm and the BW dot products v^T S[:, q] are per-thread FMAs, reduced over the warp by a
// transpose-reduction (BW-vector in 2BW - 1 + log2(32 / BW) shuffles: lane L ends with the total of
// column L mod BW), then over the 16 warps through shared memory (fixed order).  Two CTA barriers per
// column; T (dlarft forward columnwise) is built by warp 0 as the z_j = V^T v_j become known.
template <int BW>
struct SbQr {
  static constexpr int RPT = BW == 16 ? 2 : 3;
};

// d[0..BW) summed over the 32 lanes; lane L returns the total of index L % BW (fixed order)
template <int BW>
__device__ __forceinline__ double sb_warp_vec_reduce(double (&d)[BW], int lane) {
#pragma unroll
  for (int s = BW / 2; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = up ? d[i] : d[i + s];
      const double keep = up ? d[i + s] : d[i];
      d[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  double v = d[0];
#pragma unroll
  for (int o = BW; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One column step of the panel QR (J a compile-time constant: no dynamic register indexing)
template <int BW, int J>
__device__ __forceinline__ void sb_qr_col(double (&x)[SbQr<BW>::RPT][BW], double& sig, int m, double* red1,
                                          double* red2, double* Zs, double* Tm, double* taus) {
  constexpr int RPT = SbQr<BW>::RPT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qme = lane % BW;
  // ---- (A) sigma^2_J = sum_{r > J} S[r][J]^2 (fixed order), alpha = S[J][J] (row J: thread J) ----
  double s = sig;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red1[warp] = s;
  if (tid == J && J < m) red1[SB_NWARP] = x[0][J];
  __syncthreads();
  double sg = 0.0;
#pragma unroll
  for (int w = 0; w < SB_NWARP; ++w) sg += red1[w];
  const double alpha = (J < m) ? red1[SB_NWARP] : 0.0;
  double tau = 0.0, beta = alpha, scal = 0.0;
  if (J < m && sg > 0.0) {
    beta = -copysign(sqrt(fma(alpha, alpha, sg)), alpha);
    tau = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
  // ---- (B) v_r (rows r > J scaled, row J = 1, rows < J = 0); d_q = sum_r v_r S[r][q] ----
  double v[RPT];
  double d[BW];
#pragma unroll
  for (int q = 0; q < BW; ++q) d[q] = 0.0;
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = tid + k * SB_NT;
    v[k] = r > J ? x[k][J] * scal : (r == J ? 1.0 : 0.0);
#pragma unroll
    for (int q = 0; q < BW; ++q)
      if (q != J) d[q] = fma(v[k], x[k][q], d[q]);
  }
  const double dsum = sb_warp_vec_reduce<BW>(d, lane);
  if (lane < BW) red2[warp * BW + lane] = dsum;
  __syncthreads();
  double dq = 0.0;  // total for column qme
#pragma unroll
  for (int w = 0; w < SB_NWARP; ++w) dq += red2[w * BW + qme];
  // ---- (C) S[r][q] -= v_r w_q (q > J, w_q = tau d_q); v stored in column J; R diagonal; T ----
  const double wme = tau * dq;
  sig = 0.0;
#pragma unroll
  for (int q = J + 1; q < BW; ++q) {
    const double wq = __shfl_sync(0xffffffffu, wme, q);
#pragma unroll
    for (int k = 0; k < RPT; ++k) x[k][q] = fma(-v[k], wq, x[k][q]);
  }
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = tid + k * SB_NT;
    x[k][J] = r > J ? v[k] : (r == J ? beta : x[k][J]);  // column J: v below, beta on the diagonal
    if (J + 1 < BW && r > J + 1) sig = fma(x[k][(J + 1) % BW], x[k][(J + 1) % BW], sig);
  }
  if (warp == 0) {
    if (lane < J) Zs[J * BW + lane] = dq;  // z_J[l] = v_l^T v_J (qme = lane for lane < BW)
    __syncwarp();
    double acc = 0.0;
    if (lane < J)
      for (int l = lane; l < J; ++l) acc = fma(Tm[lane * BW + l], Zs[J * BW + l], acc);
    if (lane < BW) Tm[lane * BW + J] = lane < J ? -tau * acc : (lane == J ? tau : 0.0);
    __syncwarp();
  }
  if (tid == 0) taus[J] = tau;
}

template <int BW, int J>
__device__ __forceinline__ void sb_qr_cols(double (&x)[SbQr<BW>::RPT][BW], double& sig, int m, double* red1,
                                           double* red2, double* Zs, double* Tm, double* taus) {
  if constexpr (J < BW) {
    sb_qr_col<BW, J>(x, sig, m, red1, red2, Zs, Tm, taus);
    sb_qr_cols<BW, J + 1>(x, sig, m, red1, red2, Zs, Tm, taus);
  }
}

template <int BW>
__device__ void sb_panel_qr(double* S, int m, double* red1, double* red2, double* Zs, double* Tm, double* taus) {
  constexpr int RPT = SbQr<BW>::RPT;
  const int tid = threadIdx.x;
  double x[RPT][BW];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = tid + k * SB_NT;
#pragma unroll
    for (int q = 0; q < BW; ++q) x[k][q] = r < m ? S[r * BW + q] : 0.0;
  }
  double sig = 0.0;  // this thread's sigma^2 partial of the current column
#pragma unroll
  for (int k = 0; k < RPT; ++k)
    if (tid + k * SB_NT > 0) sig = fma(x[k][0], x[k][0], sig);
  sb_qr_cols<BW, 0>(x, sig, m, red1, red2, Zs, Tm, taus);
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = tid + k * SB_NT;
    if (r < m)
#pragma unroll
      for (int q = 0; q < BW; ++q) S[r * BW + q] = x[k][q];
  }
  __syncthreads();
}

template <int BW>
__global__ void __launch_bounds__(SB_NT, 1) k_sy2sb(Sy2sbArgs a) {
  if (a.check_state && (a.st->done || !a.is->proceed)) return;
  extern __shared__ __align__(16) double sm[];
  const int N = a.N, NW = a.NW, P = a.P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int LDB = 2 * BW;
  unsigned* cnt_panel = a.cnt;
  unsigned* cnt_y = a.cnt + 1;
  unsigned* v_ready = a.cnt + 2;
  unsigned* s_ready = a.cnt + 3;

  if (blockIdx.x == NW) {
    // =========================== panel CTA ===========================
    constexpr int LDP = BW, G = 32 / BW;
    const int g = lane / BW, qq = lane % BW;
    const int slot = warp * G + g, NS = SB_NWARP * G;
    double* Ps = sm;                              // [N][BW] slice rows (relative to c0)
    double* red1 = Ps + (size_t)N * LDP;          // [16 + 1]
    double* red2 = red1 + SB_NWARP + 2;           // [SB_NT]: QR column sums, then the S partial halves
    double* Zs = red2 + SB_NT;                    // [BW][BW] z_j, then S
    double* Tm = Zs + BW * BW;                    // [BW][BW] T_p
    double* Sm = Tm + BW * BW;                    // [BW][BW] S_p
    double* taus = Sm + BW * BW;
    for (int e = tid; e < N * LDP; e += SB_NT) Ps[e] = 0.0;
    const bool prof = a.prof != nullptr && tid == 0;
#define SB_STAMP(k) \
  if (prof) a.prof[(size_t)p * 16 + (k)] = clock64();
    for (int p = 0; p <= P; ++p) {
      const int c0 = p * BW, r0 = c0 + BW, nP = N - c0;
      // gathered slice (the workers applied panel p-1's full update to it)
      SB_STAMP(0);
      sb_wait(cnt_panel, (unsigned)(NW * (p + 1)));
      SB_STAMP(1);
      {
        const int tot = nP * BW;
        for (int e0 = tid; e0 < tot; e0 += 8 * SB_NT) {
          double x[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int e = e0 + t * SB_NT;
            x[t] = e < tot ? __ldcg(a.Pg + e) : 0.0;
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int e = e0 + t * SB_NT;
            if (e < tot) Ps[e] = x[t];
          }
        }
      }
      __syncthreads();
      // band entries of the diagonal block: rows a < BW of the slice, columns q <= a
      for (int e = tid; e < BW * BW; e += SB_NT) {
        const int ar = e / BW, q2 = e % BW;
        if (q2 <= ar && ar < nP) a.Bg[(size_t)(c0 + q2) * LDB + (ar - q2)] = Ps[ar * LDP + q2];
      }
      if (p == P) break;
      const int m = N - r0;  // >= 1
      SB_STAMP(2);
      double* S = Ps + BW * LDP;
      sb_panel_qr<BW>(S, m, red1, red2, Zs, Tm, taus);
      SB_STAMP(3);
      const int par = p & 1;
      double* Vp = a.Vg + (size_t)par * BW * a.ldv;
      // V_p (explicit unit upper part) and T_p first: the workers wait for them
      for (int e = tid; e < m * BW; e += SB_NT) {
        const int r = e % m, q2 = e / m;
        const double v = r < q2 ? 0.0 : (r == q2 ? 1.0 : S[r * LDP + q2]);
        Vp[(size_t)q2 * a.ldv + r] = v;
      }
      __syncthreads();
      for (int e = tid; e < BW * BW; e += SB_NT) a.Tg[(size_t)par * BW * BW + e] = Tm[e];
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(v_ready, 1u);
      }
      SB_STAMP(4);
      // off the critical path: the reflector layout V1, tau, R -> band
      for (int q2 = warp; q2 < BW; q2 += SB_NWARP) {
        const int k = c0 + q2;
        double* col = a.V1 + (size_t)k * N;
        for (int row = k + 1 + lane; row < N; row += 32) {
          const int r = row - r0;
          col[row] = r < q2 ? 0.0 : (r == q2 ? 1.0 : S[r * LDP + q2]);
        }
        if (lane == 0) a.tau1[k] = taus[q2];
      }
      for (int e = tid; e < BW * BW; e += SB_NT) {
        const int j = e / BW, q2 = e % BW;
        if (j <= q2 && j < m) a.Bg[(size_t)(c0 + q2) * LDB + (BW + j - q2)] = S[j * LDP + q2];
      }
      // ---- S_p = T_p^T sum_w Pt[w] (fixed order), symmetrised, published ----
      sb_wait(cnt_y, (unsigned)(NW * (p + 1)));
      SB_STAMP(5);
      {
        // thread (entry e, half hh): workers hh, hh + 2, ... in batches of 16 independent loads
        const int e = tid % (BW * BW), hh = tid / (BW * BW);
        constexpr int NH = SB_NT / (BW * BW);
        double acc = 0.0;
        for (int w0 = hh; w0 < NW; w0 += 16 * NH) {
          double xv[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int w = w0 + t * NH;
            xv[t] = w < NW ? __ldcg(a.Pt + (size_t)w * BW * BW + e) : 0.0;
          }
#pragma unroll
          for (int t = 0; t < 16; ++t) acc += xv[t];
        }
        red2[hh * BW * BW + e] = acc;  // red2 holds NH * BW * BW = SB_NT doubles? (see smem size)
      }
      __syncthreads();
      if (tid < BW * BW) {
        constexpr int NH = SB_NT / (BW * BW);
        double acc = 0.0;
        for (int hh = 0; hh < NH; ++hh) acc += red2[hh * BW * BW + tid];
        Sm[tid] = acc;  // V^T Y
      }
      __syncthreads();
      if (tid < BW * BW) {
        const int k = tid / BW, l = tid % BW;
        double acc = 0.0;
        for (int i = 0; i <= k; ++i) acc = fma(Tm[i * BW + k], Sm[i * BW + l], acc);  // (T^T V^T Y)[k][l]
        Zs[tid] = acc;
      }
      __syncthreads();
      // S is symmetric in exact arithmetic (T^T V^T A V T); its rounding-level skew part must not enter
      // the non-symmetric update form W' = Y - V S (it is amplified panel after panel: measured on
      // low-rank blocks), so publish (S + S^T) / 2
      if (tid < BW * BW) a.Sg[tid] = 0.5 * (Zs[tid] + Zs[(tid % BW) * BW + tid / BW]);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(s_ready, 1u);
      }
      SB_STAMP(6);
      SB_STAMP(7);
    }
    return;
  }

  // =============================== workers ===============================
  const int w = blockIdx.x;
  const int nrb = (N + SB_R - 1) / SB_R;
  const int ldr = a.ldr, maxrb = a.maxrb;
  double* Aown = sm;                                         // [maxrb][8][ldr]
  double* Vc = Aown + (size_t)maxrb * SB_R * ldr;            // [2][BW][LDC]
  double* Yc = Vc + 2 * BW * SB_LDC;                         // [2][BW][LDC]
  double* Vo = Yc + 2 * BW * SB_LDC;                         // [maxrb*8][BW] own V rows
  double* Yo = Vo + maxrb * SB_R * BW;                       // [maxrb*8][BW] own Y rows (then W')
  double* Xo = Yo + maxrb * SB_R * BW;                       // [maxrb*8][BW] scratch
  double* Tm = Xo + maxrb * SB_R * BW;                       // [BW][BW]
  double* Sm = Tm + BW * BW;                                 // [BW][BW]
  double* red = Sm + BW * BW;                                // [16][maxrb*8*BW]
  int nown = 0;
  for (int rb = w; rb < nrb; rb += NW) ++nown;
  auto row_of = [&](int s, int rr) { return (w + s * NW) * SB_R + rr; };
  // own rows = columns of the symmetric input
  for (int s = 0; s < nown; ++s)
    for (int rr = 0; rr < SB_R; ++rr) {
      const int i = row_of(s, rr);
      double* dst = Aown + ((size_t)s * SB_R + rr) * ldr;
      // row i of the symmetric block from its upper triangle (column max(i, c), row min(i, c))
      for (int c = tid; c < ldr; c += SB_NT)
        dst[c] = (i < N && c < N) ? __ldg(a.M + (c <= i ? (size_t)i * N + c : (size_t)c * N + i)) : 0.0;
    }
  __syncthreads();
  // slice of panel 0: all own rows, columns 0..BW-1
  auto publish_slice = [&](int c0) {
    const int ncol = min(BW, N - c0);
    for (int s = 0; s < nown; ++s)
      for (int e = tid; e < SB_R * ncol; e += SB_NT) {
        const int rr = e / ncol, jj = e % ncol, i = row_of(s, rr);
        if (i < N && i >= c0) a.Pg[(size_t)(i - c0) * BW + jj] = Aown[((size_t)s * SB_R + rr) * ldr + c0 + jj];
      }
    sb_arrive(cnt_panel);
  };
  publish_slice(0);

  for (int p = 0; p < P; ++p) {
    const int c0 = p * BW, r0 = c0 + BW, n = N - r0, par = p & 1;
    const int ldv = a.ldv;
    const double* Vp = a.Vg + (size_t)par * BW * ldv;
    double* Yp = a.Yg + (size_t)par * BW * ldv;
    // does this worker own any row >= r0 ?
    int s_lo = nown;
    for (int s = 0; s < nown; ++s)
      if (row_of(s, SB_R - 1) >= r0) {
        s_lo = s;
        break;
      }
    const bool wprof = a.prof != nullptr && w == 0 && tid == 0;
#define SB_WSTAMP(k) \
  if (wprof) a.prof[(size_t)p * 16 + 8 + (k)] = clock64();
    SB_WSTAMP(0);
    sb_wait(v_ready, (unsigned)(p + 1));
    SB_WSTAMP(1);
    for (int e = tid; e < BW * BW; e += SB_NT) Tm[e] = __ldcg(a.Tg + (size_t)par * BW * BW + e);
    // own V rows (0 for rows < r0 or >= N)
    for (int e = tid; e < nown * SB_R * BW; e += SB_NT) {
      const int sr = e / BW, jj = e % BW, i = row_of(sr / SB_R, sr % SB_R);
      Vo[e] = (i >= r0 && i < N) ? __ldcg(Vp + (size_t)jj * ldv + (i - r0)) : 0.0;
    }
    // ---- Y_own = A_own[:, r0:] V_p  (DMMA, V streamed in chunks) ----
    const int nch = (n + SB_KC - 1) / SB_KC;
    auto issue = [&](const double* src, double* dst, int ch) {
      const int cb = ch * SB_KC, w8 = min(SB_KC, n - cb);
      for (int e = tid; e < BW * (SB_KC / 2); e += SB_NT) {
        const int jj = e / (SB_KC / 2), cc = 2 * (e % (SB_KC / 2));
        double* d = dst + jj * SB_LDC + cc;
        const double* sp = src + (size_t)jj * ldv + cb + cc;
        if (cc + 1 < w8 && (((uintptr_t)sp & 15) == 0)) {
          cp_async16(d, sp);
        } else {
          d[0] = cc < w8 ? __ldcg(sp) : 0.0;
          d[1] = cc + 1 < w8 ? __ldcg(sp + 1) : 0.0;
        }
      }
      cp_async_commit();
    };
    double accY[4][BW / 8][2];
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int t = 0; t < BW / 8; ++t) accY[s][t][0] = accY[s][t][1] = 0.0;
    if (s_lo < nown) {
      // 4-slot ring of 128-column V chunks (the V and Y chunk buffers of the bulk update, contiguous)
      constexpr int RING = 4;
      for (int ch = 0; ch < RING - 1 && ch < nch; ++ch) issue(Vp, Vc + (size_t)ch * BW * SB_LDC, ch);
      for (int ch = 0; ch < nch; ++ch) {
        if (ch + RING - 1 < nch) {
          issue(Vp, Vc + (size_t)((ch + RING - 1) % RING) * BW * SB_LDC, ch + RING - 1);
          cp_async_wait<RING - 1>();
        } else if (nch - 1 - ch >= 2) {
          cp_async_wait<2>();
        } else if (nch - 1 - ch == 1) {
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const double* V_ = Vc + (size_t)(ch % RING) * BW * SB_LDC;
        const int cb = ch * SB_KC;
        // warp -> k-steps warp, warp + 16 (KC / 4 = 32 k-steps)
        for (int ks = warp; ks < SB_KC / 4; ks += SB_NWARP) {
          const int kk = ks * 4 + (lane & 3);
          const bool okk = cb + kk < n;
          double bf[BW / 8];
#pragma unroll
          for (int t = 0; t < BW / 8; ++t) bf[t] = V_[(t * 8 + (lane >> 2)) * SB_LDC + kk];
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            if (s < s_lo || s >= nown) continue;
            const double af = okk ? Aown[((size_t)s * SB_R + (lane >> 2)) * ldr + r0 + cb + kk] : 0.0;
#pragma unroll
            for (int t = 0; t < BW / 8; ++t) dmma_8x8x4(accY[s][t][0], accY[s][t][1], af, bf[t]);
          }
        }
        __syncthreads();
      }
      // cross-warp reduction (fixed order) -> Xo = A_own V_p
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (s >= s_lo && s < nown)
#pragma unroll
          for (int t = 0; t < BW / 8; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              red[((size_t)warp * maxrb + s) * SB_R * BW + (lane >> 2) * BW + t * 8 + 2 * (lane & 3) + h] =
                  accY[s][t][h];
      __syncthreads();
      for (int e = tid; e < nown * SB_R * BW; e += SB_NT) {
        if (e / (SB_R * BW) < s_lo) continue;
        double acc = 0.0;
        for (int ww = 0; ww < SB_NWARP; ++ww) acc += red[(size_t)ww * maxrb * SB_R * BW + e];
        Xo[e] = acc;
      }
      __syncthreads();
      // Y = X T (rows < r0 give 0 through their zero V and are never used)
      for (int e = tid; e < nown * SB_R * BW; e += SB_NT) {
        const int sr = e / BW, jj = e % BW, i = row_of(sr / SB_R, sr % SB_R);
        double acc = 0.0;
        for (int l = 0; l <= jj; ++l) acc = fma(Xo[sr * BW + l], Tm[l * BW + jj], acc);
        Yo[e] = (i >= r0 && i < N) ? acc : 0.0;
        if (i >= r0 && i < N) Yp[(size_t)jj * ldv + (i - r0)] = Yo[e];
      }
      __syncthreads();
    } else {
      for (int e = tid; e < nown * SB_R * BW; e += SB_NT) Yo[e] = 0.0;
      __syncthreads();
    }
    // partial V_own^T Y_own (fixed order over own rows)
    if (tid < BW * BW) {
      const int k = tid / BW, l = tid % BW;
      double acc = 0.0;
      for (int sr = 0; sr < nown * SB_R; ++sr) acc = fma(Vo[sr * BW + k], Yo[sr * BW + l], acc);
      a.Pt[(size_t)w * BW * BW + tid] = acc;
    }
    SB_WSTAMP(2);
    sb_arrive(cnt_y);
    sb_wait(cnt_y, (unsigned)(NW * (p + 1)));
    SB_WSTAMP(3);
    // ---- S_p, W' = Y - V S for own rows ----
    sb_wait(s_ready, (unsigned)(p + 1));
    SB_WSTAMP(4);
    for (int e = tid; e < BW * BW; e += SB_NT) Sm[e] = __ldcg(a.Sg + e);
    __syncthreads();
    for (int e = tid; e < nown * SB_R * BW; e += SB_NT) {
      const int sr = e / BW, jj = e % BW;
      double acc = Yo[e];
      for (int l = 0; l < BW; ++l) acc = fma(-Vo[sr * BW + l], Sm[l * BW + jj], acc);
      Xo[e] = acc;  // W'
    }
    __syncthreads();
    // ---- first chunk: columns [r0, r0 + BW) of own rows >= r0, then the next panel's slice ----
    {
      const int ncol = min(BW, n);
      for (int e = tid; e < nown * SB_R * ncol; e += SB_NT) {
        const int sr = e / ncol, jj = e % ncol, i = row_of(sr / SB_R, sr % SB_R);
        if (i < r0 || i >= N) continue;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < BW; ++q) {
          acc = fma(Xo[sr * BW + q], __ldcg(Vp + (size_t)q * ldv + jj), acc);
          acc = fma(Vo[sr * BW + q], __ldcg(Yp + (size_t)q * ldv + jj), acc);
        }
        Aown[((size_t)(sr / SB_R) * SB_R + sr % SB_R) * ldr + r0 + jj] -= acc;
      }
      __syncthreads();
      publish_slice(r0);
    }
    SB_WSTAMP(5);
    // ---- bulk: columns >= r0 + BW of own rows >= r0 + BW: A -= W' V^T + V Y^T ----
    if (n > BW && s_lo < nown) {
      const int cstart = BW;  // relative to r0
      const int nb = n - cstart;
      const int nchb = (nb + SB_KC - 1) / SB_KC;
      auto issue2 = [&](int ch, int buf) {
        const int cb = cstart + ch * SB_KC, w8 = min(SB_KC, n - cb);
        for (int e = tid; e < 2 * BW * (SB_KC / 2); e += SB_NT) {
          const int which = e / (BW * (SB_KC / 2));
          const int ee = e % (BW * (SB_KC / 2));
          const int jj = ee / (SB_KC / 2), cc = 2 * (ee % (SB_KC / 2));
          double* d = (which ? Yc : Vc) + buf * BW * SB_LDC + jj * SB_LDC + cc;
          const double* sp = (which ? (const double*)Yp : Vp) + (size_t)jj * ldv + cb + cc;
          if (cc + 1 < w8 && (((uintptr_t)sp & 15) == 0)) {
            cp_async16(d, sp);
          } else {
            d[0] = cc < w8 ? __ldcg(sp) : 0.0;
            d[1] = cc + 1 < w8 ? __ldcg(sp + 1) : 0.0;
          }
        }
        cp_async_commit();
      };
      issue2(0, 0);
      for (int ch = 0; ch < nchb; ++ch) {
        const int buf = ch & 1;
        if (ch + 1 < nchb) {
          issue2(ch + 1, buf ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const double* V_ = Vc + buf * BW * SB_LDC;
        const double* Y_ = Yc + buf * BW * SB_LDC;
        const int cb = cstart + ch * SB_KC;
        // n-tile = warp (16 tiles of 8 columns = 128), all 2BW/4 k-steps, every own row block
        const int nt = warp;
        if (cb + nt * 8 < n) {
          for (int s = s_lo; s < nown; ++s) {
            double* Arow = Aown + ((size_t)s * SB_R + (lane >> 2)) * ldr + r0 + cb + nt * 8 + 2 * (lane & 3);
            const int colg = r0 + cb + nt * 8 + 2 * (lane & 3);
            double2 cv = *reinterpret_cast<double2*>(Arow);
            double c0v = cv.x, c1v = cv.y;
#pragma unroll
            for (int ks = 0; ks < 2 * BW / 4; ++ks) {
              const int kk = ks * 4 + (lane & 3);  // 0..2BW-1: [W' | V] x [V ; Y]
              const int sr = s * SB_R + (lane >> 2);
              const double af = kk < BW ? -Xo[sr * BW + kk] : -Vo[sr * BW + kk - BW];
              const double bf = kk < BW ? V_[kk * SB_LDC + nt * 8 + (lane >> 2)]
                                        : Y_[(kk - BW) * SB_LDC + nt * 8 + (lane >> 2)];
              dmma_8x8x4(c0v, c1v, af, bf);
            }
            const int i = row_of(s, lane >> 2);
            if (i >= r0 + BW && i < N) {
              if (colg < N) Arow[0] = c0v;
              if (colg + 1 < N) Arow[1] = c1v;
            }
          }
        }
        __syncthreads();
      }
    }
    SB_WSTAMP(6);
  }
}

using Sy2sbKernel = void (*)(Sy2sbArgs);
inline Sy2sbKernel sy2sb_kernel(int BW) { return BW == 16 ? k_sy2sb<16> : k_sy2sb<8>; }
