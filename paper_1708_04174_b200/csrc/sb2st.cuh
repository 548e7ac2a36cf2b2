// Two-stage tridiagonalisation, stage 2: band (half-bandwidth BW) -> tridiagonal by bulge chasing,
// SURVEY §8(a) row c1 (north_star (c) "Householder tridiagonalisation plus a tridiagonal solve and
// back-transform").  Column-wise chasing (the LAPACK xSB2ST kernel order):
//   sweep i, task 0:  H from A[i+1 : i+BW+1, i];  A[i+1.., i] = (beta, 0..);  D <- H D H  (BW x BW)
//   sweep i, task k:  E = A[r1 : r1+BW, r1-BW : r1] (r1 = i + 1 + k BW):  E <- E H_{k-1} (creates the
//                     bulge), H_k from E[:, 0], E <- H_k E, D_k <- H_k D_k H_k
// The bulge never reaches beyond offset 2 BW - 2 below the diagonal, so the band lives in ONE SM's
// shared memory as 2 BW diagonals (column c at Bs[c * 2BW + (r - c)]: stride 2BW - 1, odd, so a row
// walk over columns is bank-conflict free; N = 861, BW = 16: 220 KB).
//
// Task (i+1, k) conflicts only with (i, k) and (i, k+1) (checked bit-for-bit against the sequential
// order in the numpy model of DESIGN.md §5), so sweeps run as a wavefront: warp w owns sweeps i = w mod
// 16 and starts task k of sweep i once sweep i-1 finished task k+1 (progress counters in shared memory).
// Critical path ~ 2N + N/BW tasks; a task is ~1.3k FMA in one warp, all operands exchanged by shuffles.
// Reflectors are stored for the back-transform: V2[(i KMAX + k) BW + j], tau2[i KMAX + k].
#pragma once
#include "common.cuh"

constexpr int ST_NT = 512;
constexpr int ST_NWARP = ST_NT / 32;
static_assert((4 * ST_NWARP + 64) % 8 == 0, "scratch alignment");

__host__ __device__ inline int sb2st_kmax(int N, int BW) { return N >= 3 ? (N - 2) / BW + 1 : 1; }
inline size_t sb2st_smem(int N, int BW) {
  return 8 * ((size_t)N * 2 * BW + 3 * (size_t)BW * ST_NWARP) + 4 * ST_NWARP + 64 + 64;
}

template <int BW>
struct StTask {
  static constexpr int LDB = 2 * BW, H = 32 / BW, KH = BW / H;
  double* Bs;
  int N;
  double* sv;  // per-warp scratch: v[BW], w[BW] (broadcast reads instead of shuffles)
  __device__ __forceinline__ double& at(int r, int c) const { return Bs[c * LDB + (r - c)]; }
  // symmetric element (a, b) of the diagonal block starting at r
  __device__ __forceinline__ double dsym(int r, int a, int b) const { return a >= b ? at(r + a, r + b) : at(r + b, r + a); }

  // Householder (dlarfg) from x_q (lane q of every group, valid for q < L): v_q, tau, beta
  __device__ __forceinline__ void house(double x, int L, int q, int h, double& v, double& tau, double& beta) const {
    double s = (q >= 1 && q < L) ? x * x : 0.0;
#pragma unroll
    for (int o = 1; o < BW; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double alpha = __shfl_sync(0xffffffffu, x, h * BW);
    tau = 0.0;
    beta = alpha;
    double scal = 0.0;
    if (s > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, s)), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    v = q == 0 ? 1.0 : (q < L ? x * scal : 0.0);
  }

  // D <- H D H on the L x L diagonal block at r (lower triangle stored), H = I - tau v v^T;
  // sv[0..BW) holds v (written by the caller, __syncwarp'ed)
  __device__ __forceinline__ void two_sided(int r, int L, double v, double tau, int q, int h) const {
    double p = 0.0;
#pragma unroll
    for (int t = 0; t < KH; ++t) {
      const int b = h * KH + t;
      const double vb = sv[b];
      if (q < L && b < L) p = fma(dsym(r, q, b), vb, p);
    }
#pragma unroll
    for (int o = BW; o < 32; o <<= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    p *= tau;
    double s = p * v;
#pragma unroll
    for (int o = 1; o < BW; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double wq = fma(-0.5 * tau * s, v, p);
    if (h == 0) sv[BW + q] = wq;
    __syncwarp();
    // lower triangle: lane (h, q = a) updates columns b = h, h + H, ... <= a
#pragma unroll
    for (int t = 0; t < KH; ++t) {
      const int b = h + t * H;
      const double vb = sv[b], wb = sv[BW + b];
      if (q < L && b <= q) {
        double& x = at(r + q, r + b);
        x = fma(-v, wb, fma(-wq, vb, x));
      }
    }
    __syncwarp();
  }
};

template <int BW>
__global__ void __launch_bounds__(ST_NT, 1) k_sb2st(const double* __restrict__ Bg, int N, double* __restrict__ d,
                                                   double* __restrict__ e, double* __restrict__ V2,
                                                   double* __restrict__ tau2, const DevState* st, const IterScal* is,
                                                   int check_state, long long* prof = nullptr) {
  if (check_state && (st->done || !is->proceed)) return;
  constexpr int LDB = 2 * BW, H = 32 / BW, KH = BW / H;
  extern __shared__ __align__(16) double Bs[];
  volatile int* prog = reinterpret_cast<volatile int*>(Bs + (size_t)N * LDB);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane % BW, h = lane / BW;
  // band (offsets 0..BW from stage 1, the bulge rows zero)
  for (int x = tid; x < N * LDB; x += ST_NT) {
    const int c = x / LDB, off = x % LDB;
    Bs[x] = (off <= BW && c + off < N) ? __ldcg(Bg + x) : 0.0;
  }
  if (tid < ST_NWARP) prog[tid] = 0;
  __syncthreads();
  const int KMAX = sb2st_kmax(N, BW);
  double* scr = Bs + (size_t)N * LDB + (4 * ST_NWARP + 64) / 8;  // after the counters
  double* sv = scr + (size_t)warp * 3 * BW;                           // [v | w | pv] of this warp
  const StTask<BW> T{Bs, N, sv};
#define ST_STAMP(ph) \
  if (prof && i == 0 && lane == 0) prof[k * 4 + (ph)] = clock64();
  for (int i = warp; i <= N - 3; i += ST_NWARP) {
    const int nt = (N - 2 - i) / BW + 1;
    const int ntp = (N - 1 - i) / BW + 1;  // tasks of sweep i - 1
    const int base_prev = (i - 1) * (KMAX + 1);
    double ptau = 0.0;
    for (int k = 0; k < nt; ++k) {
      if (i > 0) {  // sweep i-1 must have finished task k+1 (or all of its tasks)
        const int need = base_prev + min(k + 2, ntp);
        if (lane == 0)
          while (prog[(warp + ST_NWARP - 1) % ST_NWARP] < need) __nanosleep(20);
        __threadfence_block();
        __syncwarp();
      }
      double v, tau, beta;
      if (k == 0) {
        const int r = i + 1, L = min(BW, N - r);
        const double x = q < L ? T.at(r + q, i) : 0.0;
        T.house(x, L, q, h, v, tau, beta);
        if (h == 0) sv[q] = v;
        __syncwarp();
        if (h == 0 && q < L) T.at(r + q, i) = q == 0 ? beta : 0.0;
        ST_STAMP(1);
        T.two_sided(r, L, v, tau, q, h);
      } else {
        const int r1 = i + 1 + k * BW, L = min(BW, N - r1), pr = r1 - BW;
        // (1) E <- E H_{k-1}: lane (h, q = row a), columns c in [h KH, (h + 1) KH)
        double sa = 0.0;
        double ev[KH];
#pragma unroll
        for (int t = 0; t < KH; ++t) {
          const int c = h * KH + t;
          const double pvc = sv[2 * BW + c];
          ev[t] = q < L ? T.at(r1 + q, pr + c) : 0.0;
          sa = fma(ev[t], pvc, sa);
        }
#pragma unroll
        for (int o = BW; o < 32; o <<= 1) sa += __shfl_xor_sync(0xffffffffu, sa, o);
        double e0 = 0.0;
#pragma unroll
        for (int t = 0; t < KH; ++t) {
          const int c = h * KH + t;
          const double pvc = sv[2 * BW + c];
          ev[t] = fma(-ptau * sa, pvc, ev[t]);
          if (q < L) T.at(r1 + q, pr + c) = ev[t];
          if (c == 0) e0 = ev[t];
        }
        ST_STAMP(0);
        // (2) H_k from the first column
        const double x = __shfl_sync(0xffffffffu, e0, q);  // E(q, 0) lives on lane (h = 0, q)
        T.house(x, L, q, h, v, tau, beta);
        if (h == 0) sv[q] = v;
        __syncwarp();
        if (h == 0 && q < L) T.at(r1 + q, pr) = q == 0 ? beta : 0.0;
        ST_STAMP(1);
        // (3) E <- H_k E on columns c >= 1: lane (h, q = c), rows a in [h KH, (h + 1) KH)
        double wc = 0.0;
        double el[KH];
#pragma unroll
        for (int t = 0; t < KH; ++t) {
          const int ar = h * KH + t;
          const double va = sv[ar];
          el[t] = (ar < L && q >= 1) ? T.at(r1 + ar, pr + q) : 0.0;
          wc = fma(va, el[t], wc);
        }
#pragma unroll
        for (int o = BW; o < 32; o <<= 1) wc += __shfl_xor_sync(0xffffffffu, wc, o);
        wc *= tau;
#pragma unroll
        for (int t = 0; t < KH; ++t) {
          const int ar = h * KH + t;
          const double va = sv[ar];
          if (ar < L && q >= 1) T.at(r1 + ar, pr + q) = fma(-va, wc, el[t]);
        }
        __syncwarp();
        ST_STAMP(2);
        // (4) D_k <- H_k D_k H_k
        T.two_sided(r1, L, v, tau, q, h);
      }
      if (h == 0) V2[((size_t)i * KMAX + k) * BW + q] = v;
      if (lane == 0) tau2[(size_t)i * KMAX + k] = tau;
      if (h == 0) sv[2 * BW + q] = v;  // read by the next task's right application (after its syncwarps)
      ptau = tau;
      ST_STAMP(3);
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        prog[warp] = i * (KMAX + 1) + k + 1;
      }
    }
  }
  __syncthreads();
  for (int c = tid; c < N; c += ST_NT) {
    d[c] = Bs[c * LDB];
    if (c + 1 < N) e[c] = Bs[c * LDB + 1];
  }
}

using Sb2stKernel = void (*)(const double*, int, double*, double*, double*, double*, const DevState*,
                             const IterScal*, int, long long*);
inline Sb2stKernel sb2st_kernel(int BW) { return BW == 16 ? k_sb2st<16> : k_sb2st<8>; }
