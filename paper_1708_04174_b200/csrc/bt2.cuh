// Back-transform of the selected tridiagonal eigenvectors through the stage-2 (bulge-chasing)
// reflectors: Z <- Q2 Z with Q2 = H_{0,0} H_{0,1} ... H_{N-3,last} (sb2st.cuh), SURVEY §8(a) row c1
// (PAPER.md P:397-398 needs the eigenvectors of the original block: Q1 Q2 Z).  Applied in reverse sweep
// order; the reflectors of one sweep act on disjoint BW-row windows, so they are applied in parallel.
// One CTA owns 8 columns of Z in shared memory (the columns are independent); each sweep's reflectors
// are prefetched by cp.async into a double buffer while the previous sweep is applied.  Works in place
// on the selected columns c0 .. c0 + r - 1 of the divide-and-conquer eigenvector matrix (k_select's sel).
#pragma once
#include "common.cuh"

constexpr int BT2_NT = 256;
constexpr int BT2_NC = 8;

inline size_t bt2_smem(int N, int BW, int KMAX) {
  return 8 * ((size_t)N * BT2_NC + 2 * (size_t)KMAX * (BW + 1)) + 64;
}

template <int BW>
__global__ void __launch_bounds__(BT2_NT) k_bt2(double* __restrict__ Qf, const int* __restrict__ sel,
                                               const double* __restrict__ V2, const double* __restrict__ tau2, int N,
                                               int KMAX, const DevState* st, const IterScal* is, int check_state) {
  if (check_state && (st->done || !is->proceed)) return;
  const int r = sel[0], c0 = sel[1];
  const int cbase = blockIdx.x * BT2_NC;
  if (cbase >= r || N < 3) return;
  extern __shared__ __align__(16) double smz[];
  double* Zs = smz;                                   // [N][8]
  double* Vb = Zs + (size_t)N * BT2_NC;               // [2][KMAX][BW]
  double* Tb = Vb + 2 * (size_t)KMAX * BW;            // [2][KMAX]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncol = min(BT2_NC, r - cbase);
  for (int e = tid; e < N * BT2_NC; e += BT2_NT) {
    const int row = e / BT2_NC, c = e % BT2_NC;
    Zs[e] = c < ncol ? Qf[(size_t)(c0 + cbase + c) * N + row] : 0.0;
  }
  auto prefetch = [&](int i, int buf) {
    const int nt = (N - 2 - i) / BW + 1;
    const double* src = V2 + (size_t)i * KMAX * BW;
    double* dst = Vb + (size_t)buf * KMAX * BW;
    for (int e = 2 * tid; e < nt * BW; e += 2 * BT2_NT) cp_async16(dst + e, src + e);
    const double* ts = tau2 + (size_t)i * KMAX;
    for (int e = tid; e < nt; e += BT2_NT) cp_async8(Tb + (size_t)buf * KMAX + e, ts + e);
    cp_async_commit();
  };
  prefetch(N - 3, 0);
  int buf = 0;
  constexpr int RL = BW / 4;  // rows per lane: lane = (row group rg = lane / 8, column c = lane % 8)
  const int rg = lane >> 3, c = lane & 7;
  for (int i = N - 3; i >= 0; --i, buf ^= 1) {
    if (i > 0) {
      prefetch(i - 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int nt = (N - 2 - i) / BW + 1;
    const double* Vs = Vb + (size_t)buf * KMAX * BW;
    const double* Ts = Tb + (size_t)buf * KMAX;
    for (int k = warp; k < nt; k += BT2_NT / 32) {
      const int R0 = i + 1 + k * BW, L = min(BW, N - R0);
      double z[RL], v[RL];
      double dot = 0.0;
#pragma unroll
      for (int t = 0; t < RL; ++t) {
        const int a = rg + 4 * t;
        v[t] = a < L ? Vs[k * BW + a] : 0.0;
        z[t] = a < L ? Zs[(R0 + a) * BT2_NC + c] : 0.0;
        dot = fma(v[t], z[t], dot);
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 8);
      dot += __shfl_xor_sync(0xffffffffu, dot, 16);
      dot *= Ts[k];
#pragma unroll
      for (int t = 0; t < RL; ++t) {
        const int a = rg + 4 * t;
        if (a < L) Zs[(R0 + a) * BT2_NC + c] = fma(-dot, v[t], z[t]);
      }
    }
    __syncthreads();  // the next sweep's windows overlap this one's; buffer `buf` is refilled next round
  }
  for (int e = tid; e < N * BT2_NC; e += BT2_NT) {
    const int row = e / BT2_NC, cc = e % BT2_NC;
    if (cc < ncol) Qf[(size_t)(c0 + cbase + cc) * N + row] = Zs[e];
  }
}

using Bt2Kernel = void (*)(double*, const int*, const double*, const double*, int, int, const DevState*,
                           const IterScal*, int);
inline Bt2Kernel bt2_kernel(int BW) { return BW == 16 ? k_bt2<16> : k_bt2<8>; }
