// Batched FP64 GEMM on the FP64 tensor cores (mma.sync.aligned.m8n8k4.f64 -> SASS DMMA; sm_100a
// has no tcgen05 kind::f64, see SURVEY §0 probe), used by the large-block PSD projection for the
// divide-and-conquer eigenvector updates and the reconstruction V diag(lambda) V^T.
//
//   C[:, ccol[j]] = alpha * sum_k A[:, acol[k]] * op(B)[k, j] + beta * C[:, ccol[j]]
// column-major operands; acol / ccol optional column maps (nullptr = identity); op(B) = B or B^T.
// The K extent can be read from device memory (Kdev) so a launch captured in a CUDA graph can
// follow a data-dependent rank.
#pragma once
#include "common.cuh"

struct GemmDesc {
  const double* A;
  const double* B;
  double* C;
  int M, N, K;
  int lda, ldb, ldc;
  const int* acol;
  const int* ccol;
  const int* Kdev;     // if non-null, K = *Kdev
  const int* Ndev;     // if non-null, N = *Ndev
  const int* Noff;     // if non-null, column j of op(B) / C is j + *Noff (a device-chosen column range)
  int transB;
  double alpha, beta;
  int skip;            // 1 = this batch entry does nothing
  int upper;           // 1 = only tiles that meet the upper triangle (row <= column) are needed
};

constexpr int GM_BM = 32, GM_BN = 64, GM_BK = 16, GM_NT = 128, GM_ST = 3;
constexpr int GM_PAD = 8;

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// grid: (ceil(maxM/32), ceil(maxN/64), batch); 4 warps as 1 (M) x 4 (N), warp tile 32 x 16 (small
// tiles: the D&C merges and the reconstruction are N <= ~1000 GEMMs, so more CTAs per SM hide latency).
// K is streamed in 16-deep slices through a cp.async double buffer (the copies of slice s+1, with the
// column gather acol[] resolved by the copy engine's address, overlap the DMMAs of slice s);
// out-of-range elements are zero-filled by the copy itself.
__global__ void __launch_bounds__(GM_NT) k_gemm_f64(const GemmDesc* __restrict__ descs, const DevState* st,
                                                    const IterScal* is, int check_state) {
  if (check_state && (st->done || !is->proceed)) return;
  const GemmDesc g = descs[blockIdx.z];
  if (g.skip) return;
  const int M = g.M;
  const int N = g.Ndev ? *g.Ndev : g.N;
  const int K = g.Kdev ? *g.Kdev : g.K;
  const int joff = g.Noff ? *g.Noff : 0;
  const int i0 = blockIdx.x * GM_BM, j0 = blockIdx.y * GM_BN;
  if (i0 >= M || j0 >= N) return;
  if (g.upper && i0 > j0 + GM_BN - 1) return;  // tile strictly below the diagonal
  __shared__ __align__(16) double As[GM_ST][GM_BK][GM_BM + GM_PAD];
  __shared__ __align__(16) double Bs[GM_ST][GM_BK][GM_BN + GM_PAD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = 0, wn = warp;  // warp tile origin (wm*32, wn*16)
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  auto issue = [&](int k0, int buf) {
    // A slice (64 x 16): each k column contiguous in the rows
#pragma unroll
    for (int r = 0; r < (GM_BM * GM_BK) / GM_NT; ++r) {
      const int idx = tid + r * GM_NT;
      const int i = idx % GM_BM, k = idx / GM_BM;
      const int gi = i0 + i, gk = k0 + k;
      const bool ok = gi < M && gk < K;
      const int col = ok ? (g.acol ? g.acol[gk] : gk) : 0;
      cp_async8z(&As[buf][k][i], g.A + (ok ? (size_t)col * g.lda + gi : 0), ok);
    }
    if (!g.transB) {  // op(B)[k, j] = B[j * ldb + k]: contiguous in k
#pragma unroll
      for (int r = 0; r < (GM_BK * GM_BN) / GM_NT; ++r) {
        const int idx = tid + r * GM_NT;
        const int k = idx % GM_BK, j = idx / GM_BK;
        const int gk = k0 + k, gj = j0 + j;
        const bool ok = gk < K && gj < N;
        cp_async8z(&Bs[buf][k][j], g.B + (ok ? (size_t)(gj + joff) * g.ldb + gk : 0), ok);
      }
    } else {  // op(B)[k, j] = B[k * ldb + j]: contiguous in j
#pragma unroll
      for (int r = 0; r < (GM_BK * GM_BN) / GM_NT; ++r) {
        const int idx = tid + r * GM_NT;
        const int j = idx % GM_BN, k = idx / GM_BN;
        const int gk = k0 + k, gj = j0 + j;
        const bool ok = gk < K && gj < N;
        cp_async8z(&Bs[buf][k][j], g.B + (ok ? (size_t)gk * g.ldb + gj + joff : 0), ok);
      }
    }
    cp_async_commit();
  };

  // GM_ST-stage ring: slices sl + 1 .. sl + GM_ST - 1 are in flight while slice sl is multiplied
  const int nslices = (K + GM_BK - 1) / GM_BK;
  for (int p = 0; p < GM_ST - 1 && p < nslices; ++p) issue(p * GM_BK, p);
  for (int sl = 0; sl < nslices; ++sl) {
    const int buf = sl % GM_ST;
    if (sl + GM_ST - 1 < nslices) issue((sl + GM_ST - 1) * GM_BK, (sl + GM_ST - 1) % GM_ST);
    const int ahead = min(GM_ST - 1, nslices - 1 - sl);  // groups allowed to stay in flight
    if (ahead >= 2) cp_async_wait<2>();
    else if (ahead == 1) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GM_BK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = As[buf][kk + (lane & 3)][wm * 32 + a * 8 + (lane >> 2)];
#pragma unroll
      for (int b = 0; b < 2; ++b) bf[b] = Bs[buf][kk + (lane & 3)][wn * 16 + b * 8 + (lane >> 2)];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's issue (slice sl + GM_ST)
  }
  // epilogue: c0/c1 at (row = lane >> 2, col = 2 (lane & 3) + {0, 1}) of each 8 x 8 tile
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = i0 + wm * 32 + a * 8 + (lane >> 2);
        const int gj = j0 + wn * 16 + b * 8 + 2 * (lane & 3) + h;
        if (gi < M && gj < N) {
          const int col = g.ccol ? g.ccol[gj + joff] : gj + joff;
          double* cp = g.C + (size_t)col * g.ldc + gi;
          const double v = g.alpha * acc[a][b][h];
          *cp = (g.beta == 0.0) ? v : fma(g.beta, *cp, v);
        }
      }
}
