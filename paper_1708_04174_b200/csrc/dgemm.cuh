// FP64 tensor-core GEMM for the warm-started eigensolver (warm.cuh): square-ish N <= ~1300 products
//   C = alpha * op(A) * B + beta * C,   op(A) = A or A^T, all operands column-major, every leading
//   dimension EVEN (16-byte cp.async rows; the workspace pads N to an even pitch).
// DMMA through mma.sync.aligned.m8n8k4.f64 (sm_100a has no tcgen05 kind::f64, SURVEY §0 probe).
//
// CTA tile BM x BN, K streamed in BK-deep slices through an ST-stage cp.async ring with 16-byte copies
// (row / column tails zero-filled by the copy's src-size), WM x WN warps, warp tile (BM/WM) x (BN/WN)
// of 8 x 8 DMMA tiles.  Shared-memory pitches are padded to 4 mod 16 doubles, so the fragment loads
// (lanes (row = lane / 4, k = lane % 4)) of every half-warp hit 16 distinct 8-byte banks.
// upper = 1 computes only the tiles that meet the upper triangle (row <= column): X^T W and X^T X
// are symmetric and only their upper triangles are read.
#pragma once
#include "common.cuh"

struct DgemmDesc {
  const double* A;
  const double* B;
  double* C;
  int M, N, K;
  int lda, ldb, ldc;
  int transA;          // 0: op(A)(i, k) = A[k lda + i];  1: op(A)(i, k) = A[i lda + k]
  int upper;           // 1: only tiles with row0 <= last column of the tile
  int mirror;          // 1 (with upper, beta = 0): C(j, i) = C(i, j) written for i < j, the lower triangle
                       //   mirrors the upper bit for bit (diagonal tiles keep only their i <= j entries)
  double alpha, beta;
  const int* gate;     // optional: the product runs only while *gate == 1 (warm.cuh state)
  const int* Ndev;     // optional: N = *Ndev (a device-chosen rank, captured once in the CUDA graph)
  const int* Kdev;     // optional: K = *Kdev
};

// 16-byte cp.async with a byte count (0, 8 or 16): the remainder of the 16-byte slot is zero-filled
__device__ __forceinline__ void cp_async16n(void* smem, const void* gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}

__device__ __forceinline__ void dg_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WM, int WN, int ST, int KG>
struct DgCfg {
  static constexpr int NT = 32 * WM * WN * KG;  // KG warp groups split every slice's k steps
  static constexpr int TM = BM / WM / 8, TN = BN / WN / 8;  // DMMA tiles per warp
  static constexpr int LDA0 = BM + 4;                        // A tile [k][m] (op(A) = A)
  static constexpr int LDK = BK + 4;                         // A tile [m][k] (op(A) = A^T), B tile [n][k]
  static constexpr int ASZ = BM * LDK > BK * LDA0 ? BM * LDK : BK * LDA0;
  static constexpr int BSZ = BN * LDK;
  static constexpr size_t SMEM = sizeof(double) * (size_t)ST * (ASZ + BSZ);
  static_assert((BM * BK / 2) % NT == 0 && (BN * BK / 2) % NT == 0, "chunk split");
  static_assert(LDA0 % 16 == 4 && LDK % 16 == 4, "bank-conflict-free pitches");
  static_assert(BK % (4 * KG) == 0, "k steps per group");
  static_assert(KG == 1 || (size_t)(KG - 1) * BM * BN <= (size_t)ST * (ASZ + BSZ), "reduction buffer");
};

template <int BM, int BN, int BK, int WM, int WN, int ST, int KG>
__global__ void __launch_bounds__(32 * WM * WN * KG) k_dgemm(const DgemmDesc* __restrict__ descs, const DevState* st,
                                                             const IterScal* is, int check_state) {
  using Cf = DgCfg<BM, BN, BK, WM, WN, ST, KG>;
  constexpr int NT = Cf::NT, TM = Cf::TM, TN = Cf::TN, LDA0 = Cf::LDA0, LDK = Cf::LDK;
  if (check_state && (st->done || !is->proceed)) return;
  const DgemmDesc g = descs[blockIdx.z];
  if (g.gate && *g.gate != 1) return;
  const int M = g.M, N = g.Ndev ? *g.Ndev : g.N, K = g.Kdev ? *g.Kdev : g.K;
  const int i0 = blockIdx.x * BM, j0 = blockIdx.y * BN;
  if (i0 >= M || j0 >= N) return;
  if (g.upper && i0 > j0 + BN - 1) return;
  extern __shared__ __align__(16) double dsm[];
  double* Asm = dsm;                     // [ST][ASZ]
  double* Bsm = dsm + ST * Cf::ASZ;      // [ST][BSZ]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kg = warp / (WM * WN);  // k-step group: steps kg, kg + KG, ... of every slice
  const int wm = warp % WM, wn = (warp / WM) % WN;
  const bool tA = g.transA != 0;

  auto issue = [&](int k0, int buf) {
    double* As = Asm + buf * Cf::ASZ;
    double* Bs = Bsm + buf * Cf::BSZ;
#pragma unroll
    for (int r = 0; r < (BM * BK / 2) / NT; ++r) {
      const int c = tid + r * NT;
      if (!tA) {  // column k of the tile: BM rows = BM / 2 chunks
        const int k = c / (BM / 2), ic = (c % (BM / 2)) * 2;
        const int gk = k0 + k, gi = i0 + ic;
        const int nb = gk < K ? max(0, min(2, M - gi)) * 8 : 0;
        cp_async16n(As + k * LDA0 + ic, g.A + (nb ? (size_t)gk * g.lda + gi : 0), nb);
      } else {    // row i of op(A) = column i of A: BK k's = BK / 2 chunks
        const int i = c / (BK / 2), kc = (c % (BK / 2)) * 2;
        const int gi = i0 + i, gk = k0 + kc;
        const int nb = gi < M ? max(0, min(2, K - gk)) * 8 : 0;
        cp_async16n(As + i * LDK + kc, g.A + (nb ? (size_t)gi * g.lda + gk : 0), nb);
      }
    }
#pragma unroll
    for (int r = 0; r < (BN * BK / 2) / NT; ++r) {  // column j of B: BK k's = BK / 2 chunks
      const int c = tid + r * NT;
      const int j = c / (BK / 2), kc = (c % (BK / 2)) * 2;
      const int gj = j0 + j, gk = k0 + kc;
      const int nb = gj < N ? max(0, min(2, K - gk)) * 8 : 0;
      cp_async16n(Bs + j * LDK + kc, g.B + (nb ? (size_t)gj * g.ldb + gk : 0), nb);
    }
    cp_async_commit();
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int ns = (K + BK - 1) / BK;
#pragma unroll
  for (int p = 0; p < ST - 1; ++p) {
    if (p < ns) issue(p * BK, p);
    else cp_async_commit();  // empty groups keep the wait count uniform
  }
  const int lr = lane >> 2, lk = lane & 3;
  for (int sl = 0; sl < ns; ++sl) {
    const int buf = sl % ST;
    cp_async_wait<ST - 2>();
    __syncthreads();
    // refill the buffer slice sl - 1 used (every warp is past it after the barrier)
    if (sl + ST - 1 < ns) issue((sl + ST - 1) * BK, (sl + ST - 1) % ST);
    else cp_async_commit();
    const double* As = Asm + buf * Cf::ASZ;
    const double* Bs = Bsm + buf * Cf::BSZ;
#pragma unroll
    for (int kq = 0; kq < BK / (4 * KG); ++kq) {
      const int kk = 4 * (kq * KG + kg);
      double af[TM], bf[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) {
        const int m = wm * (BM / WM) + a * 8 + lr;
        af[a] = tA ? As[m * LDK + kk + lk] : As[(kk + lk) * LDA0 + m];
      }
#pragma unroll
      for (int b = 0; b < TN; ++b) bf[b] = Bs[(wn * (BN / WN) + b * 8 + lr) * LDK + kk + lk];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) dg_dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  if (KG > 1) {  // groups 1.. hand their partial tiles to group 0 through shared memory (fixed order)
    cp_async_wait<0>();
    __syncthreads();
    double* red = dsm;
    if (kg > 0) {
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            red[(size_t)(kg - 1) * BM * BN + ((((wn * WM + wm) * TM + a) * TN + b) * 2 + h) * 32 + lane] = acc[a][b][h];
    }
    __syncthreads();
    if (kg > 0) return;
#pragma unroll
    for (int q = 1; q < KG; ++q)
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            acc[a][b][h] += red[(size_t)(q - 1) * BM * BN + ((((wn * WM + wm) * TM + a) * TN + b) * 2 + h) * 32 + lane];
  }
  // epilogue: c0 / c1 of each 8 x 8 tile sit at (row lr, columns 2 lk, 2 lk + 1)
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const int gi = i0 + wm * (BM / WM) + a * 8 + lr;
    if (gi >= M) continue;
#pragma unroll
    for (int b = 0; b < TN; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = j0 + wn * (BN / WN) + b * 8 + 2 * lk + h;
        if (gj < N) {
          double* cp = g.C + (size_t)gj * g.ldc + gi;
          const double v = g.alpha * acc[a][b][h];
          if (g.mirror) {
            if (gi <= gj) {
              *cp = v;
              if (gi < gj) g.C[(size_t)gi * g.ldc + gj] = v;
            }
          } else {
            *cp = (g.beta == 0.0) ? v : fma(g.beta, *cp, v);
          }
        }
      }
  }
}

// Variants (debug entry point sosadmm_debug_dgemm selects one; the warm path uses DG_DEFAULT).
#define DG_VARIANTS(X)            \
  X(0, 64, 64, 16, 2, 2, 4, 1)    \
  X(1, 32, 64, 16, 1, 4, 4, 1)    \
  X(2, 64, 32, 16, 2, 2, 4, 1)    \
  X(3, 32, 64, 16, 1, 4, 4, 2)    \
  X(4, 64, 64, 16, 2, 2, 4, 2)    \
  X(5, 32, 64, 32, 1, 4, 3, 2)    \
  X(6, 64, 64, 32, 2, 2, 3, 2)    \
  X(7, 32, 32, 16, 1, 2, 4, 2)    \
  X(8, 64, 32, 16, 2, 2, 4, 2)    \
  X(9, 32, 64, 32, 1, 4, 3, 4)    \
  X(10, 32, 32, 16, 1, 2, 4, 4)   \
  X(11, 32, 32, 32, 1, 2, 3, 2)   \
  X(12, 32, 32, 32, 1, 2, 3, 4)   \
  X(13, 32, 32, 16, 2, 2, 4, 2)   \
  X(14, 32, 32, 16, 2, 2, 4, 1)   \
  X(15, 32, 32, 32, 2, 2, 3, 2)   \
  X(16, 32, 32, 32, 2, 2, 2, 2)   \
  X(17, 32, 32, 64, 2, 2, 2, 2)   \
  X(18, 32, 32, 32, 2, 2, 3, 4)   \
  X(19, 32, 64, 32, 2, 2, 3, 2)
constexpr int DG_NVAR = 20;
constexpr int DG_DEFAULT = 16;

// set the dynamic shared-memory attribute of every variant (outside any stream capture)
inline void dgemm_prepare() {
#define DG_ATTR(V, BM, BN, BK, WM, WN, ST, KG)                                                          \
  cudaFuncSetAttribute(k_dgemm<BM, BN, BK, WM, WN, ST, KG>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       (int)DgCfg<BM, BN, BK, WM, WN, ST, KG>::SMEM);
  DG_VARIANTS(DG_ATTR)
#undef DG_ATTR
}

inline void dgemm_launch(int variant, const DgemmDesc* d_descs, int batch, int maxM, int maxN, cudaStream_t s,
                         const DevState* st, const IterScal* is, int check) {
#define DG_CASE(V, BM, BN, BK, WM, WN, ST, KG)                                                                   \
  if (variant == V) {                                                                                        \
    using Cf = DgCfg<BM, BN, BK, WM, WN, ST, KG>;                                                            \
    dim3 gr((maxM + BM - 1) / BM, (maxN + BN - 1) / BN, batch);                                              \
    k_dgemm<BM, BN, BK, WM, WN, ST, KG><<<gr, Cf::NT, Cf::SMEM, s>>>(d_descs, st, is, check);                    \
    return;                                                                                                  \
  }
  DG_VARIANTS(DG_CASE)
#undef DG_CASE
}
