// Setup-time inverse of K = I + A_low^T P^{-1} A_low (t' x t', SPD, cond <= ~20 on the configs)
// on the GPU.  PAPER.md P:479-480: "its preferred factorization can be cached before iterating";
// CDCS-sos caches a sparse Cholesky.  Here the cache is the explicit K^{-1}, so that each
// iteration applies it as one bandwidth-bound dense GEMV (k_kinv) instead of two latency-bound
// triangular solves.  Three blocked stages, all trailing work on the DMMA GEMM:
//   1. K = L L^T      right-looking Cholesky, panel width 64 (diagonal block in one CTA,
//                     L21 = A21 L11^{-T} and A22 -= L21 L21^T as GEMMs);
//   2. X = L^{-1}     block forward substitution L X = I;
//   3. K^{-1} = X^T X.
#pragma once
#include <vector>

#include "common.cuh"
#include "gemm_f64.cuh"

constexpr int SPD_NB = 64;

// Unblocked Cholesky of the nb x nb diagonal block at (j0, j0) (column-major, leading dim t) and
// the inverse of that factor into Linv (nb x nb, column-major).
__global__ void __launch_bounds__(256) k_chol_diag(double* K, int t, int j0, int nb, double* Linv, int* fail) {
  __shared__ double L[SPD_NB][SPD_NB + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += 256) {
    const int i = e % nb, j = e / nb;
    L[i][j] = K[(size_t)(j0 + j) * t + j0 + i];
  }
  __syncthreads();
  for (int k = 0; k < nb; ++k) {
    if (tid == 0) {
      const double dkk = L[k][k];
      if (!(dkk > 0.0)) *fail = 1;
      L[k][k] = sqrt(fmax(dkk, 1e-300));
    }
    __syncthreads();
    const double dk = L[k][k];
    for (int i = k + 1 + tid; i < nb; i += 256) L[i][k] /= dk;
    __syncthreads();
    for (int e = tid; e < nb * nb; e += 256) {
      const int i = e % nb, j = e / nb;
      if (j > k && i >= j) L[i][j] -= L[i][k] * L[j][k];
    }
    __syncthreads();
  }
  // Linv = L^{-1} (lower): column c by forward substitution, one thread per column (each thread
  // reads back only the entries of its own column, so global memory is enough)
  if (tid < nb) {
    const int c = tid;
    double* xc = Linv + (size_t)c * SPD_NB;  // leading dimension SPD_NB for every block
    for (int i = 0; i < nb; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= L[i][k] * xc[k];
      xc[i] = (i < c) ? 0.0 : s / L[i][i];
    }
  }
  __syncthreads();
  for (int e = tid; e < nb * nb; e += 256) {
    const int i = e % nb, j = e / nb;
    K[(size_t)(j0 + j) * t + j0 + i] = (i >= j) ? L[i][j] : 0.0;
  }
}

// dst (rows x cols, ld t) = src (ld ldsrc)
__global__ void k_copy2d(double* dst, int ldd, const double* src, int lds, int rows, int cols) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)rows * cols) return;
  const int i = (int)(e % rows), j = (int)(e / rows);
  dst[(size_t)j * ldd + i] = src[(size_t)j * lds + i];
}

__global__ void k_transpose(double* dst, const double* src, int t) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int i = bx + threadIdx.x, j = by + y;
    if (i < t && j < t) tile[y][threadIdx.x] = src[(size_t)j * t + i];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int i = by + threadIdx.x, j = bx + y;
    if (i < t && j < t) dst[(size_t)j * t + i] = tile[threadIdx.x][y];
  }
}

__global__ void k_set_identity_block(double* R, int ldr, int rows, int col0, int nb) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * nb) return;
  const int i = e % rows, j = e / rows;
  R[(size_t)(col0 + j) * ldr + i] = (i == j) ? 1.0 : 0.0;
}

// Scratch of gpu_spd_inverse (carved from the caller's workspace: the library allocates nothing).
inline size_t spdinv_scratch_bytes(int t) {
  const size_t nb = SPD_NB, nblk = (t + nb - 1) / nb, tt = (size_t)t * t;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  return al(8 * t * nb) + al(8 * nblk * nb * nb) + al(8 * tt) + al(8 * nb * t) + al(sizeof(int)) +
         al(sizeof(GemmDesc) * (4 * nblk + 2)) + al(8 * tt) + 256;
}

// In-place K <- K^{-1} (t x t, column-major, full symmetric on input).  Returns 0, or 1 when K is
// not numerically positive definite, 2 on a CUDA error.  Temporaries live in `scratch`
// (>= spdinv_scratch_bytes(t) bytes of device memory).
inline int gpu_spd_inverse(double* K, int t, cudaStream_t s, char* scratch) {
  const int nb = SPD_NB;
  const int nblk = (t + nb - 1) / nb;
  double *T = nullptr, *Linv = nullptr, *X = nullptr, *R = nullptr;
  int* fail = nullptr;
  GemmDesc* dg = nullptr;
  std::vector<GemmDesc> gd;
  size_t used = ((uintptr_t)scratch + 255) / 256 * 256 - (uintptr_t)scratch;
  auto take = [&](size_t bytes) -> void* {
    void* p = scratch + used;
    used += (bytes + 255) / 256 * 256;
    return p;
  };
  auto gemm = [&](const double* A, int lda, const double* B, int ldb, int transB, double* C, int ldc, int M, int N,
                  int Kd, double alpha, double beta) {
    GemmDesc g{};
    g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.transB = transB; g.C = C; g.ldc = ldc;
    g.M = M; g.N = N; g.K = Kd; g.alpha = alpha; g.beta = beta;
    gd.push_back(g);
  };
  // plan every GEMM first (descriptors uploaded once)
  struct Step { int kind, j0, nbj, gi; };
  std::vector<Step> plan;
  const size_t tt = (size_t)t * t;
  T = (double*)take(sizeof(double) * (size_t)t * nb);
  Linv = (double*)take(sizeof(double) * (size_t)nblk * nb * nb);
  X = (double*)take(sizeof(double) * tt);
  R = (double*)take(sizeof(double) * (size_t)nb * t);
  fail = (int*)take(sizeof(int));
  // 1. Cholesky
  for (int b = 0; b < nblk; ++b) {
    const int j0 = b * nb, nbj = std::min(nb, t - j0), j1 = j0 + nbj, rest = t - j1;
    plan.push_back({0, j0, nbj, -1});
    if (rest > 0) {
      plan.push_back({1, j0, nbj, (int)gd.size()});
      gemm(K + (size_t)j0 * t + j1, t, Linv + (size_t)b * nb * nb, nb, 1, T, t, rest, nbj, nbj, 1.0, 0.0);
      plan.push_back({2, j0, nbj, (int)gd.size()});
      gemm(T, t, T, t, 1, K + (size_t)j1 * t + j1, t, rest, rest, nbj, -1.0, 1.0);
      plan.push_back({3, j0, nbj, -1});  // copy T -> L21
    }
  }
  // 2. X = L^{-1}: block row i: R = -L[i, 0:i] X[0:i, 0:i]; R[:, i] = I; X[i, 0:i+1] = Linv_ii R
  for (int b = 0; b < nblk; ++b) {
    const int j0 = b * nb, nbj = std::min(nb, t - j0);
    plan.push_back({4, j0, nbj, (int)gd.size()});  // (nbj x j0) = -L[i,0:j0] X[0:j0,0:j0]; then R[:, i] = I
    gemm(K + j0, t, X, t, 0, R, nb, nbj, j0, j0, -1.0, 0.0);
    plan.push_back({5, j0, nbj, (int)gd.size()});
    gemm(Linv + (size_t)b * nb * nb, nb, R, nb, 0, X + j0, t, nbj, j0 + nbj, nbj, 1.0, 0.0);
  }
  // 3. K^{-1} = X^T X: transpose X into T-sized? use K as X^T storage
  plan.push_back({6, 0, 0, (int)gd.size()});
  gemm(K, t, X, t, 0, nullptr, t, t, t, t, 1.0, 0.0);  // C filled below (X^T X into R? no: into X2)
  if (gd.size() > 4 * (size_t)nblk + 2) return 2;
  dg = (GemmDesc*)take(sizeof(GemmDesc) * (4 * (size_t)nblk + 2));
  // the last GEMM writes into a fresh buffer (X is its input)
  double* Y = (double*)take(sizeof(double) * tt);
  gd.back().C = Y;
  cudaMemcpyAsync(dg, gd.data(), sizeof(GemmDesc) * gd.size(), cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(fail, 0, sizeof(int), s);
  cudaMemsetAsync(X, 0, sizeof(double) * tt, s);
  for (const Step& st : plan) {
    const int b = st.j0 / nb;
    switch (st.kind) {
      case 0:
        k_chol_diag<<<1, 256, 0, s>>>(K, t, st.j0, st.nbj, Linv + (size_t)b * nb * nb, fail);
        break;
      case 1:
      case 2:
      case 4:
      case 5: {
        const GemmDesc& g = gd[st.gi];
        dim3 gr((g.M + GM_BM - 1) / GM_BM, (g.N + GM_BN - 1) / GM_BN, 1);
        if (g.M > 0 && g.N > 0) k_gemm_f64<<<gr, GM_NT, 0, s>>>(dg + st.gi, nullptr, nullptr, 0);
        if (st.kind == 4) {
          // R[:, i-block] = identity block
          k_set_identity_block<<<(st.nbj * st.nbj + 255) / 256, 256, 0, s>>>(R, nb, st.nbj, st.j0, st.nbj);
        }
        break;
      }
      case 3: {
        const int j1 = st.j0 + st.nbj, rest = t - j1;
        const long long cnt = (long long)rest * st.nbj;
        k_copy2d<<<(int)((cnt + 255) / 256), 256, 0, s>>>(K + (size_t)st.j0 * t + j1, t, T, t, rest, st.nbj);
        break;
      }
      case 6: {
        // K <- X^T (transposed copy), then Y = K * X
        dim3 tb(32, 8), tg((t + 31) / 32, (t + 31) / 32);
        k_transpose<<<tg, tb, 0, s>>>(K, X, t);
        const GemmDesc& g = gd[st.gi];
        dim3 gr((g.M + GM_BM - 1) / GM_BM, (g.N + GM_BN - 1) / GM_BN, 1);
        k_gemm_f64<<<gr, GM_NT, 0, s>>>(dg + st.gi, nullptr, nullptr, 0);
        cudaMemcpyAsync(K, Y, sizeof(double) * tt, cudaMemcpyDeviceToDevice, s);
        break;
      }
    }
  }
  int hfail = 0;
  cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return hfail ? 1 : (cudaGetLastError() == cudaSuccess ? 0 : 2);
}
