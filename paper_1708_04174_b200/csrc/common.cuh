// Common device helpers for the sosadmm kernels (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#define SOS_WARP 32

// Device-resident scalar state of the iterate (u, v) = ((xi, y, tau), (z, s, kappa)).
struct DevState {
  double tau, kappa;
  long long iter;        // k of u^k
  int done;              // latched termination (all kernels early-exit when set)
  int status;            // sosadmm_status of the last check
  double res_pri, res_dual, res_gap, pobj, dobj, pinf, dinf;
  int nonfinite;         // set when a non-finite residual / scalar is seen
  long long nonfinite_iter;
  long long max_iters;
  double tol;
};

// Per-iteration scratch scalars written by the t-phase kernel.
struct IterScal {
  double omega3;   // tau + kappa
  double coef;     // multiplier of h in u_hat_12 = q - coef h; equals u_hat_3 (reading C15)
  double u3;       // u_hat_3 = (w3 + zeta^T q) / (1 + zeta^T h)
  double tau_new, kappa_new;
  double bsig2;    // b^T sigma_2
  int proceed;     // 1 if this iteration continues past the t-phase
};

// Number of per-CTA partial sums the gather kernel produces.
enum { PART_BX = 0, PART_PRES, PART_AXI, PART_DRES, PART_BY, PART_BXLO, NPART };

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  // deterministic: fixed shuffle tree then fixed smem order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) r += sh[i];
  }
  return r;  // valid in thread 0
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// zero-filling variant: copies `bytes` (0 or 8) and fills the rest of the 8-byte slot with zeros
__device__ __forceinline__ void cp_async8z(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0) : "memory");
}

__device__ __forceinline__ bool sos_finite(double x) { return isfinite(x); }

constexpr double SOS_RT2 = 1.4142135623730951;       // fl(sqrt 2)
constexpr double SOS_IRT2 = 0.70710678118654757;     // fl(1/sqrt 2)

// svec position q (0-based, 'U' packed column-major) -> (i, j), i <= j.
__device__ __forceinline__ void svec_ij(long long q, int& i, int& j) {
  double jd = floor((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
  long long jj = (long long)jd;
  while (jj * (jj + 1) / 2 > q) --jj;
  while ((jj + 1) * (jj + 2) / 2 <= q) ++jj;
  j = (int)jj;
  i = (int)(q - jj * (jj + 1) / 2);
}

// ---- double-double helpers (error-free transformations) for the few dot products whose
// accuracy decides u_hat_3 (reading C15) ----
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return dd{s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  const double e = s.lo + a.lo + b.lo;
  const double hi = s.hi + e;
  return dd{hi, e - (hi - s.hi)};
}
__device__ __forceinline__ dd dd_prod(double a, double b) {
  const double p = a * b;
  return dd{p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_warp_sum(dd v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd w{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
    v = dd_add(v, w);
  }
  return v;
}
template <int NT>
__device__ __forceinline__ dd dd_block_sum(dd v, double* sh) {  // sh: 2 * NT/32 doubles
  v = dd_warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    sh[2 * w] = v.hi;
    sh[2 * w + 1] = v.lo;
  }
  __syncthreads();
  dd r{0.0, 0.0};
  if (threadIdx.x == 0)
    for (int i = 0; i < NT / 32; ++i) r = dd_add(r, dd{sh[2 * i], sh[2 * i + 1]});
  return r;  // valid in thread 0
}

// The five per-CTA partials of the gather (b^T x in double-double, then pres, axi, dres, by) with the
// trees of dd_block_sum / block_sum — per-warp shuffle tree, then the warp partials in warp order, so the
// same bits — but ONE barrier, and the five sums by five threads.  sh: 6 * NT/32 doubles.  dres_own:
// thread 0 writes dres_val as the DRES partial (sharded: the all-reduced value) instead of the sum.
template <int NT>
__device__ __forceinline__ void gather_part_sums(dd bx, double p_pres, double p_axi, double p_dres, double p_by,
                                                 double* sh, double* part, int gb, int blk, bool dres_own,
                                                 double dres_val) {
  constexpr int W = NT / 32;
  bx = dd_warp_sum(bx);
  double v[4] = {p_pres, p_axi, p_dres, p_by};
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  if (l == 0) {
    sh[w] = bx.hi;
    sh[W + w] = bx.lo;
#pragma unroll
    for (int q = 0; q < 4; ++q) sh[(2 + q) * W + w] = v[q];
  }
  __syncthreads();
  if (t == 0) {
    dd r{0.0, 0.0};
    for (int i = 0; i < W; ++i) r = dd_add(r, dd{sh[i], sh[W + i]});
    part[PART_BX * gb + blk] = r.hi;
    part[PART_BXLO * gb + blk] = r.lo;
    if (dres_own) part[PART_DRES * gb + blk] = dres_val;
  } else if (t <= 4) {
    const int q = t - 1;
    const int k = q == 0 ? PART_PRES : (q == 1 ? PART_AXI : (q == 2 ? PART_DRES : PART_BY));
    if (!(dres_own && k == PART_DRES)) {
      double r = 0.0;
#pragma unroll
      for (int i = 0; i < W; ++i) r += sh[(2 + q) * W + i];
      part[k * gb + blk] = r;
    }
  }
}
