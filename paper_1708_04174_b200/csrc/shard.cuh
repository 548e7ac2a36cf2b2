// Multi-GPU block sharding of one program (north_star: "partition the blocks across the
// GPUs of one 8xB200 box and NCCL-allreduce the length-m A2 x partial sums over NVLink each
// iteration").
//
// The PSD blocks are owned by ranks; the free columns are counted by rank 0.  Per iteration every
// rank forms the partial sums of the gather (`E:SecondBlockElimination`: the -A w_1 term)
// over the columns it owns,
//     buf = [ (A w_1)_alpha (m) | (A xi)_alpha (m) | sum ||(A^T y + z)_orth||^2 | two low-column
//             dual-residual sums ]                                   (2m + 3 doubles),
// one ncclAllReduce(sum) over NVLink completes them, and everything that follows the gather (the
// diagonal scale, the t' x t' Woodbury solve, the rank-one HSDE correction and the tau / kappa
// update) runs replicated and bit-identically on every rank; the scatter, the PSD
// projections and the dual update touch the owned blocks only.  A rank with no PSD block still runs
// the replicated part.
#pragma once
#include "affine.cuh"

constexpr int SH_NT = 256;

struct ShardArgs {
  const int* colown;   // n: 1 if this rank accounts for column j in the partial sums
  double* buf;         // 2m + 3: all-reduced partial sums (NCCL mode); peer mode: 2 x (2m + 3) by epoch parity
  double* part;        // 3 * nblk_part: per-CTA partials of the three scalars
  int nparts;          // number of per-CTA partial slots per scalar
  // ---- peer mode (f4: the reduction fused into the consumer over peer memory, no NCCL call) ----
  unsigned long long* epoch;             // device round counter (replicated; nullptr = NCCL mode)
  unsigned long long* flags;             // [world] arrival epochs written by the peers (P2P stores)
  double* const* peer_buf;               // [world] every rank's 2 x (2m + 3) partial buffers (own included)
  unsigned long long* const* peer_flags; // [world] every rank's flag array
  double* red3;                          // the three reduced scalars (k_tphase's shard_scal)
  int world, rank;
};

// Partial-sum buffer of this round: peer mode alternates two buffers by epoch parity (a rank can be at
// most one round ahead of a peer still reading its previous round), NCCL mode has one.
__device__ __forceinline__ double* shard_buf(const ShardArgs& s, int m) {
  return s.epoch ? s.buf + (size_t)(*s.epoch & 1ull) * (2 * (size_t)m + 3) : s.buf;
}

// Per-row partial sums over the owned columns (the sharded counterpart of k_gather's first half).
__global__ void __launch_bounds__(SH_NT) k_gather_part(AffineArgs a, ShardArgs s) {
  __shared__ double sh[SH_NT / 32];
  if (a.st->done) return;
  const int r = blockIdx.x * SH_NT + threadIdx.x;
  double dres = 0.0;
  if (r < a.m) {
    const double yr = a.y[r];
    double gx = 0.0, gz = 0.0;
    for (int e = a.seg_ptr[r]; e < a.seg_ptr[r + 1]; ++e) {
      const int j = a.seg_col[e];
      if (!s.colown[j]) continue;
      const double v = a.seg_val[e];
      const double xj = a.xi[j], zj = a.z[j];
      gx = fma(v, xj, gx);
      gz = fma(v, zj, gz);
      const double d = fma(v, yr, zj);
      dres = fma(d, d, dres);
    }
    double gl = 0.0, axl = 0.0;
    for (int e = a.lr_ptr[r]; e < a.lr_ptr[r + 1]; ++e) {
      const int j = a.low_col[a.lr_idx[e]];
      if (!s.colown[j]) continue;
      const double v = a.lr_val[e];
      const double xj = a.xi[j];
      gl = fma(v, xj + a.z[j], gl);
      axl = fma(v, xj, axl);
    }
    double* buf = shard_buf(s, a.m);
    buf[r] = (gx + gz) + gl;
    buf[a.m + r] = gx + axl;
  }
  const double v = block_sum<SH_NT>(dres, sh);
  if (threadIdx.x == 0) s.part[blockIdx.x] = v;
}

// Low-column dual residuals over the owned low and empty columns (k_tphase's dl, dl0):
// one warp per low column, (A_low^T y + z - c tau)^2 and (A_low^T y + z)^2.
__global__ void __launch_bounds__(SH_NT) k_lowdual_part(AffineArgs a, ShardArgs s) {
  __shared__ double sh[SH_NT / 32];
  if (a.st->done) return;
  const double tau = a.st->tau;
  const int wid = (blockIdx.x * SH_NT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  double dl = 0.0, dl0 = 0.0;
  if (wid < a.tl && s.colown[a.low_col[wid]]) {
    double sy = 0.0;
    for (int e = a.lc_ptr[wid] + lane; e < a.lc_ptr[wid + 1]; e += 32) sy = fma(a.lc_val[e], a.y[a.lc_row[e]], sy);
    sy = warp_sum(sy);
    if (lane == 0) {
      const double d0 = sy + a.z[a.low_col[wid]];
      const double d = d0 - a.c_low[wid] * tau;
      dl = d * d;
      dl0 = d0 * d0;
    }
  }
  // empty orthogonal columns: one per thread after the warps of the low columns
  const int nwarps = gridDim.x * (SH_NT / 32);
  for (int j = blockIdx.x * SH_NT + threadIdx.x; j < a.n_empty; j += nwarps * 32) {
    const int col = a.empty_cols[j];
    if (s.colown[col]) {
      const double zj = a.z[col];
      dl = fma(zj, zj, dl);
      dl0 = fma(zj, zj, dl0);
    }
  }
  double v = block_sum<SH_NT>(dl, sh);
  if (threadIdx.x == 0) s.part[s.nparts + blockIdx.x] = v;
  v = block_sum<SH_NT>(dl0, sh);
  if (threadIdx.x == 0) s.part[2 * s.nparts + blockIdx.x] = v;
}

// Fixed-order reduction of the per-CTA scalar partials into buf[2m .. 2m+2] (before the allreduce).
__global__ void __launch_bounds__(SH_NT) k_shard_scalars(AffineArgs a, ShardArgs s, int nb_gather, int nb_low) {
  __shared__ double sh[SH_NT / 32];
  if (a.st->done) return;
  const int cnt[3] = {nb_gather, nb_low, nb_low};
  for (int q = 0; q < 3; ++q) {
    double v = 0.0;
    for (int i = threadIdx.x; i < cnt[q]; i += SH_NT) v += s.part[q * s.nparts + i];
    v = block_sum<SH_NT>(v, sh);
    if (threadIdx.x == 0) shard_buf(s, a.m)[2 * a.m + q] = v;
  }
}

// After the allreduce: the rest of k_gather, replicated (x = P^{-1}(w2 - g), residual partials).
__global__ void __launch_bounds__(GATHER_NT) k_gather_fin(AffineArgs a, ShardArgs s) {
  __shared__ double sh[6 * (GATHER_NT / 32)];
  if (a.st->done) return;
  const double tau = a.st->tau;
  const int r = blockIdx.x * GATHER_NT + threadIdx.x;
  double p_pres = 0, p_axi = 0, p_by = 0;
  dd bxd{0.0, 0.0};
  if (r < a.m) {
    const double g = s.buf[r];
    const double axi = s.buf[a.m + r];
    const double yr = a.y[r];
    const double xr = ((yr + a.s[r]) - g) * a.Pinv[r];
    a.x[r] = xr;
    const double pr = axi - a.b[r] * tau;
    bxd = dd_prod(a.b[r], xr);
    p_pres = pr * pr;
    p_axi = axi * axi;
    p_by = a.b[r] * yr;
  }
  gather_part_sums<GATHER_NT>(bxd, p_pres, p_axi, 0.0, p_by, sh, a.part, a.gather_blocks, blockIdx.x, true,
                              (blockIdx.x == 0) ? s.buf[2 * a.m] : 0.0);
}

// ---- peer mode ----
// Arrival: this rank's partials of round E are complete (stream order); publish E + 1 into every peer's
// flag slot `rank` (system-scope release after a system fence: the peers read the partials over NVLink)
// and advance the local epoch.  One thread.
__global__ void k_peer_signal(AffineArgs a, ShardArgs s) {
  if (a.st->done) return;
  const unsigned long long e = *s.epoch + 1ull;
  __threadfence_system();
  for (int q = 0; q < s.world; ++q) {
    unsigned long long* f = s.peer_flags[q] + s.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
  }
  *s.epoch = e;
}

__device__ __forceinline__ unsigned long long peer_ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double peer_ld(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// k_gather_fin with the allreduce fused in: wait until every rank published round E (local flags,
// written by the peers), then read the round's partial sums of EVERY rank straight from their memory
// (NVLink peer loads) and add them in rank order — deterministic, and the same order as the one-GPU
// emulation's device sum.  CTA 0 also reduces the three scalars into red3 for k_tphase.
__global__ void __launch_bounds__(GATHER_NT) k_gather_fin_peer(AffineArgs a, ShardArgs s) {
  __shared__ double sh[6 * (GATHER_NT / 32)];
  if (a.st->done) return;
  const unsigned long long e = *s.epoch;  // = E + 1 after k_peer_signal
  if (threadIdx.x == 0) {
    unsigned long long t0 = 0;
    unsigned spins = 0;
    for (int q = 0; q < s.world; ++q)
      while (peer_ld_acquire(s.flags + q) < e) {
        __nanosleep(64);
        if ((++spins & 0xFFFu) == 0) {  // a lost peer traps after 20 s instead of hanging the GPU
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          if (t0 == 0) t0 = now;
          else if (now - t0 > 20000000000ull) __trap();
        }
      }
    __threadfence_system();
  }
  __syncthreads();
  const size_t len = 2 * (size_t)a.m + 3, off = (size_t)((e - 1ull) & 1ull) * len;
  auto sum = [&](size_t i) {
    double v = 0.0;
    for (int q = 0; q < s.world; ++q) v += peer_ld(s.peer_buf[q] + off + i);
    return v;
  };
  const double tau = a.st->tau;
  const int r = blockIdx.x * GATHER_NT + threadIdx.x;
  double p_pres = 0, p_axi = 0, p_by = 0;
  dd bxd{0.0, 0.0};
  if (r < a.m) {
    const double g = sum(r);
    const double axi = sum(a.m + r);
    const double yr = a.y[r];
    const double xr = ((yr + a.s[r]) - g) * a.Pinv[r];
    a.x[r] = xr;
    const double pr = axi - a.b[r] * tau;
    bxd = dd_prod(a.b[r], xr);
    p_pres = pr * pr;
    p_axi = axi * axi;
    p_by = a.b[r] * yr;
  }
  double dres0 = 0.0;
  if (blockIdx.x == 0 && threadIdx.x < 3) {
    const double v = sum(2 * (size_t)a.m + threadIdx.x);
    s.red3[threadIdx.x] = v;
    if (threadIdx.x == 0) dres0 = v;
  }
  gather_part_sums<GATHER_NT>(bxd, p_pres, p_axi, 0.0, p_by, sh, a.part, a.gather_blocks, blockIdx.x, true,
                              (blockIdx.x == 0) ? dres0 : 0.0);
}

// get_iterate in sharded mode: keep the owned entries of a column vector, zero the rest, so that an
// allreduce(sum) over the ranks assembles the full vector exactly.
__global__ void k_mask_owned(const double* src, const int* colown, double* dst, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) dst[j] = colown[j] ? src[j] : 0.0;
}
