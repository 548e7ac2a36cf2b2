// Divide-and-conquer eigensolver for the symmetric tridiagonal T (second stage of the large-block
// PSD projection, north_star (c) "a tridiagonal solve").  Textbook Cuppen recursion restated for
// the GPU:
//   * a balanced bisection tree of depth D; all leaves (size 1 or 2) sit at depth D, so every level
//     merges disjoint nodes and the eigenvector matrices ping-pong between two N x N buffers;
//   * a cut at position k (T[k,k+1] = e_k) gives T = diag(T1', T2') + rho u u^T with rho = |e_k|,
//     u = e_k + sign(e_k) e_{k+1}, T1'/T2' with |e_k| subtracted from the two adjacent diagonals;
//   * a merge solves D + rho z z^T (z = [last row of Q1; sign(e_k) first row of Q2]):
//     - sort, deflate small |z_i| and close pairs by Givens rotations (LAPACK dlaed2 rules),
//     - one warp per secular root, origin at the nearer pole, bracketed rational (two-pole)
//       iteration with bisection safeguard,
//     - Gu-Eisenstat recomputation of z so that the eigenvectors u_j = z_hat / (d - lambda_j) are
//       numerically orthogonal,
//     - Q_new = Q_old[:, nondeflated] * U on the FP64 tensor cores (k_gemm_f64); deflated columns
//       are copied; eigenvalues are merged into ascending order.
#pragma once
#include "common.cuh"
#include "gemm_f64.cuh"

constexpr double DC_EPS = 2.220446049250313e-16;
constexpr int DC_NT = 256;

struct DcNode {
  int s, n1, n;
  long long u_off;  // offset of this node's k x k matrix U in the level's U buffer
};

struct DcArgs {
  int N;
  const double* d;     // tridiagonal diagonal (N)
  const double* e;     // off-diagonal (N-1)
  double* dmod;        // modified diagonal for the leaves
  double* Q[2];        // N x N ping-pong eigenvector buffers
  double* lam[2];      // eigenvalues
  const DcNode* nodes; // all nodes, level by level
  const int* pos2node; // per level: node index of every position (D x N)
  // position-indexed scratch (N each)
  double *ndd, *ndz, *dfv, *tau_r, *zhat, *lam_r;
  int *ndcol, *dfcol, *org, *outcol;
  // node-indexed
  int* node_k;
  int* node_nd;
  double* node_rho;
  double* U;           // level U buffer (<= N^2)
  int* rot_pq;         // 2 ints per rotation (position-indexed, N)
  double* rot_cs;      // 2 doubles per rotation
  int* rot_cnt;        // node-indexed
  const DevState* st;
  const IterScal* is;
  int check_state;
  // top-level selection (partial spectrum): the projection needs only the spectral
  // side with fewer eigenpairs (k_select's rule), so the root merge forms only those eigenvectors.
  // topsel = [selected root count, first selected root, side (0 = lambda > 0, 1 = lambda < 0,
  // -1 = all)]; topsel_on = 0 keeps every eigenvector (the stage tests).
  int* topsel;
  int topsel_on;
  const int* topsel_full;  // optional device flag: nonzero = keep every eigenvector this time (warm.cuh re-seed)
};

__device__ __forceinline__ bool dc_skip(const DcArgs& a) {
  return a.check_state && (a.st->done || !a.is->proceed);
}

// Leaves of size 1 or 2 (closed form); also sets Q[buf] diagonal blocks.
__global__ void k_dc_leaf(DcArgs a, int first_leaf, int nleaves, int buf) {
  if (dc_skip(a)) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nleaves) return;
  const DcNode nd = a.nodes[first_leaf + t];
  const int N = a.N, s = nd.s, n = nd.n;
  double* Q = a.Q[buf];
  double* lam = a.lam[buf];
  // cuts: at the left boundary (if s > 0) and at the right boundary (if s + n < N)
  auto dm = [&](int i) {
    double v = a.d[i];
    if (i == s && s > 0) v -= fabs(a.e[s - 1]);
    if (i == s + n - 1 && s + n < N) v -= fabs(a.e[s + n - 1]);
    return v;
  };
  if (n == 1) {
    lam[s] = dm(s);
    Q[(size_t)s * N + s] = 1.0;
  } else {
    const double p = dm(s), r = dm(s + 1), q = a.e[s];
    double c = 1.0, sn = 0.0, l1 = p, l2 = r;
    if (q != 0.0) {
      const double th = (r - p) / (2.0 * q);
      const double t2 = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(fma(th, th, 1.0)));
      c = 1.0 / sqrt(fma(t2, t2, 1.0));
      sn = t2 * c;
      l1 = p - t2 * q;
      l2 = r + t2 * q;
    }
    // eigenvectors: (c, -sn) for l1, (sn, c) for l2
    double v1a = c, v1b = -sn, v2a = sn, v2b = c;
    if (l1 > l2) {
      double tt = l1; l1 = l2; l2 = tt;
      tt = v1a; v1a = v2a; v2a = tt;
      tt = v1b; v1b = v2b; v2b = tt;
    }
    lam[s] = l1;
    lam[s + 1] = l2;
    Q[(size_t)s * N + s] = v1a;
    Q[(size_t)s * N + s + 1] = v1b;
    Q[(size_t)(s + 1) * N + s] = v2a;
    Q[(size_t)(s + 1) * N + s + 1] = v2b;
  }
}

// Bottom subtrees solved directly (replacing the lowest merge levels, whose kernels are latency-bound:
// ~7 dependent launches per level for nodes of a few rows).  One warp per node of size n <= DCJ_MAXN at
// depth D - L: the node's tridiagonal with the rank-one cuts of its ancestors applied at its boundaries
// (d_s -= |e_{s-1}|, d_{s+n-1} -= |e_{s+n-1}|, exactly the matrices the level-L merges would have
// diagonalised), then the implicit symmetric QR iteration with the Wilkinson shift (Golub-Van Loan,
// "implicit symmetric QR step with Wilkinson shift" + deflation of negligible off-diagonals) on the
// tridiagonal itself, and the eigenpairs in ascending order into lam[buf][s..s+n) and the node's
// diagonal block of Q[buf] — the format every merge expects of its children.
//   * step k of a chase: R = [[c, s], [-s, c]] with R [x; z] = [r; 0] on rows / columns (k, k+1): the
//     2 x 2 block (a, b; b, g) -> (c^2 a + 2cs b + s^2 g, cs (g - a) + (c^2 - s^2) b; ., s^2 a - 2cs b +
//     c^2 g), the coupling f = e_{k+1} -> c f and the bulge s f at (k+2, k); Z <- Z R^T;
//   * the scalars (d, e in shared memory, the running a, b, x, z in registers) are computed redundantly
//     by every lane; lane i owns row i of Z (shared memory, column-major by lane: conflict-free);
//   * deflation: lane i tests e_i (|e_i| <= eps (|d_i| + |d_{i+1}|) or <= eps ||T||) and a ballot
//     gives the unreduced trailing block [l, h]; the eigen-residual stays at the backward-error level
//     n eps ||T|| of the merges above.
// (Rounds 1-2 solved these nodes by cyclic Jacobi in a 256-thread CTA: ~60 us per launch in the graph,
// ~110 rounds of two barriers each.)
constexpr int DCJ_MAXN = 16;
constexpr int DCJ_NT = 32;
__global__ void __launch_bounds__(DCJ_NT) k_dc_qrnode(DcArgs a, int node0, int buf) {
  if (dc_skip(a)) return;
  constexpr int NM = DCJ_MAXN;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ double ds[NM + 1], es[NM + 1];
  __shared__ double Zs[NM][32];
  const DcNode nd = a.nodes[node0 + blockIdx.x];
  const int N = a.N, s = nd.s, n = nd.n, lane = threadIdx.x;
  double dv = 0.0, ev = 0.0;
  if (lane < n) {
    dv = a.d[s + lane];
    if (lane == 0 && s > 0) dv -= fabs(a.e[s - 1]);
    if (lane == n - 1 && s + n < N) dv -= fabs(a.e[s + n - 1]);
  }
  if (lane + 1 < n) ev = a.e[s + lane];
  if (lane <= NM) {
    ds[lane] = dv;
    es[lane] = ev;
  }
#pragma unroll
  for (int k = 0; k < NM; ++k) Zs[k][lane] = (k == lane) ? 1.0 : 0.0;
  double dm = fabs(dv), em = fabs(ev);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dm = fmax(dm, __shfl_xor_sync(FULL, dm, o));
    em = fmax(em, __shfl_xor_sync(FULL, em, o));
  }
  const double floor_abs = DC_EPS * fma(2.0, em, dm);
  __syncwarp();
  for (int it = 0; it < 30 * NM; ++it) {
    bool nz = false;
    if (lane + 1 < n) {
      const double ae = fabs(es[lane]);
      if (ae <= DC_EPS * (fabs(ds[lane]) + fabs(ds[lane + 1])) || ae <= floor_abs) es[lane] = 0.0;
      else nz = true;
    }
    const unsigned m = __ballot_sync(FULL, nz);
    __syncwarp();
    if (m == 0) break;
    const int h = 32 - __clz(m);                          // e_{h-1} != 0, e_h = 0
    const unsigned below = ~m & ((1u << (h - 1)) - 1u);  // zero couplings below h - 1
    const int l = below ? 32 - __clz(below) : 0;          // the unreduced block is [l, h]
    // Wilkinson shift from the trailing 2 x 2 block (d_{h-1}, e_{h-1}; e_{h-1}, d_h)
    const double dh1 = ds[h - 1], dh = ds[h], eh = es[h - 1];
    const double del = 0.5 * (dh1 - dh);
    const double h2 = fma(del, del, eh * eh);  // > 0: e_{h-1} is not negligible
    const double hy = h2 * rsqrt(h2);
    const double mu = dh - eh * eh / (del + (del >= 0.0 ? hy : -hy));
    double av = ds[l], bv = es[l];  // running d_k, e_k
    double x = av - mu, zz = bv;
    double zk = Zs[l][lane];        // running z_k of this lane's row
    for (int k = l; k < h; ++k) {
      const double gv = ds[k + 1];
      const double f = (k + 1 < h) ? es[k + 1] : 0.0;
      const double zk1 = Zs[k + 1][lane];
      // the chain x -> x' needs only 1 / r^2: b' = (x z (g - a) + (x^2 - z^2) b) / r^2
      const double r2 = fma(x, x, zz * zz);
      const double num = fma(x * zz, gv - av, (x - zz) * (x + zz) * bv);
      double c = 1.0, sn = 0.0, r = 0.0, bn = bv;
      if (r2 > 0.0) {
        const double ri = rsqrt(r2);
        c = x * ri;
        sn = zz * ri;
        r = r2 * ri;
        bn = num * (ri * ri);
      }
      if (k > l) es[k - 1] = r;
      const double cc = c * c, ss = sn * sn, csb = 2.0 * c * sn * bv;
      ds[k] = fma(ss, gv, fma(cc, av, csb));
      av = fma(ss, av, fma(cc, gv, -csb));
      Zs[k][lane] = fma(c, zk, sn * zk1);
      zk = fma(-sn, zk, c * zk1);
      if (k + 1 < h) {
        zz = sn * f;
        bv = c * f;
        x = bn;
      } else {
        ds[k + 1] = av;
        es[k] = bn;
        Zs[k + 1][lane] = zk;
      }
    }
    __syncwarp();
  }
  // ascending order (ties by index): lane j ranks eigenvalue j, then the columns go out contiguously
  int rank = 0;
  double lj = 0.0;
  if (lane < n) {
    lj = ds[lane];
    for (int i = 0; i < n; ++i) {
      const double li = ds[i];
      rank += (li < lj) || (li == lj && i < lane);
    }
    a.lam[buf][s + rank] = lj;
  }
  double* Q = a.Q[buf];
  for (int j = 0; j < n; ++j) {
    const int rj = __shfl_sync(FULL, rank, j);
    if (lane < n) Q[(size_t)(s + rj) * N + (s + lane)] = Zs[j][lane];
  }
}

// ordered stream compaction over [0, n) by one CTA of DC_NT threads: out[rank] = map(i) for the i
// with pred(i), in increasing i; returns the count (every thread).  wcnt: DC_NT/32 ints of SMEM.
template <class P, class M>
__device__ int dc_compact(int n, P pred, M map, int* out, int* wcnt) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int base = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += DC_NT) {
    const int i = i0 + tid;
    const bool p = i < n && pred(i);
    const unsigned m = __ballot_sync(0xffffffffu, p);
    if (lane == 0) wcnt[warp] = __popc(m);
    __syncthreads();
    int o = base;
    for (int w = 0; w < warp; ++w) o += wcnt[w];
    if (p) out[o + __popc(m & ((1u << lane) - 1u))] = map(i);
    for (int w = 0; w < DC_NT / 32; ++w) base += wcnt[w];
    __syncthreads();
  }
  return base;
}

// ---- merge step 1: z, sort, deflation (one CTA per node) ---------------------------------
constexpr int DC_MAXN = 1280;
__global__ void __launch_bounds__(DC_NT) k_dc_prep(DcArgs a, int node0, int ob) {
  if (dc_skip(a)) return;
  const int node = node0 + blockIdx.x;
  const DcNode nd = a.nodes[node];
  const int N = a.N, s = nd.s, n1 = nd.n1, n = nd.n;
  double* Qo = a.Q[ob];
  const double* lo = a.lam[ob];
  __shared__ double dsh[DC_MAXN], zsh[DC_MAXN];
  __shared__ int perm[DC_MAXN];
  __shared__ int ndl[DC_MAXN], dfl[DC_MAXN];
  __shared__ double red[DC_NT / 32];
  __shared__ int nk, ndf, nrot;
  __shared__ double rho_s;
  const int tid = threadIdx.x;
  const double er = a.e[s + n1 - 1];
  const double rho = fabs(er);
  const double sg = (er < 0.0) ? -1.0 : 1.0;
  // sorted merge of the two ascending child spectra (ties: left child first); the children's
  // eigenvalues are staged in shared memory (zsh as scratch) so the binary searches hit SMEM
  for (int i = tid; i < n; i += DC_NT) zsh[i] = lo[s + i];
  __syncthreads();
  for (int i = tid; i < n; i += DC_NT) {
    const double di = zsh[i];
    int rank;
    if (i < n1) {  // count right elements < di
      int l = 0, h = n - n1;
      while (l < h) {
        const int mid = (l + h) >> 1;
        if (zsh[n1 + mid] < di) l = mid + 1; else h = mid;
      }
      rank = i + l;
    } else {  // count left elements <= di
      int l = 0, h = n1;
      while (l < h) {
        const int mid = (l + h) >> 1;
        if (zsh[mid] <= di) l = mid + 1; else h = mid;
      }
      rank = (i - n1) + l;
    }
    perm[rank] = i;
  }
  __syncthreads();
  for (int r = tid; r < n; r += DC_NT) dsh[r] = zsh[perm[r]];
  __syncthreads();
  double z2 = 0.0, dmax = 0.0;
  for (int r = tid; r < n; r += DC_NT) {
    const int i = perm[r];
    const double zi = (i < n1) ? Qo[(size_t)(s + i) * N + (s + n1 - 1)] : sg * Qo[(size_t)(s + i) * N + (s + n1)];
    zsh[r] = zi;
    z2 = fma(zi, zi, z2);
    dmax = fmax(dmax, fabs(dsh[r]));
  }
  // block reductions (sum, max)
  z2 = warp_sum(z2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if ((tid & 31) == 0) red[tid >> 5] = z2;
  __syncthreads();
  double zn2 = 0.0;
  for (int w = 0; w < DC_NT / 32; ++w) zn2 += red[w];
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = dmax;
  __syncthreads();
  double dm = 0.0;
  for (int w = 0; w < DC_NT / 32; ++w) dm = fmax(dm, red[w]);
  __syncthreads();
  const double zn = sqrt(zn2);
  double zmax = 0.0;
  for (int r = tid; r < n; r += DC_NT) {
    zsh[r] = (zn > 0.0) ? zsh[r] / zn : 0.0;
    zmax = fmax(zmax, fabs(zsh[r]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
  if ((tid & 31) == 0) red[tid >> 5] = zmax;
  __syncthreads();
  double zm = 0.0;
  for (int w = 0; w < DC_NT / 32; ++w) zm = fmax(zm, red[w]);
  const double rhop = rho * zn2;  // rho z z^T = rhop zn zn^T with |zn| = 1
  const double tol = 8.0 * DC_EPS * fmax(dm, zm);
  // deflation (dlaed2 rules).  Type 1 (|z_r| small) is decided in parallel and compacted in order;
  // the close-pair scan (type 2), whose rotations change z and d of the running pair, runs in one
  // thread over the remaining candidates only.  Rotations are recorded for k_dc_rot.  The pair test
  // |t c s| <= tol is evaluated as |t z_r z_pj| <= tol (z_r^2 + z_pj^2) (c s = -z_r z_pj /
  // (z_r^2 + z_pj^2)), so hypot and divisions run only when a rotation happens.
  __shared__ int cand[DC_MAXN];
  __shared__ int wcnt[2][DC_NT / 32];
  __shared__ int ncand_s, ndf1_s;
  {
    const int warp = tid >> 5, lane = tid & 31;
    int base_c = 0, base_d = 0;
    for (int r0 = 0; r0 < n; r0 += DC_NT) {
      const int r = r0 + tid;
      const bool valid = r < n;
      const bool t1 = valid && rhop * fabs(zsh[r]) <= tol;
      const bool cd = valid && !t1;
      const unsigned mc = __ballot_sync(0xffffffffu, cd), md = __ballot_sync(0xffffffffu, t1);
      if (lane == 0) {
        wcnt[0][warp] = __popc(mc);
        wcnt[1][warp] = __popc(md);
      }
      __syncthreads();
      int oc = base_c, od = base_d;
      for (int w = 0; w < warp; ++w) {
        oc += wcnt[0][w];
        od += wcnt[1][w];
      }
      const unsigned below = (1u << lane) - 1u;
      if (cd) cand[oc + __popc(mc & below)] = r;
      if (t1) dfl[od + __popc(md & below)] = r;
      for (int w = 0; w < DC_NT / 32; ++w) {
        base_c += wcnt[0][w];
        base_d += wcnt[1][w];
      }
      __syncthreads();
    }
    if (tid == 0) {
      ncand_s = base_c;
      ndf1_s = base_d;
    }
  }
  __syncthreads();
  // Type 2 (close pairs).  The sequential rule: step c pairs r = cand[c] with pj = cand[c-1] (its
  // values modified iff step c-1 rotated).  Step 1 (parallel): the pair test of every consecutive
  // pair on the ORIGINAL values, compacted into a list of flagged steps (ndl as scratch).  Step 2
  // (one thread): only rotation chains are walked — a chain starts at a flagged step whose
  // predecessor did not rotate and continues while the modified pj keeps rotating, so the work is
  // the number of flagged steps + rotations, not n.  Step 3 (parallel): ordered compaction of the
  // non-deflated candidates and the type-2 deflations (= the pj of every rotation, in step order).
  const int nc = ncand_s, ndf1 = ndf1_s;
  auto ptest = [&](double zr, double dr, double zp, double dp) {
    return fabs((dr - dp) * zr * zp) <= tol * fma(zr, zr, zp * zp);
  };
  __shared__ int rotf[DC_MAXN];
  __shared__ int wcnt3[DC_NT / 32];
  for (int c = tid; c < nc; c += DC_NT) rotf[c] = 0;
  const int nf = dc_compact(
      nc,
      [&](int c) {
        return c >= 1 && ptest(zsh[cand[c]], dsh[cand[c]], zsh[cand[c - 1]], dsh[cand[c - 1]]);
      },
      [&](int c) { return c; }, ndl, wcnt3);
  if (tid == 0) {
    int nr = 0, cend = 0;  // steps < cend are settled
    for (int u = 0; u < nf; ++u) {
      int c = ndl[u];
      if (c < cend) continue;
      int pj = cand[c - 1];
      double zp = zsh[pj], dp = dsh[pj];
      for (; c < nc; ++c) {
        const int r = cand[c];
        const double zr = zsh[r], dr = dsh[r];
        if (!ptest(zr, dr, zp, dp)) break;
        const double tt = sqrt(fma(zr, zr, zp * zp));
        const double cv = zr / tt, sv = -zp / tt;
        zsh[r] = tt;
        zsh[pj] = 0.0;
        const int rp = s + nr;
        a.rot_pq[2 * rp] = s + perm[pj];
        a.rot_pq[2 * rp + 1] = s + perm[r];
        a.rot_cs[2 * rp] = cv;
        a.rot_cs[2 * rp + 1] = sv;
        ++nr;
        const double t1 = dp * cv * cv + dr * sv * sv;
        const double dnew = dp * sv * sv + dr * cv * cv;
        dsh[r] = dnew;
        dsh[pj] = t1;
        rotf[c] = 1;
        pj = r;
        zp = tt;
        dp = dnew;
      }
      cend = c + 1;
    }
    nrot = nr;
    rho_s = rhop;
  }
  __syncthreads();
  const int nkeep = dc_compact(
      nc, [&](int c) { return !(c + 1 < nc && rotf[c + 1]); }, [&](int c) { return cand[c]; }, ndl, wcnt3);
  const int ndf2 = dc_compact(
      nc, [&](int c) { return c + 1 < nc && rotf[c + 1]; }, [&](int c) { return cand[c]; }, dfl + ndf1, wcnt3);
  if (tid == 0) {
    nk = nkeep;
    ndf = ndf1 + ndf2;
  }
  __syncthreads();
  const int k = nk, df = ndf, nr = nrot;
  for (int i = tid; i < k; i += DC_NT) {
    const int r = ndl[i];
    a.ndd[s + i] = dsh[r];
    a.ndz[s + i] = zsh[r];
    a.ndcol[s + i] = s + perm[r];
  }
  for (int i = tid; i < df; i += DC_NT) {
    const int r = dfl[i];
    a.dfv[s + i] = dsh[r];
    a.dfcol[s + i] = s + perm[r];
  }
  if (tid == 0) {
    a.node_k[node] = k;
    a.node_nd[node] = df;
    a.node_rho[node] = rho_s;
    a.rot_cnt[node] = nr;
  }
}

// ---- merge step 2: secular roots, one warp per root ----------------------------------------
// f(lambda) = 1/rho + sum_i z_i^2 / (d_i - lambda), increasing between consecutive poles.
__global__ void __launch_bounds__(DC_NT) k_dc_secular(DcArgs a, int level) {
  if (dc_skip(a)) return;
  const int N = a.N;
  const int p = (blockIdx.x * DC_NT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (p >= N) return;
  const int node = a.pos2node[(size_t)level * N + p];
  const DcNode nd = a.nodes[node];
  const int s = nd.s, j = p - s, k = a.node_k[node];
  if (j >= k) return;
  const double* d = a.ndd + s;
  const double* z = a.ndz + s;
  const double rho = a.node_rho[node];
  const double rinv = 1.0 / rho;
  int org;
  double lo, hi;
  if (k == 1) {
    if (lane == 0) {
      a.org[p] = 0;
      a.tau_r[p] = rho * z[0] * z[0];
      a.lam_r[p] = d[0] + rho * z[0] * z[0];
    }
    return;
  }
  if (j < k - 1) {
    const double mid = 0.5 * (d[j + 1] - d[j]);
    double f = 0.0;
    for (int i = lane; i < k; i += 32) f += z[i] * z[i] / ((d[i] - d[j]) - mid);
    f = rinv + warp_sum(f);
    if (f >= 0.0) {
      org = j;
      lo = 0.0;
      hi = mid;
    } else {
      org = j + 1;
      lo = -mid;
      hi = 0.0;
    }
  } else {
    double zz = 0.0;
    for (int i = lane; i < k; i += 32) zz = fma(z[i], z[i], zz);
    zz = warp_sum(zz);
    org = k - 1;
    lo = 0.0;
    hi = rho * zz;
  }
  const double dorg = d[org];
  const double dl = d[j] - dorg;                             // left pole (shifted)
  const double dr = (j < k - 1) ? d[j + 1] - dorg : 0.0;     // right pole (shifted)
  double tau = 0.5 * (lo + hi);
  for (int it = 0; it < 200; ++it) {
    double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0, asum = 0.0;
    for (int i = lane; i < k; i += 32) {
      const double del = (d[i] - dorg) - tau;
      const double r = z[i] / del;
      const double term = z[i] * r;
      if (i <= j) {
        psi += term;
        dpsi = fma(r, r, dpsi);
      } else {
        phi += term;
        dphi = fma(r, r, dphi);
      }
      asum += fabs(term);
    }
    psi = warp_sum(psi);
    dpsi = warp_sum(dpsi);
    phi = warp_sum(phi);
    dphi = warp_sum(dphi);
    asum = warp_sum(asum);
    const double g = rinv + psi + phi;
    if (g < 0.0) lo = tau; else hi = tau;
    if (fabs(g) <= 8.0 * DC_EPS * (rinv + asum) * (1.0 + 0.0625 * k) || g == 0.0) break;
    // two-pole rational model through (tau, g, g')
    const double D1 = dl - tau;
    double eta;
    bool ok = true;
    if (j < k - 1) {
      const double D2 = dr - tau;
      const double B1 = dpsi * D1 * D1, B2 = dphi * D2 * D2;
      const double c = g - B1 / D1 - B2 / D2;
      const double bq = c * (D1 + D2) + B1 + B2;  // c eta^2 - bq eta + D1 D2 g = 0
      const double cq = D1 * D2 * g;
      if (c == 0.0) {
        eta = cq / bq;
      } else {
        const double disc = bq * bq - 4.0 * c * cq;
        if (disc < 0.0) {
          ok = false;
          eta = 0.0;
        } else {
          const double sq = sqrt(disc);
          const double qq = 0.5 * (bq + (bq >= 0.0 ? sq : -sq));
          const double e1 = qq / c, e2 = (qq != 0.0) ? cq / qq : e1;
          const bool in1 = (tau + e1 > lo) && (tau + e1 < hi);
          const bool in2 = (tau + e2 > lo) && (tau + e2 < hi);
          if (in1 && in2) eta = (fabs(e1) < fabs(e2)) ? e1 : e2;
          else if (in1) eta = e1;
          else if (in2) eta = e2;
          else ok = false;
        }
      }
    } else {
      const double B1 = dpsi * D1 * D1;
      const double c = g - B1 / D1;
      eta = (c != 0.0) ? D1 + B1 / c : 0.0;
      if (c == 0.0) ok = false;
    }
    double tn = tau + eta;
    if (!ok || !(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
    const bool conv = fabs(tn - tau) <= 2.0 * DC_EPS * fabs(tn);
    tau = tn;
    if (conv || hi - lo <= 2.0 * DC_EPS * fmax(fabs(lo), fabs(hi))) break;
  }
  if (lane == 0) {
    a.org[p] = org;
    a.tau_r[p] = tau;
    a.lam_r[p] = dorg + tau;
  }
}

// ---- merge step 3: Gu-Eisenstat z_hat, one warp per position i ------------------------------
__global__ void __launch_bounds__(DC_NT) k_dc_zhat(DcArgs a, int level) {
  if (dc_skip(a)) return;
  const int N = a.N;
  const int p = (blockIdx.x * DC_NT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (p >= N) return;
  const int node = a.pos2node[(size_t)level * N + p];
  const int s = a.nodes[node].s, i = p - s, k = a.node_k[node];
  if (i >= k) return;
  const double* d = a.ndd + s;
  const double rho = a.node_rho[node];
  double prod = 1.0;
  for (int j = lane; j < k; j += 32) {
    const double del = (d[i] - d[a.org[s + j]]) - a.tau_r[s + j];  // d_i - lambda_j
    if (j == i) prod *= -del / rho;
    else prod *= -del / (d[j] - d[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) prod *= __shfl_xor_sync(0xffffffffu, prod, o);
  if (lane == 0) a.zhat[p] = copysign(sqrt(fmax(prod, 0.0)), a.ndz[p]);
}

// ---- merge step 4: eigenvector matrix U (k x k) and output ranks, one warp per root j -------
__global__ void __launch_bounds__(DC_NT) k_dc_vec(DcArgs a, int level, int nb, int top) {
  if (dc_skip(a)) return;
  const int N = a.N;
  const int p = (blockIdx.x * DC_NT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (p >= N) return;
  const int node = a.pos2node[(size_t)level * N + p];
  const DcNode nd = a.nodes[node];
  const int s = nd.s, j = p - s, k = a.node_k[node], df = a.node_nd[node];
  if (j >= k) return;
  const double* d = a.ndd + s;
  const double dj = d[a.org[p]], tj = a.tau_r[p];
  double* U = a.U + nd.u_off + (size_t)j * nd.n;  // column stride n (static upper bound of k)
  if (!top || (j >= a.topsel[1] && j < a.topsel[1] + a.topsel[0])) {  // root: selected columns only
    double nrm = 0.0;
    for (int i = lane; i < k; i += 32) {
      const double u = a.zhat[s + i] / ((d[i] - dj) - tj);
      U[i] = u;
      nrm = fma(u, u, nrm);
    }
    nrm = warp_sum(nrm);
    const double inv = 1.0 / sqrt(nrm);
    for (int i = lane; i < k; i += 32) U[i] *= inv;
  }
  // rank among (roots ascending) U (deflated values; deflated first on ties)
  const double lj = a.lam_r[p];
  int cnt = 0;
  for (int q = lane; q < df; q += 32) cnt += (a.dfv[s + q] <= lj) ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) {
    const int rank = j + cnt;
    a.outcol[p] = s + rank;
    a.lam[nb][s + rank] = lj;
  }
}

// ---- merge step 1b: the deflation rotations applied to the columns of Q_old (drot:
// x' = c x + s y, y' = c y - s x), one thread per row.  In dlaed2's scan every rotation pairs the
// running column pj with a fresh column r, and r becomes the next pj, so the rotated r column is
// carried in a register (only the fresh column is loaded; it does not depend on earlier rotations,
// so those loads overlap) and the finished pj column is stored at once. ----
constexpr int DCR_NT = 128;
__global__ void __launch_bounds__(DCR_NT) k_dc_rot(DcArgs a, int level, int ob) {
  if (dc_skip(a)) return;
  const int N = a.N;
  const int row = blockIdx.x * DCR_NT + threadIdx.x;
  if (row >= N) return;
  const int node = a.pos2node[(size_t)level * N + row];
  const int s = a.nodes[node].s;
  const int nr = a.rot_cnt[node];
  if (nr == 0) return;
  double* Qo = a.Q[ob];
  int ccol = -1;
  double cval = 0.0;
  for (int q = 0; q < nr; ++q) {
    const int cp = a.rot_pq[2 * (s + q)], cq = a.rot_pq[2 * (s + q) + 1];
    const double c = a.rot_cs[2 * (s + q)], sn = a.rot_cs[2 * (s + q) + 1];
    const double y = Qo[(size_t)cq * N + row];
    double x;
    if (cp == ccol) {
      x = cval;
    } else {
      if (ccol >= 0) Qo[(size_t)ccol * N + row] = cval;  // chain ended: flush
      x = Qo[(size_t)cp * N + row];
    }
    Qo[(size_t)cp * N + row] = fma(c, x, sn * y);
    ccol = cq;
    cval = fma(c, y, -sn * x);
  }
  Qo[(size_t)ccol * N + row] = cval;
}

// ---- root merge, between the secular roots and the eigenvectors: which side is projected ----
// k_select's rule on the final spectrum (roots and deflated values): r = min(#lambda > 0,
// #lambda < 0), positives on ties; the selected roots are a contiguous range since roots ascend.
__global__ void __launch_bounds__(DC_NT) k_dc_topsel(DcArgs a, int root) {
  if (dc_skip(a)) return;
  const int s = a.nodes[root].s, k = a.node_k[root], df = a.node_nd[root];
  __shared__ int cnt[4];
  if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
  __syncthreads();
  int rp = 0, rn = 0, dp = 0, dn = 0;
  for (int j = threadIdx.x; j < k; j += DC_NT) {
    rp += a.lam_r[s + j] > 0.0;
    rn += a.lam_r[s + j] < 0.0;
  }
  for (int q = threadIdx.x; q < df; q += DC_NT) {
    dp += a.dfv[s + q] > 0.0;
    dn += a.dfv[s + q] < 0.0;
  }
  atomicAdd(&cnt[0], rp);
  atomicAdd(&cnt[1], rn);
  atomicAdd(&cnt[2], dp);
  atomicAdd(&cnt[3], dn);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (!a.topsel_on || (a.topsel_full && *a.topsel_full)) {
      a.topsel[0] = k;
      a.topsel[1] = 0;
      a.topsel[2] = -1;
    } else if (cnt[0] + cnt[2] <= cnt[1] + cnt[3]) {  // positives: the last #roots>0 roots
      a.topsel[0] = cnt[0];
      a.topsel[1] = k - cnt[0];
      a.topsel[2] = 0;
    } else {  // negatives: the first #roots<0 roots
      a.topsel[0] = cnt[1];
      a.topsel[1] = 0;
      a.topsel[2] = 1;
    }
  }
}

// ---- merge step 6: deflated eigenpairs (copied columns).  grid (node, column chunk): one warp per
// deflated column computes its rank among the merged spectrum, then copies the column. ----
constexpr int DCF_COLS = DC_NT / 32;  // deflated columns per CTA (one per warp)
__global__ void __launch_bounds__(DC_NT) k_dc_final(DcArgs a, int node0, int ob, int nb, int top) {
  if (dc_skip(a)) return;
  const int node = node0 + blockIdx.x;
  const DcNode nd = a.nodes[node];
  const int N = a.N, s = nd.s, n = nd.n, k = a.node_k[node], df = a.node_nd[node];
  const double* Qo = a.Q[ob];
  double* Qn = a.Q[nb];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.y * DCF_COLS + warp;
  if (q >= df) return;
  const double x = a.dfv[s + q];
  // roots strictly below x, deflated values below x (ties by index)
  int cnt = 0;
  for (int j = lane; j < k; j += 32) cnt += (a.lam_r[s + j] < x) ? 1 : 0;
  for (int q2 = lane; q2 < df; q2 += 32) {
    const double y = a.dfv[s + q2];
    cnt += (y < x || (y == x && q2 < q)) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  const int col = s + cnt;
  if (lane == 0) a.lam[nb][col] = x;
  if (top) {  // root: copy only the selected side's deflated eigenvectors
    const int side = a.topsel[2];
    if ((side == 0 && !(x > 0.0)) || (side == 1 && !(x < 0.0))) return;
  }
  const double* src = Qo + (size_t)a.dfcol[s + q] * N;
  double* dst = Qn + (size_t)col * N;
  for (int r = s + lane; r < s + n; r += 32) dst[r] = src[r];
}
