// PSD-cone projection of large Gram blocks (N > 64).
//
//   a  --(k_tridiag, one cluster)-->  T = H^T a H, reflectors V, tau
//      --(divide and conquer, dc.cuh)-->  T = Z diag(lambda) Z^T
//      --(k_select)-->  the spectral side with fewer eigenpairs: r = min(#lambda>0, #lambda<0)
//      --(k_bt_larft, k_bt_apply: compact-WY blocks on DMMA)-->  W = H Z_side diag(sqrt|lambda_side|)
//                                                              (only r columns)
//      --(k_gemm_f64, DMMA)-->  M = W W^T
// M is Pi_{S+}(a) when the positive side was chosen, and Pi_{S+}(-a) = Pi_{S+}(a) - a (Moreau)
// when the negative side was; k_pack reads the per-block side flag.  Picking the smaller side
// makes the back-transform and the reconstruction O(N^2 r) instead of O(N^3) near convergence,
// where the projected Gram matrices have low rank (SURVEY §7 H1 "partial spectrum").
#pragma once
#include <string>
#include <vector>

#include "common.cuh"
#include "dc.cuh"
#include "gemm_f64.cuh"
#include "tridiag.cuh"
#include "backtransform.cuh"
#include "sy2sb.cuh"
#include "sb2st.cuh"
#include "bt2.cuh"
#include "warm.cuh"

struct LargeBlock {
  int b = 0, N = 0, C = 1, D = 0;
  long long smem_cols = 0;
  size_t trd_smem = 0;
  int ksw = 0;                // first step done by the single-CTA tail (N - 2: no tail)
  size_t tail_smem = 0;
  TridiagArgs ta_tail{};
  double* M = nullptr;
  double *d = nullptr, *e = nullptr, *tau = nullptr, *V = nullptr;
  DcArgs dc{};
  std::vector<int> level_node0, level_nn, level_nmax;
  int leaf0 = 0, nleaves = 0;
  GemmDesc* gdesc = nullptr;  // per level (node-indexed), then the reconstruction descriptor
  std::vector<int> gdesc_off;
  int* sel = nullptr;         // [r, c0, side]
  double* Twy = nullptr;      // compact-WY T factors of the reflector blocks (backtransform.cuh)
  double* Gwy = nullptr;      // their Gram partials per row chunk
  int recon = 0;              // index of the reconstruction descriptor in gdesc
  double* W = nullptr;
  TridiagArgs ta{};
  // two-stage tridiagonalisation (sy2sb.cuh -> sb2st.cuh, back-transform bt2.cuh then the WY blocks)
  bool two = false;
  int BW = 16, KMAX = 1, nref = 0;
  size_t sy_smem = 0, st_smem = 0, bt2_smem_b = 0;
  Sy2sbArgs sa{};
  double *V2 = nullptr, *tau2 = nullptr, *Bg = nullptr;
  unsigned* cnt = nullptr;
  std::vector<int> node_n;  // host copy: size of every D&C node (index = node id), for the work accounting
  int jl = 0;               // levels 1..jl are replaced by the QR solve of their output nodes (k_dc_qrnode)
  // warm-started projection (warm.cuh): refinement of the previous eigenvectors, cold path as fallback
  bool warm = false;
  WarmArgs wa{};
  DgemmDesc* wdesc = nullptr;  // [WM_MAXS][5]: W = Af X, S = X^T W, P = X^T X, X' = X M, W' = W M; then Y = Xs Ss
  int wrecon = 0;              // index of the warm reconstruction descriptor (Y Xs^T) in gdesc
  int* sel_all = nullptr;      // [N, 0, 0]: the cold path back-transforms every column (unscaled) into X0
};

struct LargeEig {
  std::vector<LargeBlock> blocks;
  int* side = nullptr;   // per PSD block: 1 = block matrix holds Pi(-a)
  const DevState* st = nullptr;
  const IterScal* is = nullptr;
  int check_state = 1;
};

// ---------------------------------------------------------------------------------------------
__global__ void k_select(const double* lam, int* sel, int* side, int b, int N, const DevState* st,
                         const IterScal* is, int check_state) {
  if (check_state && (st->done || !is->proceed)) return;
  __shared__ int cp, cn;
  if (threadIdx.x == 0) cp = cn = 0;
  __syncthreads();
  int p = 0, q = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    p += lam[i] > 0.0;
    q += lam[i] < 0.0;
  }
  atomicAdd(&cp, p);
  atomicAdd(&cn, q);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (cp <= cn) {
      sel[0] = cp;
      sel[1] = N - cp;
      sel[2] = 0;
    } else {
      sel[0] = cn;
      sel[1] = 0;
      sel[2] = 1;
    }
    side[b] = sel[2];
  }
}

// ---------------------------------------------------------------------------------------------
struct LargeLayout {
  size_t bytes = 0;
};

inline void dc_build_tree(int N, std::vector<DcNode>& nodes, std::vector<int>& level_node0,
                          std::vector<int>& level_nn, std::vector<int>& level_nmax, int& D, int& leaf0,
                          int& nleaves, std::vector<int>& pos2node) {
  D = 0;
  while ((1 << (D + 1)) <= N) ++D;  // 2^D <= N < 2^(D+1): leaves of size 1 or 2
  // nodes per depth (depth 0 = root), recursive bisection
  std::vector<std::vector<DcNode>> by_depth(D + 1);
  by_depth[0].push_back(DcNode{0, N / 2, N, 0});
  for (int dep = 0; dep < D; ++dep)
    for (const DcNode& nd : by_depth[dep]) {
      const int n1 = nd.n / 2, n2 = nd.n - n1;
      by_depth[dep + 1].push_back(DcNode{nd.s, n1 / 2, n1, 0});
      by_depth[dep + 1].push_back(DcNode{nd.s + n1, n2 / 2, n2, 0});
    }
  // fix the split of every internal node: n1 = size of its left child
  for (int dep = 0; dep < D; ++dep)
    for (size_t q = 0; q < by_depth[dep].size(); ++q) by_depth[dep][q].n1 = by_depth[dep + 1][2 * q].n;
  // levels bottom-up: level h (1..D) merges depth D-h; leaves are depth D
  nodes.clear();
  level_node0.assign(D + 1, 0);
  level_nn.assign(D + 1, 0);
  level_nmax.assign(D + 1, 0);
  pos2node.assign((size_t)(D + 1) * N, 0);
  leaf0 = 0;
  nleaves = (int)by_depth[D].size();
  for (const DcNode& nd : by_depth[D]) nodes.push_back(nd);
  for (int h = 1; h <= D; ++h) {
    level_node0[h] = (int)nodes.size();
    long long uoff = 0;
    for (DcNode nd : by_depth[D - h]) {
      nd.u_off = uoff;
      uoff += (long long)nd.n * nd.n;
      const int id = (int)nodes.size();
      for (int p = nd.s; p < nd.s + nd.n; ++p) pos2node[(size_t)h * N + p] = id;
      level_nmax[h] = std::max(level_nmax[h], nd.n);
      nodes.push_back(nd);
    }
    level_nn[h] = (int)nodes.size() - level_node0[h];
  }
}

constexpr int TRD_MAX_DYN_SMEM = 227 * 1024 - 2048;  // leaves room for the static tables
constexpr int DYN_SMEM_MAX = 232448;                  // sm_100a opt-in maximum per block

// Two-stage sizes: band half-width (the stage-2 band of 2 BW diagonals must fit one SM: BW = 16 up to
// N = 880, BW = 8 above), workers (8-row blocks, at most 147 so the grid fits 148 SMs at one CTA each).
inline int ts_bw(int N) { return sb2st_smem(N, 16) <= (size_t)DYN_SMEM_MAX ? 16 : 8; }
inline int ts_workers(int N) { return std::min(147, (N + SB_R - 1) / SB_R); }
inline int ts_maxrb(int N) {
  const int nrb = (N + SB_R - 1) / SB_R, nw = ts_workers(N);
  return (nrb + nw - 1) / nw;
}
// Default: the one-cluster kernel k_tridiag.  The two-stage reduction (sy2sb -> sb2st -> bt2) is selected
// with SOSADMM_TRIDIAG=twostage: it is correct and tested (tests/test_gpu_stages.py) but measured slower on
// B200 at every config size (N = 861: stage 1 2.8 ms + stage 2 4.4 ms vs 4.5 ms; DESIGN.md §5 has the
// per-phase profile and why: stage 2 is issue / shared-memory bound on one SM with a 2N-task critical
// path, stage 1 pays three global hand-offs per 16-column panel).
inline bool ts_enabled() {
  const char* env = getenv("SOSADMM_TRIDIAG");
  return env && std::string(env) == "twostage";
}

// Cluster size: 16 CTAs (the non-portable maximum) from N = 161 on — measured faster than 8 at
// N = 231 (0.62 -> 0.56 ms) and N = 325 (1.07 -> 0.93 ms): the per-step fixed cost barely depends on
// C while the fused pass shrinks with it.
inline int tridiag_cluster_size(int N) { return N > 160 ? 16 : 4; }

// Row storage (doubles) of CTA c of C for rows i >= kb stored from column kb.
inline long long tridiag_rows_need(int N, int C, int c, int kb) {
  long long s = 0;
  for (int i = c; i < N; i += C)
    if (i >= kb) s += i + 1 - kb;
  return s;
}
// Shared-memory budget (doubles) for the row storage of the cluster head (per CTA, rows from 0).
inline long long tridiag_row_budget(int N, int C) {
  const long long cap = TRD_MAX_DYN_SMEM / 8 - trd_fixed_doubles(N, C, (N + C - 1) / C);
  long long need = 0;
  for (int c = 0; c < C; ++c)  // + 15 doubles of bank-alignment padding per row (k_tridiag)
    need = std::max(need, tridiag_rows_need(N, C, c, 0) + 15LL * ((N - c + C - 1) / C));
  return std::min(cap, need);
}
// Number of trailing rows n the single-CTA tail takes over (the whole lower triangle of the last n
// rows in one SM's shared memory); 0 = no tail.  Capped at TRD_TAIL_MAX: below it the per-step fixed
// cost of the cluster exchanges (~5k cycles) exceeds one SM's share of the trailing work.
constexpr int TRD_TAIL_MAX = 0;  // disabled: measured slower than the cluster (profiles/r01_*)
inline int tridiag_tail_rows(int N) {
  int n = 0;
  for (int t = 16; t <= std::min(N - 3, TRD_TAIL_MAX); ++t) {
    const long long need = trd_fixed_doubles(N, 1, t) + (long long)t * (t + 1) / 2;
    if (need > TRD_MAX_DYN_SMEM / 8) break;
    n = t;
  }
  return n;
}

template <class F>
inline size_t large_carve(const std::vector<int>& blk_N, const std::vector<int>& large, char* base, int** side,
                          F&& per_block) {
  size_t used = 0;
  auto take = [&](size_t bytes) -> char* {
    used = (used + 255) / 256 * 256;
    char* p = base ? base + used : nullptr;
    used += std::max<size_t>(bytes, 8);
    return p;
  };
  char* sp = take(4 * std::max<size_t>(blk_N.size(), 1));  // per-block side flags
  if (side) *side = (int*)sp;
  for (int b : large) {
    const int N = blk_N[b];
    std::vector<DcNode> nodes;
    std::vector<int> l0, lnn, lmax, p2n;
    int D, leaf0, nleaves;
    dc_build_tree(N, nodes, l0, lnn, lmax, D, leaf0, nleaves, p2n);
    const size_t NN = (size_t)N * N;
    char* p[96];  // (74 buffers per block)
    int q = 0;
    p[q++] = take(8 * N);                 // d
    p[q++] = take(8 * N);                 // e
    p[q++] = take(8 * N);                 // tau
    p[q++] = take(8 * NN);                // V
    p[q++] = take(8 * NN);                // Q0
    p[q++] = take(8 * NN);                // Q1
    p[q++] = take(8 * N);                 // lam0
    p[q++] = take(8 * N);                 // lam1
    p[q++] = take(sizeof(DcNode) * nodes.size());
    p[q++] = take(4 * p2n.size());
    for (int t = 0; t < 6; ++t) p[q++] = take(8 * N);   // ndd ndz dfv tau_r zhat lam_r
    for (int t = 0; t < 4; ++t) p[q++] = take(4 * N);   // ndcol dfcol org outcol
    p[q++] = take(4 * nodes.size());      // node_k
    p[q++] = take(4 * nodes.size());      // node_nd
    p[q++] = take(8 * nodes.size());      // node_rho
    p[q++] = take(8 * NN);                // U
    p[q++] = take(8 * N);                 // rot_pq (2 ints)
    p[q++] = take(16 * N);                // rot_cs
    p[q++] = take(4 * nodes.size());      // rot_cnt
    p[q++] = take(sizeof(GemmDesc) * (nodes.size() + 2));
    p[q++] = take(4 * 8);                 // sel [r, c0, side] + the D&C root selection (topsel)
    p[q++] = take(8 * ((size_t)3 * N + 2));  // tridiagonalisation hand-over state
    p[q++] = take(8 * (size_t)BTW_NB * BTW_NB * ((N - 2 + BTW_NB - 1) / BTW_NB));  // Twy
    p[q++] = take(8 * (size_t)BTW_NB * BTW_NB * ((N - 2 + BTW_NB - 1) / BTW_NB) * bt_gram_chunks(N));  // Gwy
    {  // two-stage buffers
      const int BW = ts_bw(N), ldv = sy2sb_ldv(N), KM = sb2st_kmax(N, BW);
      p[q++] = take(8 * (size_t)N * 2 * BW);            // Bg (band)
      p[q++] = take(8 * (size_t)BW * N);                // Pg (panel slice, row-major)
      p[q++] = take(8 * (size_t)2 * BW * ldv);          // Vg
      p[q++] = take(8 * (size_t)2 * BW * ldv);          // Yg
      p[q++] = take(8 * (size_t)3 * BW * BW);           // Tg (2), Sg
      p[q++] = take(8 * (size_t)ts_workers(N) * BW * BW);  // Pt
      p[q++] = take(64);                                // counters
      p[q++] = take(8 * (size_t)N * KM * BW);           // V2
      p[q++] = take(8 * (size_t)N * KM);                // tau2
    }
    {  // warm-start buffers (warm.cuh), pitch ldn = N rounded up to even
      const size_t NL = (size_t)N * ((N + 1) & ~1);
      const int nt = (N + 31) / 32;
      for (int t = 0; t < 14; ++t) p[q++] = take(8 * NL);  // Af X0 X1 W W1 S P E Mm Y Srot Rrot Esum Eprev
      p[q++] = take(8 * N);                                // lam
      p[q++] = take(8 * N);                                // lamt
      for (int t = 0; t < 9; ++t) p[q++] = take(4 * (size_t)(N + 1));  // order pos diff cid cpos cl_start cl_size cl_voff cl_rbase
      p[q++] = take(4 * 4);                                // sel
      p[q++] = take(4 * (size_t)N);                        // idx
      p[q++] = take(8 * (size_t)WM_CAP * N);               // Vcl
      p[q++] = take(8 * (size_t)nt * nt);                  // partA
      p[q++] = take(8 * (size_t)nt * nt);                  // cross
      p[q++] = take(8 * 3 * (size_t)nt * nt);              // roff (three sign classes)
      p[q++] = take(8 * (size_t)nt * N);                   // grow
      p[q++] = take(8 * (size_t)nt * N);                   // gcol
      p[q++] = take(8 * 5 * (size_t)nt);                   // rdpart (defect, two weighted defects, two sign counts)
      p[q++] = take(8 * (size_t)nt);                       // g2part
      p[q++] = take(4 * (size_t)(nt + 2));                 // cnt
      p[q++] = take(8 * (size_t)WM_PAIRS);                 // pairs
      p[q++] = take(sizeof(WarmState));                    // ws
      p[q++] = take(sizeof(DgemmDesc) * (WM_MAXS * 5 + 2));  // wdesc
      p[q++] = take(4 * 4);                                // sel_all
    }
    per_block(b, N, p, nodes, l0, lnn, lmax, D, leaf0, nleaves, p2n);
  }
  return used + 256;
}

inline size_t large_eig_bytes(const std::vector<int>& blk_N, const std::vector<int>& large) {
  return large_carve(blk_N, large, nullptr, nullptr, [](int, int, char**, auto&, auto&, auto&, auto&, int, int, int, auto&) {});
}

// Warm-started projection (warm.cuh) on by default for the contexts of sosadmm_setup; SOSADMM_WARM=0 keeps
// the cold path every iteration (for A/B measurements).  Not combined with the opt-in two-stage reduction.
inline bool warm_enabled() {
  const char* e = getenv("SOSADMM_WARM");
  return !(e && e[0] == '0') && !ts_enabled();
}

inline int large_eig_init(LargeEig& le, const std::vector<int>& blk_N, const std::vector<long long>& blk_mat,
                          const std::vector<int>& large, double* mats, char* base, DevState* st, IterScal* is,
                          cudaStream_t s, std::string& msg, bool warm = false) {
  le.st = st;
  le.is = is;
  le.blocks.clear();
  cudaError_t err = cudaSuccess;
  int* side_p = nullptr;
  large_carve(blk_N, large, base, &side_p, [&](int b, int N, char** p, std::vector<DcNode>& nodes,
                                                   std::vector<int>& l0, std::vector<int>& lnn,
                                                   std::vector<int>& lmax, int D, int leaf0, int nleaves,
                                                   std::vector<int>& p2n) {
    LargeBlock lb;
    lb.b = b;
    lb.N = N;
    lb.M = mats + blk_mat[b];
    lb.C = tridiag_cluster_size(N);
    lb.smem_cols = tridiag_row_budget(N, lb.C);
    lb.trd_smem = tridiag_smem_bytes(N, lb.C, (N + lb.C - 1) / lb.C, lb.smem_cols);
    {
      const int nt = tridiag_tail_rows(N);
      lb.ksw = (nt >= 16 && N - nt > 8) ? N - nt : N - 2;
      const int S = N - lb.ksw;
      lb.tail_smem = tridiag_smem_bytes(N, 1, S, tridiag_rows_need(N, 1, 0, lb.ksw) + 15LL * S);
    }
    int q = 0;
    lb.d = (double*)p[q++];
    lb.e = (double*)p[q++];
    lb.tau = (double*)p[q++];
    lb.V = (double*)p[q++];
    DcArgs& dc = lb.dc;
    dc.N = N;
    dc.d = lb.d;
    dc.e = lb.e;
    dc.dmod = nullptr;
    dc.Q[0] = (double*)p[q++];
    dc.Q[1] = (double*)p[q++];
    dc.lam[0] = (double*)p[q++];
    dc.lam[1] = (double*)p[q++];
    DcNode* dnodes = (DcNode*)p[q++];
    int* dp2n = (int*)p[q++];
    dc.nodes = dnodes;
    dc.pos2node = dp2n;
    dc.ndd = (double*)p[q++];
    dc.ndz = (double*)p[q++];
    dc.dfv = (double*)p[q++];
    dc.tau_r = (double*)p[q++];
    dc.zhat = (double*)p[q++];
    dc.lam_r = (double*)p[q++];
    dc.ndcol = (int*)p[q++];
    dc.dfcol = (int*)p[q++];
    dc.org = (int*)p[q++];
    dc.outcol = (int*)p[q++];
    dc.node_k = (int*)p[q++];
    dc.node_nd = (int*)p[q++];
    dc.node_rho = (double*)p[q++];
    dc.U = (double*)p[q++];
    dc.rot_pq = (int*)p[q++];
    dc.rot_cs = (double*)p[q++];
    dc.rot_cnt = (int*)p[q++];
    dc.st = st;
    dc.is = is;
    dc.check_state = 1;
    lb.gdesc = (GemmDesc*)p[q++];
    lb.sel = (int*)p[q++];
    dc.topsel = lb.sel + 4;
    dc.topsel_on = 1;  // the warm mode's cold path keeps every eigenvector only when it re-seeds X (topsel_full)
    dc.topsel_full = nullptr;
    lb.warm = warm;
    double* hand = (double*)p[q++];
    lb.Twy = (double*)p[q++];
    lb.Gwy = (double*)p[q++];
    lb.recon = (int)nodes.size();
    lb.node_n.clear();
    for (const DcNode& nd : nodes) lb.node_n.push_back(nd.n);
    lb.D = D;
    lb.jl = 0;
    for (int h = 1; h < D; ++h)
      if (lmax[h] <= DCJ_MAXN) lb.jl = h;
    lb.level_node0 = l0;
    lb.level_nn = lnn;
    lb.level_nmax = lmax;
    lb.leaf0 = leaf0;
    lb.nleaves = nleaves;
    // GEMM descriptors: one per merge node (Q_new = Q_old[:, nd] U), then the reconstruction
    std::vector<GemmDesc> gd(nodes.size() + 2);
    for (int h = 1; h <= D; ++h) {
      const int ob = (h - 1) & 1, nb = h & 1;
      for (int t = 0; t < lnn[h]; ++t) {
        const int id = l0[h] + t;
        const DcNode& nd = nodes[id];
        GemmDesc g{};
        g.A = dc.Q[ob] + nd.s;
        g.lda = N;
        g.acol = dc.ndcol + nd.s;
        g.B = dc.U + nd.u_off;
        g.ldb = nd.n;
        g.C = dc.Q[nb] + nd.s;
        g.ldc = N;
        g.ccol = dc.outcol + nd.s;
        g.M = nd.n;
        g.N = nd.n;
        g.K = nd.n;
        g.Kdev = dc.node_k + id;
        g.Ndev = dc.node_k + id;
        if (h == D) {  // root: only the selected eigenvector columns (k_dc_topsel)
          g.Ndev = dc.topsel;
          g.Noff = dc.topsel + 1;
        }
        g.alpha = 1.0;
        g.beta = 0.0;
        gd[id] = g;
      }
    }
    const int fb = D & 1;  // buffer holding the final eigenpairs
    lb.W = dc.Q[1 - fb];
    {
      GemmDesc g{};
      g.A = lb.W;
      g.lda = N;
      g.B = lb.W;
      g.ldb = N;
      g.transB = 1;
      g.C = lb.M;
      g.ldc = N;
      g.M = N;
      g.N = N;
      g.K = N;
      g.Kdev = lb.sel;
      g.alpha = 1.0;
      g.beta = 0.0;
      g.upper = 1;  // k_pack reads the upper triangle of the projection only
      gd[nodes.size()] = g;
    }
    lb.wrecon = (int)nodes.size() + 1;  // filled below (warm buffers are carved after the two-stage ones)
    if (err == cudaSuccess) err = cudaMemcpyAsync(dnodes, nodes.data(), sizeof(DcNode) * nodes.size(), cudaMemcpyHostToDevice, s);
    if (err == cudaSuccess) err = cudaMemcpyAsync(dp2n, p2n.data(), 4 * p2n.size(), cudaMemcpyHostToDevice, s);
    if (err == cudaSuccess) err = cudaMemcpyAsync(lb.gdesc, gd.data(), sizeof(GemmDesc) * gd.size(), cudaMemcpyHostToDevice, s);
    // tridiagonalisation arguments
    TridiagArgs& ta = lb.ta;
    ta.M = lb.M;
    ta.N = N;
    ta.C = lb.C;
    ta.smem_rows_doubles = lb.smem_cols;
    ta.d = lb.d;
    ta.e = lb.e;
    ta.tau = lb.tau;
    ta.V = lb.V;
    ta.st = st;
    ta.is = is;
    ta.check_state = 1;
    ta.prof = nullptr;
    ta.kb = 0;
    ta.ke = lb.ksw;
    ta.hand = hand;
    lb.ta_tail = ta;
    lb.ta_tail.C = 1;
    lb.ta_tail.kb = lb.ksw;
    lb.ta_tail.ke = N - 2;
    lb.ta_tail.smem_rows_doubles = tridiag_rows_need(N, 1, 0, lb.ksw) + 15LL * (N - lb.ksw);
    lb.nref = N - 2;
    lb.two = ts_enabled();
    {
      const int BW = ts_bw(N), ldv = sy2sb_ldv(N);
      lb.BW = BW;
      lb.KMAX = sb2st_kmax(N, BW);
      Sy2sbArgs& sa = lb.sa;
      sa.M = lb.M;
      sa.N = N;
      sa.BW = BW;
      sa.NW = ts_workers(N);
      sa.maxrb = ts_maxrb(N);
      sa.ldr = sy2sb_ldr(N);
      sa.P = sy2sb_panels(N, BW);
      sa.Bg = (double*)p[q++];
      sa.V1 = lb.V;
      sa.tau1 = lb.tau;
      sa.Pg = (double*)p[q++];
      sa.Vg = (double*)p[q++];
      sa.Yg = (double*)p[q++];
      sa.ldv = ldv;
      sa.Tg = (double*)p[q++];
      sa.Sg = sa.Tg + 2 * BW * BW;
      sa.Pt = (double*)p[q++];
      sa.cnt = (unsigned*)p[q++];
      sa.st = st;
      sa.is = is;
      sa.check_state = 1;
      lb.Bg = sa.Bg;
      lb.cnt = sa.cnt;
      lb.V2 = (double*)p[q++];
      lb.tau2 = (double*)p[q++];
      lb.sy_smem = std::max(sy2sb_worker_smem(N, BW, sa.maxrb), sy2sb_panel_smem(N, BW));
      lb.st_smem = sb2st_smem(N, BW);
      lb.bt2_smem_b = bt2_smem(N, BW, lb.KMAX);
      if (lb.two) lb.nref = sa.P * BW;
      if (lb.two && (lb.sy_smem > (size_t)DYN_SMEM_MAX || lb.st_smem > (size_t)DYN_SMEM_MAX || sa.maxrb > 4))
        lb.two = false;  // outside the two-stage envelope (N > 1280): one-stage kernel
    }
    {  // warm-start state and descriptors
      const int ldn = (N + 1) & ~1, nt = (N + 31) / 32;
      WarmArgs& wa = lb.wa;
      wa.N = N;
      wa.ldn = ldn;
      wa.nt = nt;
      wa.Mblk = lb.M;
      double** big[14] = {&wa.Af, &wa.X0, &wa.X1, &wa.W, &wa.W1, &wa.S, &wa.P, &wa.E, &wa.Mm, &wa.Y, &wa.Srot, &wa.Rrot,
                          &wa.Esum, &wa.Eprev};
      for (int t = 0; t < 14; ++t) *big[t] = (double*)p[q++];
      {
        const char* e = getenv("SOSADMM_WARM_PRED");
        wa.predict = (e && e[0] == '0') ? 0 : ((e && e[0] == '2') ? 2 : 1);
      }
      {
        const char* e = getenv("SOSADMM_WARM_BACKOFF");
        wa.bo_cap = e ? std::max(1, std::min(6, atoi(e))) : 3;
      }
      {
        const char* e = getenv("SOSADMM_WARM_WTEST");
        wa.wtest = (e && e[0] == '0') ? 0 : 1;
      }
      wa.lam = (double*)p[q++];
      wa.lamt = (double*)p[q++];
      int** ib[9] = {&wa.order, &wa.pos, &wa.diff, &wa.cid, &wa.cpos, &wa.cl_start, &wa.cl_size, &wa.cl_voff,
                     &wa.cl_rbase};
      for (int t = 0; t < 9; ++t) *ib[t] = (int*)p[q++];
      wa.sel = (int*)p[q++];
      wa.idx = (int*)p[q++];
      wa.Vcl = (double*)p[q++];
      wa.partA = (double*)p[q++];
      wa.cross = (double*)p[q++];
      wa.roff = (double*)p[q++];
      wa.grow = (double*)p[q++];
      wa.gcol = (double*)p[q++];
      wa.rdpart = (double*)p[q++];
      wa.g2part = (double*)p[q++];
      wa.cnt = (int*)p[q++];
      wa.pairs = (int*)p[q++];
      wa.ws = (WarmState*)p[q++];
      lb.wdesc = (DgemmDesc*)p[q++];
      lb.sel_all = (int*)p[q++];
      wa.lam_cold = dc.lam[D & 1];
      if (warm) lb.dc.topsel_full = &wa.ws->need_full;
      wa.side = nullptr;  // le.side, set after the carve
      wa.st = st;
      wa.is = is;
      // step j works on X_j = X[j & 1] and W_j = a X_j = W[j & 1]: step 0 forms W_0 = a X_0 and P_0 (unless
      // the previous iteration's certified P of the same X survives, ws->pgate = 0); every update forms
      // X_{j+1} = X_j M and W_{j+1} = W_j M in ONE batched launch (same M), so later steps skip a X.
      std::vector<DgemmDesc> wd(WM_MAXS * 5 + 2);
      for (int j = 0; j < WM_MAXS; ++j) {
        double* Xc = (j & 1) ? wa.X1 : wa.X0;
        double* Xn = (j & 1) ? wa.X0 : wa.X1;
        double* Wc = (j & 1) ? wa.W1 : wa.W;
        double* Wn = (j & 1) ? wa.W : wa.W1;
        DgemmDesc g{};
        g.M = N; g.N = N; g.K = N; g.lda = ldn; g.ldb = ldn; g.ldc = ldn; g.alpha = 1.0; g.beta = 0.0;
        g.gate = &wa.ws->gate;
        DgemmDesc gw = g;  // W_0 = Af X_0 (step 0 only)
        gw.A = wa.Af; gw.B = Xc; gw.C = Wc;
        DgemmDesc gs = g;  // S = X^T W (upper)
        gs.A = Xc; gs.transA = 1; gs.B = Wc; gs.C = wa.S; gs.upper = 1; gs.mirror = 1;
        DgemmDesc gp = gs;  // P = X^T X (upper)
        gp.B = Xc; gp.C = wa.P;
        if (j == 0) gp.gate = &wa.ws->pgate;
        DgemmDesc gx = g;  // X' = X M
        gx.A = Xc; gx.B = wa.Mm; gx.C = Xn;
        DgemmDesc gv = g;  // W' = W M
        gv.A = Wc; gv.B = wa.Mm; gv.C = Wn;
        wd[5 * j] = gw;
        wd[5 * j + 1] = gs;
        wd[5 * j + 2] = gp;
        wd[5 * j + 3] = gx;
        wd[5 * j + 4] = gv;
      }
      {  // finish: Y = Xs Ss (Xs in Mm, Ss in E, Y in Y; r x r from sel)
        DgemmDesc g{};
        g.A = wa.Mm; g.lda = ldn; g.B = wa.E; g.ldb = ldn; g.C = wa.Y; g.ldc = ldn;
        g.M = N; g.N = N; g.K = N; g.Ndev = wa.sel; g.Kdev = wa.sel; g.alpha = 1.0; g.beta = 0.0;
        wd[WM_MAXS * 5] = g;
      }
      {  // predictor: X1 = X0 (I + Esum), gated on ws->pred
        DgemmDesc g{};
        g.A = wa.X0; g.lda = ldn; g.B = wa.Mm; g.ldb = ldn; g.C = wa.X1; g.ldc = ldn;
        g.M = N; g.N = N; g.K = N; g.alpha = 1.0; g.beta = 0.0; g.gate = &wa.ws->pred;
        wd[WM_MAXS * 5 + 1] = g;
      }
      {  // warm reconstruction M = Y Xs^T (upper tiles) into the block matrix
        GemmDesc g{};
        g.A = wa.Y; g.lda = ldn; g.B = wa.Mm; g.ldb = ldn; g.transB = 1; g.C = lb.M; g.ldc = N;
        g.M = N; g.N = N; g.K = N; g.Kdev = wa.sel; g.alpha = 1.0; g.beta = 0.0; g.upper = 1;
        if (err == cudaSuccess) err = cudaMemcpyAsync(lb.gdesc + lb.wrecon, &g, sizeof(g), cudaMemcpyHostToDevice, s);
      }
      const int sa3[4] = {N, 0, 0, 0};
      if (err == cudaSuccess) err = cudaMemcpyAsync(lb.wdesc, wd.data(), sizeof(DgemmDesc) * wd.size(), cudaMemcpyHostToDevice, s);
      if (err == cudaSuccess) err = cudaMemcpyAsync(lb.sel_all, sa3, sizeof(sa3), cudaMemcpyHostToDevice, s);
      if (err == cudaSuccess) err = cudaMemsetAsync(wa.ws, 0, sizeof(WarmState), s);
      if (err == cudaSuccess) err = cudaMemsetAsync(wa.X1, 0, 8 * (size_t)N * ldn, s);
      if (err == cudaSuccess) err = cudaMemsetAsync(wa.X0, 0, 8 * (size_t)N * ldn, s);
    }
    le.blocks.push_back(lb);
  });
  le.side = side_p;
  for (auto& lb : le.blocks) lb.wa.side = side_p;
  if (err != cudaSuccess) {
    msg = cudaGetErrorString(err);
    return 1;
  }
  if (le.side) {
    err = cudaMemsetAsync(le.side, 0, 4 * std::max<size_t>(blk_N.size(), 1), s);
    if (err != cudaSuccess) {
      msg = cudaGetErrorString(err);
      return 1;
    }
  }
  if (!le.blocks.empty()) {
#define TRD_PTR(MB, CCX) k_tridiag<MB, CCX>,
    for (TridiagKernel kt : {TRD_KERNELS(TRD_PTR)}) {
#undef TRD_PTR
      if (err == cudaSuccess) err = cudaFuncSetAttribute(kt, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (err == cudaSuccess)
        err = cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, TRD_MAX_DYN_SMEM);
    }
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(k_bt_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)bt_apply_smem_bytes(DC_MAXN));
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(k_warm_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WM_CL_SMEM);
    if (err == cudaSuccess) dgemm_prepare();
    for (int bw : {8, 16}) {
      if (err == cudaSuccess)
        err = cudaFuncSetAttribute(sy2sb_kernel(bw), cudaFuncAttributeMaxDynamicSharedMemorySize, DYN_SMEM_MAX);
      if (err == cudaSuccess)
        err = cudaFuncSetAttribute(sb2st_kernel(bw), cudaFuncAttributeMaxDynamicSharedMemorySize, DYN_SMEM_MAX);
      if (err == cudaSuccess)
        err = cudaFuncSetAttribute(bt2_kernel(bw), cudaFuncAttributeMaxDynamicSharedMemorySize, DYN_SMEM_MAX);
    }
    if (err != cudaSuccess) {
      msg = std::string("k_tridiag attributes: ") + cudaGetErrorString(err);
      return 1;
    }
  }
  return 0;
}

// Two-stage reduction: stage 1 (dense -> band) as one cooperative persistent grid, stage 2 (band ->
// tridiagonal) on one SM.  The hand-off counters are zeroed in the same stream first.
inline void large_block_tridiag2(LargeEig& le, LargeBlock& lb, cudaStream_t s, bool check) {
  (void)le;
  lb.sa.check_state = check;
  cudaMemsetAsync(lb.cnt, 0, 16, s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(lb.sa.NW + 1, 1, 1);
  cfg.blockDim = dim3(SB_NT, 1, 1);
  cfg.dynamicSmemBytes = lb.sy_smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, sy2sb_kernel(lb.BW), lb.sa);
  sb2st_kernel(lb.BW)<<<1, ST_NT, lb.st_smem, s>>>(lb.Bg, lb.N, lb.d, lb.e, lb.V2, lb.tau2, le.st, le.is, check,
                                                    nullptr);
}

inline void large_block_tridiag(LargeEig& le, LargeBlock& lb, cudaStream_t s, bool check) {
  if (lb.two) {
    large_block_tridiag2(le, lb, s, check);
    return;
  }
  lb.ta.check_state = check;
  lb.ta_tail.check_state = check;
  lb.ta_tail.prof = lb.ta.prof;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(lb.C, 1, 1);
    cfg.blockDim = dim3(TRD_NT, 1, 1);
    cfg.dynamicSmemBytes = lb.trd_smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = lb.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, tridiag_kernel_mc(tridiag_maxb(lb.N), lb.C), lb.ta);
  }
  if (lb.ksw < lb.N - 2)
    tridiag_kernel_mc(tridiag_maxb(lb.N), 1)<<<1, TRD_NT, lb.tail_smem, s>>>(lb.ta_tail);
}

// side, ev (5 events): optional second stream — the deflation rotations and the deflated copies of
// each merge then run beside the secular / eigenvector / GEMM chain (5 dependent launches per level
// instead of 7): rot needs prep, final needs rot, secular (and the root selection); the GEMM needs
// rot; the next level needs final.
inline void large_block_dc(LargeEig& le, LargeBlock& lb, cudaStream_t s, bool check, cudaStream_t side = nullptr,
                           const cudaEvent_t* ev = nullptr) {
  const int N = lb.N;
  lb.dc.check_state = check;
  if (side) {  // the eigenvector buffers were zeroed on `side` beside the tridiagonalisation (ev[4])
    cudaStreamWaitEvent(s, ev[4], 0);
  } else {
    cudaMemsetAsync(lb.dc.Q[0], 0, sizeof(double) * N * N, s);
    cudaMemsetAsync(lb.dc.Q[1], 0, sizeof(double) * N * N, s);
  }
  if (lb.jl > 0)  // the bottom subtrees in one launch: their root nodes' eigenpairs by Jacobi
    k_dc_qrnode<<<lb.level_nn[lb.jl], DCJ_NT, 0, s>>>(lb.dc, lb.level_node0[lb.jl], lb.jl & 1);
  else
    k_dc_leaf<<<(lb.nleaves + 127) / 128, 128, 0, s>>>(lb.dc, lb.leaf0, lb.nleaves, 0);
  const int wblocks = (N * 32 + DC_NT - 1) / DC_NT;
  for (int h = lb.jl + 1; h <= lb.D; ++h) {
    const int ob = (h - 1) & 1, nb = h & 1;
    const int n0 = lb.level_node0[h], nn = lb.level_nn[h], nmax = lb.level_nmax[h];
    const bool two = side != nullptr;
    cudaStream_t s2 = two ? side : s;
    k_dc_prep<<<nn, DC_NT, 0, s>>>(lb.dc, n0, ob);
    if (two) {
      cudaEventRecord(ev[0], s);
      cudaStreamWaitEvent(s2, ev[0], 0);
    }
    k_dc_rot<<<(N + DCR_NT - 1) / DCR_NT, DCR_NT, 0, s2>>>(lb.dc, h, ob);
    if (two) cudaEventRecord(ev[1], s2);
    k_dc_secular<<<wblocks, DC_NT, 0, s>>>(lb.dc, h);
    if (h == lb.D) k_dc_topsel<<<1, DC_NT, 0, s>>>(lb.dc, n0);  // root: which eigenvectors to form
    if (two) {
      cudaEventRecord(ev[2], s);
      cudaStreamWaitEvent(s2, ev[2], 0);
    }
    k_dc_final<<<dim3(nn, (nmax + DCF_COLS - 1) / DCF_COLS), DC_NT, 0, s2>>>(lb.dc, n0, ob, nb, h == lb.D ? 1 : 0);
    if (two) cudaEventRecord(ev[3], s2);
    k_dc_zhat<<<wblocks, DC_NT, 0, s>>>(lb.dc, h);
    k_dc_vec<<<wblocks, DC_NT, 0, s>>>(lb.dc, h, nb, h == lb.D ? 1 : 0);
    if (two) cudaStreamWaitEvent(s, ev[1], 0);  // the GEMM reads the rotated columns
    dim3 gg((nmax + GM_BM - 1) / GM_BM, (nmax + GM_BN - 1) / GM_BN, nn);
    k_gemm_f64<<<gg, GM_NT, 0, s>>>(lb.gdesc + n0, le.st, le.is, check);
    if (two) cudaStreamWaitEvent(s, ev[3], 0);  // next level reads the deflated copies
  }
}

// compact-WY T factors of the reflector blocks (depend on the tridiagonalisation only)
inline void large_block_wy(LargeEig& le, LargeBlock& lb, cudaStream_t s, bool check) {
  const int N = lb.N, nref = lb.nref;
  const int nbw = (nref + BTW_NB - 1) / BTW_NB;
  k_bt_gram<<<dim3(nbw, bt_gram_chunks(N)), BTW_NT, 0, s>>>(lb.V, lb.Gwy, N, nref, le.st, le.is, check);
  k_bt_larft<<<nbw, BTW_NT, 0, s>>>(lb.Gwy, bt_gram_chunks(N), lb.tau, lb.Twy, nref, le.st, le.is, check);
}

inline void large_block_recon(LargeEig& le, LargeBlock& lb, cudaStream_t s, bool check, bool with_wy = true) {
  const int N = lb.N;
  const int fb = lb.D & 1;
  const int nref = lb.nref;
  k_select<<<1, 256, 0, s>>>(lb.dc.lam[fb], lb.sel, le.side, lb.b, N, le.st, le.is, check);
  if (with_wy) large_block_wy(le, lb, s, check);
  if (lb.two)  // Z_r <- Q2 Z_r (stage-2 reflectors), in place on the selected columns
    bt2_kernel(lb.BW)<<<(N / 2 + BT2_NC) / BT2_NC, BT2_NT, lb.bt2_smem_b, s>>>(
        lb.dc.Q[fb], lb.sel, lb.V2, lb.tau2, N, lb.KMAX, le.st, le.is, check);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(BTC_P * ((N / 2 + BTW_NC - 1) / BTW_NC), 1, 1);
    cfg.blockDim = dim3(BTC_NT, 1, 1);
    cfg.dynamicSmemBytes = bt_apply_smem_bytes(N);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = BTC_P;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_bt_apply, (const double*)lb.dc.Q[fb], (const double*)lb.dc.lam[fb],
                       (const double*)lb.V, (const double*)lb.Twy, (const int*)lb.sel, lb.W, N, nref, le.st,
                       le.is, (int)check, N, 1);
  }
  dim3 gr((N + GM_BM - 1) / GM_BM, (N + GM_BN - 1) / GM_BN, 1);
  k_gemm_f64<<<gr, GM_NT, 0, s>>>(lb.gdesc + lb.recon, le.st, le.is, check);
}

// ---- warm mode (warm.cuh) ----------------------------------------------------------------------
__global__ void k_zero2(double* a, double* b, long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    a[e] = 0.0;
    b[e] = 0.0;
  }
}
// the predictor X1 = X0 (I + G): reads only what the previous iteration left (X0, Esum, the warm state), so
// in the CUDA graph it runs on a branch beside the affine projection (launch_iteration) instead of after it
inline void large_block_warm_pred(LargeEig& le, LargeBlock& lb, cudaStream_t s) {
  k_warm_pred<<<dim3(lb.wa.nt, lb.wa.nt), 256, 0, s>>>(lb.wa);
  dgemm_launch(DG_DEFAULT, lb.wdesc + 5 * WM_MAXS + 1, 1, lb.N, lb.N, s, le.st, le.is, 1);
}
// pred_done: the predictor already ran on another branch; s joins it here
inline void large_block_warm_begin(LargeEig& le, LargeBlock& lb, cudaStream_t s, const WarmArgs& wa,
                                   cudaEvent_t pred_done = nullptr) {
  if (wa.predict) {
    if (pred_done) cudaStreamWaitEvent(s, pred_done, 0);
    else large_block_warm_pred(le, lb, s);
  }
  k_warm_begin<<<dim3(wa.nt, wa.nt), 256, 0, s>>>(wa);
}
// refinement step j: W = Af X_j, [S, P] = X_j^T [W, X_j], stop test, clusters, M = V (I + E), X_{j+1} = X_j M.
// nest (graph capture only: s captures the step's IF body, nest is a stream outside any capture): the
// cluster kernels and k_warm_M go into nested IF nodes the stop test sets only when clusters exist, so a
// step without clusters launches GEMM, scan, E, GEMM only.
inline cudaError_t graph_new_handle(cudaStream_t s, unsigned long long* h);
inline cudaError_t graph_if_body(cudaStream_t s, unsigned long long h, cudaGraph_t* body);
inline cudaError_t large_block_warm_step(LargeEig& le, LargeBlock& lb, cudaStream_t s, int j, const WarmArgs& wa0,
                                         cudaStream_t nest = nullptr) {
  const int N = lb.N;
  WarmArgs wa = wa0;
  cudaError_t e = cudaSuccess;
  if (nest) {
    e = graph_new_handle(s, &wa.hclA);
    if (e == cudaSuccess) e = graph_new_handle(s, &wa.hclB);
    if (e != cudaSuccess) return e;
  }
  if (j == 0) dgemm_launch(DG_DEFAULT, lb.wdesc, 1, N, N, s, le.st, le.is, 1);  // W_0 = a X_0
  dgemm_launch(DG_DEFAULT, lb.wdesc + 5 * j + 1, 2, N, N, s, le.st, le.is, 1);   // S, P (upper tiles)
  k_warm_scan<<<dim3(wa.nt, wa.nt), 256, 0, s>>>(wa, j);
  auto nested = [&](unsigned long long h, auto&& body_fn) -> cudaError_t {
    if (!nest) {
      body_fn(s);
      return cudaSuccess;
    }
    cudaGraph_t body = nullptr;
    cudaError_t ee = graph_if_body(s, h, &body);
    if (ee == cudaSuccess) ee = cudaStreamBeginCaptureToGraph(nest, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (ee != cudaSuccess) return ee;
    body_fn(nest);
    cudaGraph_t out = nullptr;
    return cudaStreamEndCapture(nest, &out);
  };
  e = nested(wa.hclA, [&](cudaStream_t q) {
    k_warm_cluster<<<WM_CLB, WM_CLT, WM_CL_SMEM, q>>>(wa);
    k_warm_rot<<<dim3(wa.nt, 32), 256, 0, q>>>(wa);
  });
  if (e != cudaSuccess) return e;
  k_warm_E<<<dim3(wa.nt, wa.nt), 256, 0, s>>>(wa);
  e = nested(wa.hclB, [&](cudaStream_t q) { k_warm_M<<<dim3(wa.nt, wa.nt), 256, 0, q>>>(wa); });
  if (e != cudaSuccess) return e;
  dgemm_launch(DG_DEFAULT, lb.wdesc + 5 * j + 3, 2, N, N, s, le.st, le.is, 1);   // X M, W M
  return cudaSuccess;
}
// cold path of the warm mode: tridiagonalisation, WY factors, divide and conquer (every eigenvector when
// it re-seeds X, else the projected side only: k_dc_topsel reads ws->need_full); with side streams
// (sw, sd and 8 events) as in the concurrent variant, or sequential on s when sw == nullptr.
inline void large_block_cold(LargeEig& le, LargeBlock& lb, cudaStream_t s, cudaStream_t sw = nullptr,
                             cudaStream_t sd = nullptr, const cudaEvent_t* evs = nullptr) {
  const int N = lb.N;
  if (sw) {
    cudaEventRecord(evs[6], s);
    cudaStreamWaitEvent(sd, evs[6], 0);
    k_zero2<<<296, 256, 0, sd>>>(lb.dc.Q[0], lb.dc.Q[1], (long long)N * N);  // (kernel: conditional body)
    cudaEventRecord(evs[7], sd);
    large_block_tridiag(le, lb, s, true);
    cudaEventRecord(evs[0], s);
    cudaStreamWaitEvent(sw, evs[0], 0);
    large_block_wy(le, lb, sw, true);
    cudaEventRecord(evs[1], sw);
    large_block_dc(le, lb, s, true, sd, evs + 3);
    cudaStreamWaitEvent(s, evs[1], 0);
  } else {
    large_block_tridiag(le, lb, s, true);
    large_block_wy(le, lb, s, true);
    large_block_dc(le, lb, s, true);
  }
}
// full tail of the cold path: every eigenvector back-transformed, unscaled, into X0 (pitch ldn)
inline void large_block_bt_all(LargeEig& le, LargeBlock& lb, cudaStream_t s) {
  const int N = lb.N, fb = lb.D & 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(BTC_P * ((N + BTW_NC - 1) / BTW_NC), 1, 1);
  cfg.blockDim = dim3(BTC_NT, 1, 1);
  cfg.dynamicSmemBytes = bt_apply_smem_bytes(N);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = BTC_P;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_bt_apply, (const double*)lb.dc.Q[fb], (const double*)lb.dc.lam[fb],
                     (const double*)lb.V, (const double*)lb.Twy, (const int*)lb.sel_all, lb.wa.X0, N, lb.nref,
                     le.st, le.is, 1, lb.wa.ldn, 0);
}
// finish (warm success or full cold tail): side and index list, Xs / Ss gather, Y = Xs Ss, M = Y Xs^T
inline void large_block_warm_finish(LargeEig& le, LargeBlock& lb, cudaStream_t s) {
  const int N = lb.N;
  k_warm_select<<<1, WM_NT, 0, s>>>(lb.wa, lb.b);
  k_warm_gather<<<296, 256, 0, s>>>(lb.wa);
  dgemm_launch(DG_DEFAULT, lb.wdesc + 5 * WM_MAXS, 1, N, N, s, le.st, le.is, 1);
  dim3 gr((N + GM_BM - 1) / GM_BM, (N + GM_BN - 1) / GM_BN, 1);
  k_gemm_f64<<<gr, GM_NT, 0, s>>>(lb.gdesc + lb.wrecon, le.st, le.is, 1);
}
// un-graphed warm projection of one block: the refinement steps, then (host decisions after a sync) the
// cold path and its tail, or the finish.  ev (optional, 3 events): after the refinement / cold
// tridiagonalisation, after the cold D&C + back-transform, after the reconstruction.
inline cudaError_t large_block_warm_ungraphed(LargeEig& le, LargeBlock& lb, cudaStream_t s, cudaEvent_t* ev) {
  large_block_warm_begin(le, lb, s, lb.wa);
  for (int j = 0; j < WM_MAXS; ++j) large_block_warm_step(le, lb, s, j, lb.wa);
  WarmState h{};
  DevState hs{};
  cudaError_t e = cudaMemcpyAsync(&h, lb.wa.ws, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hs, le.st, sizeof(hs), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  if (h.status != 1 && !hs.done) {
    large_block_tridiag(le, lb, s, true);
    if (ev) cudaEventRecord(ev[0], s);
    large_block_wy(le, lb, s, true);
    large_block_dc(le, lb, s, true);
    k_warm_cold_switch<<<1, 1, 0, s>>>(lb.wa);  // (counter only: no graph handles here)
    if (h.need_full) {
      large_block_bt_all(le, lb, s);
      if (ev) cudaEventRecord(ev[1], s);
      large_block_warm_finish(le, lb, s);
    } else {
      if (ev) cudaEventRecord(ev[1], s);
      large_block_recon(le, lb, s, true, false);
    }
  } else {
    if (ev) cudaEventRecord(ev[0], s);
    if (ev) cudaEventRecord(ev[1], s);
    large_block_warm_finish(le, lb, s);
  }
  if (ev) cudaEventRecord(ev[2], s);
  return cudaSuccess;
}

// Stage-major over the large blocks; ev (optional, 3 events) is recorded after the
// tridiagonalisations, after the divide-and-conquer solves and after the reconstructions.
inline void large_eig_launch(LargeEig& le, cudaStream_t s, bool check, cudaEvent_t* ev = nullptr) {
  bool any_cold = false;
  for (auto& lb : le.blocks) any_cold |= !lb.warm;
  if (!any_cold) {  // every block in warm mode (the events then bracket the last block's phases)
    for (auto& lb : le.blocks) large_block_warm_ungraphed(le, lb, s, ev);
    return;
  }
  for (auto& lb : le.blocks)
    if (lb.warm) large_block_warm_ungraphed(le, lb, s, nullptr);
  for (auto& lb : le.blocks)
    if (!lb.warm) large_block_tridiag(le, lb, s, check);
  if (ev) cudaEventRecord(ev[0], s);
  for (auto& lb : le.blocks)
    if (!lb.warm) large_block_dc(le, lb, s, check);
  if (ev) cudaEventRecord(ev[1], s);
  for (auto& lb : le.blocks)
    if (!lb.warm) large_block_recon(le, lb, s, check);
  if (ev) cudaEventRecord(ev[2], s);
}

// Graph helpers: a conditional handle of the graph being captured on s, and an IF node appended to s's
// capture (its body graph returned for capture-to-graph on another stream).
inline cudaError_t graph_new_handle(cudaStream_t s, unsigned long long* h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, nullptr, nullptr);
  if (e != cudaSuccess) return e;
  if (cs != cudaStreamCaptureStatusActive) return cudaErrorStreamCaptureUnsupported;
  cudaGraphConditionalHandle hh;
  e = cudaGraphConditionalHandleCreate(&hh, g, 0, cudaGraphCondAssignDefault);
  *h = (unsigned long long)hh;
  return e;
}
inline cudaError_t graph_if_body(cudaStream_t s, unsigned long long h, cudaGraph_t* body) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess) return e;
  if (cs != cudaStreamCaptureStatusActive) return cudaErrorStreamCaptureUnsupported;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = (cudaGraphConditionalHandle)h;
  p.conditional.type = cudaGraphCondTypeIf;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, g, deps, nd, &p);
  if (e != cudaSuccess) return e;
  *body = p.conditional.phGraph_out[0];
  return cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
}

// Warm block inside a stream capture on sb (every branch an IF node, its body captured to graph on sbody):
//   begin -> step 0 .. WM_MAXS-1 (each set by begin / the previous stop test) -> cold eigensolver (set by
//   begin or a failed test; ends with k_warm_cold_switch) -> full tail (bt of every column + finish) or
//   partial tail (k_select + bt of the projected side + reconstruction) -> warm finish (set on success).
inline cudaError_t large_block_warm_graph(LargeEig& le, LargeBlock& lb, cudaStream_t sb, cudaStream_t sbody,
                                          cudaStream_t sw, cudaStream_t sd, const cudaEvent_t* evs,
                                          cudaStream_t snest = nullptr, cudaEvent_t pred_done = nullptr) {
  WarmArgs wg = lb.wa;
  cudaError_t e = cudaSuccess;
  // the first `unc` refinement steps as plain nodes (their kernels gated on ws->gate) instead of IF nodes
  int unc = 3;
  if (const char* ev = getenv("SOSADMM_WARM_UNCOND")) unc = std::max(0, std::min(WM_MAXS, atoi(ev)));
  for (int j = 0; j < WM_MAXS && e == cudaSuccess; ++j) {
    if (j < unc) wg.hstep[j] = 0;
    else e = graph_new_handle(sb, &wg.hstep[j]);
  }
  for (unsigned long long* h : {&wg.hcold, &wg.hfull, &wg.hpart, &wg.hfin})
    if (e == cudaSuccess) e = graph_new_handle(sb, h);
  if (e != cudaSuccess) return e;
  large_block_warm_begin(le, lb, sb, wg, pred_done);
  const int nbody = WM_MAXS + 4;
  for (int j = 0; j < nbody; ++j) {
    if (j < unc) {
      e = large_block_warm_step(le, lb, sb, j, wg, snest);
      if (e != cudaSuccess) return e;
      continue;
    }
    const unsigned long long h = j < WM_MAXS ? wg.hstep[j] : (j == WM_MAXS ? wg.hcold : (j == WM_MAXS + 1 ? wg.hfull : (j == WM_MAXS + 2 ? wg.hpart : wg.hfin)));
    cudaGraph_t body = nullptr;
    e = graph_if_body(sb, h, &body);
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(sbody, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    if (j < WM_MAXS) {
      e = large_block_warm_step(le, lb, sbody, j, wg, snest);
      if (e != cudaSuccess) {
        cudaGraph_t out = nullptr;
        cudaStreamEndCapture(sbody, &out);
        return e;
      }
    } else if (j == WM_MAXS) {
      large_block_cold(le, lb, sbody, sw, sd, evs);
      k_warm_cold_switch<<<1, 1, 0, sbody>>>(wg);
    } else if (j == WM_MAXS + 1) {
      large_block_bt_all(le, lb, sbody);
      large_block_warm_finish(le, lb, sbody);
    } else if (j == WM_MAXS + 2) {
      large_block_recon(le, lb, sbody, true, false);
    } else {
      large_block_warm_finish(le, lb, sbody);
    }
    cudaGraph_t out = nullptr;
    e = cudaStreamEndCapture(sbody, &out);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// Concurrent variant (graph path): every large block runs its chain on its own stream (block 0 on
// s), and inside a chain the WY factors run on a side stream beside the divide-and-conquer solve.
// fork: event already recorded on s; aux: >= 3 * nblocks streams; evs: >= 8 * nblocks events;
// body: one stream per block outside the capture (warm blocks' conditional bodies).
inline cudaError_t large_eig_launch_concurrent(LargeEig& le, cudaStream_t s, bool check, cudaEvent_t fork,
                                               const cudaStream_t* aux, const cudaEvent_t* evs,
                                               const cudaStream_t* body, const cudaStream_t* nest = nullptr,
                                               const cudaEvent_t* pred_done = nullptr) {
  const int nb = (int)le.blocks.size();
  for (int b = 0; b < nb; ++b) {
    LargeBlock& lb = le.blocks[b];
    cudaStream_t sb = b == 0 ? s : aux[3 * b];
    cudaStream_t sw = aux[3 * b + 1];
    cudaStream_t sd = aux[3 * b + 2];
    if (b > 0) cudaStreamWaitEvent(sb, fork, 0);
    if (lb.warm) {
      const cudaError_t e = large_block_warm_graph(le, lb, sb, body[b], sw, sd, evs + 8 * b, nest ? nest[b] : nullptr,
                                                   pred_done ? pred_done[b] : nullptr);
      if (e != cudaSuccess) return e;
      if (b > 0) cudaEventRecord(evs[8 * b + 2], sb);
      continue;
    }
    // the D&C eigenvector buffers are zeroed beside the tridiagonalisation
    cudaStreamWaitEvent(sd, fork, 0);
    cudaMemsetAsync(lb.dc.Q[0], 0, sizeof(double) * lb.N * lb.N, sd);
    cudaMemsetAsync(lb.dc.Q[1], 0, sizeof(double) * lb.N * lb.N, sd);
    cudaEventRecord(evs[8 * b + 7], sd);
    large_block_tridiag(le, lb, sb, check);
    cudaEventRecord(evs[8 * b], sb);         // tridiagonal + reflectors ready
    cudaStreamWaitEvent(sw, evs[8 * b], 0);
    large_block_wy(le, lb, sw, check);
    cudaEventRecord(evs[8 * b + 1], sw);
    large_block_dc(le, lb, sb, check, sd, evs + 8 * b + 3);
    cudaStreamWaitEvent(sb, evs[8 * b + 1], 0);
    large_block_recon(le, lb, sb, check, false);
    if (b > 0) cudaEventRecord(evs[8 * b + 2], sb);
  }
  for (int b = 1; b < nb; ++b) cudaStreamWaitEvent(s, evs[8 * b + 2], 0);
  return cudaSuccess;
}

inline int large_eig_launches(const LargeEig& le) {
  int k = 0;
  for (const auto& lb : le.blocks) {
    if (lb.warm) {  // begin, the refinement steps (IF nodes; an upper bound), the finish; cold path excluded
      k += 3 + 1 + WM_MAXS * 7 + 4;
      continue;
    }
    k += (lb.two ? 3 : (lb.ksw < lb.N - 2 ? 2 : 1)) + 2 + 1 + 7 * (lb.D - lb.jl) + 1 + 5 + (lb.two ? 1 : 0);
  }
  return k;
}

// Algorithmic FP64 flops of the last projection of one large block, from the device-side sizes it used
// (the roofline counts the method's own work, not dense upper bounds):
//   w[0] tridiagonalisation 4/3 N^3;  w[1] divide-and-conquer merge GEMMs sum 2 n k K over the merge nodes
//   (k = non-deflated count; the root forms only the selected columns);  w[2] back-transform 2 N^2 r
//   (+ 2 N^2 r through the stage-2 reflectors on the two-stage path);  w[3] reconstruction N (N + 32) r
//   (lower-triangle tiles of W W^T);  w[4] = r, w[5] = number of deflated-to-zero merges (context).
inline int large_block_work(const LargeBlock& lb, cudaStream_t s, double* w) {
  const int N = lb.N;
  std::vector<int> nk(lb.node_n.size());
  int top[4] = {0, 0, 0, 0}, sel[3] = {0, 0, 0};
  if (cudaMemcpyAsync(nk.data(), lb.dc.node_k, 4 * nk.size(), cudaMemcpyDeviceToHost, s) ||
      cudaMemcpyAsync(top, lb.dc.topsel, 12, cudaMemcpyDeviceToHost, s) ||
      cudaMemcpyAsync(sel, lb.sel, 12, cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
    return 1;
  double dc = 0.0, zero = 0.0;
  for (int h = lb.jl + 1; h <= lb.D; ++h)
    for (int t = 0; t < lb.level_nn[h]; ++t) {
      const int id = lb.level_node0[h] + t;
      const double n = lb.node_n[id], k = nk[id];
      const double cols = (h == lb.D && lb.dc.topsel_on) ? top[0] : k;
      dc += 2.0 * n * cols * k;
      zero += k == 0;
    }
  const double r = sel[0];
  w[0] = 4.0 / 3.0 * (double)N * N * N;
  w[1] = dc;
  w[2] = 2.0 * (double)N * N * r * (lb.two ? 2.0 : 1.0);
  w[3] = (double)N * (N + 32) * r;
  w[4] = r;
  w[5] = zero;
  return 0;
}

inline void large_eig_free(LargeEig& le) { le.blocks.clear(); }
