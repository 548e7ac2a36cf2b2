// sosadmm — C ABI implementation (see include/sosadmm.h for the contract and citations).
//
// Host side: structural analysis and the once-per-problem cache of SURVEY §8(a) row a0
// (P^{-1}, the t' x t' factor, M^{-1} zeta, 1 + zeta^T M^{-1} zeta).
// Device side: the per-iteration kernels of affine.cuh, psd_jacobi.cuh and psd_large.cuh, captured
// once into a CUDA graph and replayed; termination is decided on the device (done flag), so
// iterate(k) needs no host round trip inside the loop.
#include "../../include/sosadmm.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "affine.cuh"
#include "dgemm.cuh"
#include "psd_jacobi.cuh"
#include "psd_large.cuh"
#include "shard.cuh"
#include "spdinv.cuh"

namespace {

constexpr size_t kAlign = 256;
constexpr double SQRT2_HOST = 1.4142135623730951;  // fl(sqrt 2)

// NCCL is resolved at run time from the libnccl.so.2 already loaded by the process (torch's), so the
// library itself loads without NCCL and there is a single NCCL copy per process.
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  if (!api.tried) {
    api.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
      api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
      api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.getErrorString;
    }
  }
  return api;
}

struct ShardSpec {
  int rank = 0, world = 1;
  const int32_t* block_owner = nullptr;  // nullptr: every block on this rank
  bool sharded = false;                  // true: NCCL partial-sum allreduce in the loop
  bool emulated = false;                 // debug: no communicator; sosadmm_debug_group_iterate sums on one GPU
  bool peer = false;                     // f4: partial sums reduced over peer memory inside k_gather_fin_peer
};

constexpr int PEER_MAXW = 8;

struct GroupBufs {
  double* buf[8];
  int world;
};

struct Arena {
  char* base = nullptr;  // nullptr = dry run (size accounting only)
  size_t used = 0;
  template <class T>
  T* take(size_t count) {
    used = (used + kAlign - 1) / kAlign * kAlign;
    T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
    used += std::max<size_t>(count, 1) * sizeof(T);
    return p;
  }
};

struct Analysis {
  int m = 0, n = 0, t = 0, tl = 0, npsd = 0, nblk = 0;
  std::vector<int> code;
  std::vector<double> aval;
  std::vector<int> seg_ptr, seg_col, segpos;
  std::vector<double> seg_val;
  std::vector<int> low_col, lr_ptr, lr_idx, lr_col, lc_ptr, lc_row;
  std::vector<double> lr_val, lc_val;
  std::vector<int> empty_cols;
  std::vector<double> D, Pinv, b, c;
  std::vector<long long> blk_col, blk_mat;
  std::vector<int> blk_N;
  std::vector<int> cta_blk;
  std::vector<long long> cta_q0;
  std::vector<int> small_blk, large_blk;
  long long mat_total = 0;
  int max_small_N = 0;
  std::vector<long long> blk_vp;  // small blocks: offset of the warm-start eigenvector matrix (-1: none)
  long long vp_total = 0;
  std::vector<int> colown;  // 1: this rank accounts for the column in the sharded partial sums
};

// Column classification and the orthogonal / low-rank split (Proposition 1, P:302-311;
// Proposition 3): a PSD column with at most one nonzero and c_j = 0 is orthogonal.
sosadmm_err analyse(const sosadmm_problem* p, Analysis& an, std::string& msg, const ShardSpec& sp = ShardSpec()) {
  if (!p || p->m <= 0 || p->n_free < 0 || p->n_psd < 0 || !p->A_colptr || !p->b || !p->c ||
      (p->n_psd > 0 && !p->psd_dim)) {
    msg = "null pointer or negative size in sosadmm_problem";
    return SOSADMM_E_ARG;
  }
  if (p->m > (1LL << 30)) {
    msg = "m too large";
    return SOSADMM_E_ARG;
  }
  an.m = (int)p->m;
  an.t = (int)p->n_free;
  long long n = p->n_free;
  for (int b = 0; b < p->n_psd; ++b) {
    const int N = p->psd_dim[b];
    if (N <= 0) {
      msg = "PSD block dimension must be positive";
      return SOSADMM_E_ARG;
    }
    if (N > SOSADMM_MAX_BLOCK) {
      msg = "PSD block " + std::to_string(b) + " has dimension " + std::to_string(N) + " > " +
            std::to_string(SOSADMM_MAX_BLOCK) + " (largest supported block)";
      return SOSADMM_E_STRUCT;
    }
    n += (long long)N * (N + 1) / 2;
  }
  if (n > (1LL << 30)) {
    msg = "n too large";
    return SOSADMM_E_ARG;
  }
  an.n = (int)n;
  an.npsd = an.n - an.t;
  an.nblk = p->n_psd;
  const long long nnz = p->A_colptr[n];
  if (p->A_colptr[0] != 0 || nnz < 0) {
    msg = "bad CSC column pointers";
    return SOSADMM_E_ARG;
  }
  if (nnz > 0 && (!p->A_rowidx || !p->A_val)) {
    msg = "null A_rowidx / A_val with nnz > 0";
    return SOSADMM_E_ARG;
  }
  for (long long j = 0; j < n; ++j)
    if (p->A_colptr[j + 1] < p->A_colptr[j]) {
      msg = "CSC column pointers must be nondecreasing";
      return SOSADMM_E_ARG;
    }
  for (long long e = 0; e < nnz; ++e)
    if (p->A_rowidx[e] < 0 || p->A_rowidx[e] >= an.m) {
      msg = "CSC row index out of range at entry " + std::to_string(e);
      return SOSADMM_E_ARG;
    }
  an.b.assign(p->b, p->b + an.m);
  an.c.assign(p->c, p->c + an.n);
  an.code.assign(an.n, -2);
  an.aval.assign(an.n, 0.0);
  std::vector<int> cnt(an.m, 0);
  if (sp.sharded)
    for (int j = an.t; j < an.n; ++j)
      if (p->c[j] != 0.0) {
        // every rank evaluates c^T xi over all low columns in k_tphase, but only owned PSD columns are
        // updated: a PSD column with c_j != 0 would make the ranks' tau/kappa diverge
        msg = "sharded mode needs c_j = 0 on every PSD column (column " + std::to_string(j) + ")";
        return SOSADMM_E_STRUCT;
      }
  for (int j = an.t; j < an.n; ++j) {
    const long long e0 = p->A_colptr[j], e1 = p->A_colptr[j + 1];
    if (e1 - e0 <= 1 && p->c[j] == 0.0) {
      if (e1 == e0 || p->A_val[e0] == 0.0) {
        an.code[j] = -1;
        an.empty_cols.push_back(j);
      } else {
        an.code[j] = p->A_rowidx[e0];
        an.aval[j] = p->A_val[e0];
        cnt[p->A_rowidx[e0]]++;
      }
    }
  }
  // low columns: free ones and every non-orthogonal PSD column
  for (int j = 0; j < an.n; ++j)
    if (j < an.t || an.code[j] <= -2) {
      an.code[j] = -2 - (int)an.low_col.size();
      an.low_col.push_back(j);
    }
  an.tl = (int)an.low_col.size();
  if (an.tl > 16384) {
    msg = "low-rank width t' = " + std::to_string(an.tl) + " exceeds the supported 16384";
    return SOSADMM_E_STRUCT;
  }
  // CSR of A_orth (rows -> columns), D exactly: sum of (A/w)^2 w^2 per row
  an.seg_ptr.assign(an.m + 1, 0);
  for (int r = 0; r < an.m; ++r) an.seg_ptr[r + 1] = an.seg_ptr[r] + cnt[r];
  an.seg_col.resize(an.seg_ptr[an.m]);
  an.segpos.assign(an.n, -1);
  an.seg_val.resize(an.seg_ptr[an.m]);
  an.D.assign(an.m, 0.0);
  {
    std::vector<int> fill(an.seg_ptr.begin(), an.seg_ptr.end() - 1);
    for (int j = an.t; j < an.n; ++j)
      if (an.code[j] >= 0) {
        const int r = an.code[j];
        an.segpos[j] = fill[r];
        an.seg_col[fill[r]] = j;
        an.seg_val[fill[r]] = an.aval[j];
        fill[r]++;
        // A_orth A_orth^T is diagonal with entries sum_j A_rj^2; for indicator data the entries are
        // 1 or fl(sqrt 2) (scalar SOS, Proposition 1) or 1 on off-diagonal svec entries (off-diagonal
        // blocks of a matrix SOS, Proposition 2), whose squares are the integers 1 and 2 — counted
        // exactly (never fl(sqrt 2)^2 = 2.0000000000000004, reading C10)
        const double v = an.aval[j];
        an.D[r] += (v == 1.0 || v == -1.0) ? 1.0 : ((v == SQRT2_HOST || v == -SQRT2_HOST) ? 2.0 : v * v);
      }
  }
  an.Pinv.resize(an.m);
  for (int r = 0; r < an.m; ++r) an.Pinv[r] = 1.0 / (1.0 + an.D[r]);
  // A_low CSC and CSR
  an.lc_ptr.assign(an.tl + 1, 0);
  for (int jl = 0; jl < an.tl; ++jl) {
    const int j = an.low_col[jl];
    an.lc_ptr[jl + 1] = an.lc_ptr[jl] + (int)(p->A_colptr[j + 1] - p->A_colptr[j]);
  }
  an.lc_row.resize(an.lc_ptr[an.tl]);
  an.lc_val.resize(an.lc_ptr[an.tl]);
  std::vector<int> rc(an.m, 0);
  for (int jl = 0; jl < an.tl; ++jl) {
    const int j = an.low_col[jl];
    int o = an.lc_ptr[jl];
    for (long long e = p->A_colptr[j]; e < p->A_colptr[j + 1]; ++e, ++o) {
      an.lc_row[o] = p->A_rowidx[e];
      an.lc_val[o] = p->A_val[e];
      rc[p->A_rowidx[e]]++;
    }
  }
  an.lr_ptr.assign(an.m + 1, 0);
  for (int r = 0; r < an.m; ++r) an.lr_ptr[r + 1] = an.lr_ptr[r] + rc[r];
  an.lr_idx.resize(an.lr_ptr[an.m]);
  an.lr_val.resize(an.lr_ptr[an.m]);
  {
    std::vector<int> fill(an.lr_ptr.begin(), an.lr_ptr.end() - 1);
    for (int jl = 0; jl < an.tl; ++jl)
      for (int o = an.lc_ptr[jl]; o < an.lc_ptr[jl + 1]; ++o) {
        const int r = an.lc_row[o];
        an.lr_idx[fill[r]] = jl;
        an.lr_val[fill[r]] = an.lc_val[o];
        fill[r]++;
      }
  }
  an.lr_col.resize(an.lr_idx.size());  // direct column of each row entry (one indirection less in the gather)
  for (size_t e = 0; e < an.lr_idx.size(); ++e) an.lr_col[e] = an.low_col[an.lr_idx[e]];
  // PSD blocks (only the blocks this rank owns are scattered, projected and packed)
  long long col = an.t;
  an.mat_total = 0;
  an.vp_total = 0;
  an.colown.assign(an.n, 0);
  for (int j = 0; j < an.t; ++j) an.colown[j] = sp.rank == 0 ? 1 : 0;
  for (int b = 0; b < an.nblk; ++b) {
    const int N = p->psd_dim[b];
    const int owner = sp.block_owner ? sp.block_owner[b] : sp.rank;
    if (owner < 0 || owner >= sp.world) {
      msg = "block_owner[" + std::to_string(b) + "] out of range";
      return SOSADMM_E_ARG;
    }
    const bool mine = owner == sp.rank;
    an.blk_col.push_back(col);
    an.blk_N.push_back(N);
    an.blk_mat.push_back(an.mat_total);
    an.mat_total += (long long)N * N;
    const long long L = (long long)N * (N + 1) / 2;
    if (mine) {
      for (long long q = 0; q < L; ++q) an.colown[col + q] = 1;
      for (long long q0 = 0; q0 < L; q0 += POS_PER_CTA) {
        an.cta_blk.push_back(b);
        an.cta_q0.push_back(q0);
      }
      if (N <= JAC_MAXN) {
        an.small_blk.push_back(b);
        an.max_small_N = std::max(an.max_small_N, N);
        an.blk_vp.push_back(an.vp_total);
        an.vp_total += (long long)N * N;
      } else {
        an.large_blk.push_back(b);
      }
    }
    if ((long long)an.blk_vp.size() < (long long)an.blk_N.size()) an.blk_vp.push_back(-1);
    col += L;
  }
  return SOSADMM_OK;
}

// Dense SPD inverse on the host (t' x t', row-major): Cholesky K = L L^T, then K^{-1} = L^{-T} L^{-1}.
bool spd_inverse(std::vector<double>& K, int t) {
  std::vector<double>& L = K;  // in place, lower triangle
  for (int j = 0; j < t; ++j) {
    double d = L[(size_t)j * t + j];
    for (int k = 0; k < j; ++k) d -= L[(size_t)j * t + k] * L[(size_t)j * t + k];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    L[(size_t)j * t + j] = d;
    for (int i = j + 1; i < t; ++i) {
      double s = L[(size_t)i * t + j];
      const double* li = &L[(size_t)i * t];
      const double* lj = &L[(size_t)j * t];
      for (int k = 0; k < j; ++k) s -= li[k] * lj[k];
      L[(size_t)i * t + j] = s / d;
    }
  }
  // W = L^{-1} (lower), row-major
  std::vector<double> W((size_t)t * t, 0.0);
  for (int i = 0; i < t; ++i) {
    W[(size_t)i * t + i] = 1.0 / L[(size_t)i * t + i];
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s += L[(size_t)i * t + k] * W[(size_t)k * t + j];
      W[(size_t)i * t + j] = -s / L[(size_t)i * t + i];
    }
  }
  // K^{-1} = W^T W
  for (int i = 0; i < t; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0.0;
      for (int k = i; k < t; ++k) s += W[(size_t)k * t + i] * W[(size_t)k * t + j];
      K[(size_t)i * t + j] = s;
      K[(size_t)j * t + i] = s;
    }
  return true;
}

struct DevPtrs {
  int *seg_ptr, *seg_col, *segpos, *low_col, *lr_ptr, *lr_idx, *lr_col, *lc_ptr, *lc_row, *empty_cols, *code;
  double *xis, *zs;
  double *seg_val, *lr_val, *lc_val, *c_low, *h1_low, *beta_low, *Kinv, *b, *Pinv, *h2, *aval;
  double *xi, *z, *y, *s, *x, *uhat2, *yt, *zt, *ulow, *aty, *part, *asvec, *mats, *tmp, *kpart = nullptr;
  DevState* st;
  IterScal* is;
  long long *blk_col, *blk_mat, *cta_q0;
  int *blk_N, *cta_blk, *small_blk;
  int* colown;
  double* jvp;         // warm-start eigenvectors of the small blocks
  long long* blk_vp;
  double *shbuf, *shpart;
  double* hist;        // residual history ring (affine.cuh SOS_HIST entries of 5 doubles)
  unsigned long long *pflags, *pepoch;  // peer mode: [PEER_MAXW] arrival epochs, the round counter
  double** ppeer_buf;                    // [PEER_MAXW] device pointers (peer mode)
  unsigned long long** ppeer_flags;      // [PEER_MAXW]
  double* pred3;                         // the three reduced scalars
};

}  // namespace

struct sosadmm_ctx {
  Analysis an;
  sosadmm_err err = SOSADMM_OK;
  std::string msg;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* own_mem = nullptr;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  AffineArgs aa{};
  JacobiArgs ja{};
  LargeEig le;
  double* d_tmp = nullptr;  // n-length scratch for unit entry points
  cudaGraphExec_t graph = nullptr;
  cudaGraph_t graph_raw = nullptr;
  int gather_blocks = 1;
  double tol = 1e-4;
  long long max_iters = 2000;
  long long launches = 0;
  // host mirrors for get_structure
  std::vector<int> row_of;
  // sharded mode (shard.cuh)
  ShardSpec sp;
  ncclComm_t comm = nullptr;
  ShardArgs sh{};
  DevPtrs dp{};
  std::vector<void*> ipc_open;  // peer bases opened with cudaIpcOpenMemHandle (closed in destroy)
  int nb_low = 1;
  // parallel branches of the PSD projection inside the CUDA graph
  static constexpr int kMaxAux = 1 + 3 * 8;
  cudaStream_t aux[kMaxAux] = {};
  cudaStream_t body[8] = {};  // capture streams of the warm blocks' conditional bodies (outside the main capture)
  cudaStream_t nest[8] = {};  // and of the bodies nested inside them
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_blk[8 * 8] = {};
  // warm predictor branches (one per large block), forked at the start of the iteration beside the affine chain
  cudaStream_t pre[8] = {};
  cudaEvent_t ev_pre0 = nullptr, ev_pre[8] = {};
  bool early_pred = true;  // SOSADMM_EARLY_PRED=0 / sosadmm_set_shared_gpu: the predictor after the scatter, as un-graphed
  bool no_early_pred_env = false;
  // early-stop polling of sosadmm_iterate: pinned copies of the device state after each chunk of replays
  DevState* h_poll = nullptr;
  cudaEvent_t ev_poll[2] = {};
  bool aux_ok = false;
  bool nest_ok = true;  // nested conditional nodes in the warm step bodies (cleared if the capture rejects them)
};

namespace {

#define CK_CTX(ctx, call)                                                              \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      (ctx)->err = SOSADMM_E_CUDA;                                                     \
      (ctx)->msg = std::string(#call) + ": " + cudaGetErrorString(e_);                 \
      return (ctx)->err;                                                               \
    }                                                                                  \
  } while (0)

// Device buffer layout (identical in the dry run and the real carve).
template <class F>
void layout(const Analysis& an, Arena& ar, F&& bind) {
  bind(ar);
}


int low_blocks(const Analysis& an) {
  return std::max(1, std::max((an.tl + SH_NT / 32 - 1) / (SH_NT / 32), ((int)an.empty_cols.size() + SH_NT - 1) / SH_NT));
}

void carve(const Analysis& an, Arena& ar, DevPtrs& d, int gather_blocks) {
  const size_t m = an.m, n = an.n, tl = an.tl;
  d.seg_ptr = ar.take<int>(m + 1);
  d.seg_col = ar.take<int>(an.seg_col.size());
  d.segpos = ar.take<int>(n);
  d.xis = ar.take<double>(std::max<size_t>(an.seg_col.size(), 1));
  d.zs = ar.take<double>(std::max<size_t>(an.seg_col.size(), 1));
  d.seg_val = ar.take<double>(an.seg_val.size());
  d.low_col = ar.take<int>(tl);
  d.lr_ptr = ar.take<int>(m + 1);
  d.lr_idx = ar.take<int>(an.lr_idx.size());
  d.lr_col = ar.take<int>(an.lr_col.size());
  d.lr_val = ar.take<double>(an.lr_val.size());
  d.lc_ptr = ar.take<int>(tl + 1);
  d.lc_row = ar.take<int>(an.lc_row.size());
  d.lc_val = ar.take<double>(an.lc_val.size());
  d.c_low = ar.take<double>(tl);
  d.h1_low = ar.take<double>(tl);
  d.beta_low = ar.take<double>(tl);
  d.Kinv = ar.take<double>(tl * (tl + (tl & 1)));  // leading dimension tl rounded up to even
  d.empty_cols = ar.take<int>(an.empty_cols.size());
  d.b = ar.take<double>(m);
  d.Pinv = ar.take<double>(m);
  d.h2 = ar.take<double>(m);
  d.code = ar.take<int>(n);
  d.aval = ar.take<double>(n);
  d.xi = ar.take<double>(n);
  d.z = ar.take<double>(n);
  d.y = ar.take<double>(m);
  d.s = ar.take<double>(m);
  d.x = ar.take<double>(m);
  d.uhat2 = ar.take<double>(m);
  d.yt = ar.take<double>(tl);
  d.zt = ar.take<double>(tl);
  d.ulow = ar.take<double>(tl);
  d.aty = ar.take<double>(tl);
  if (tl >= KINV_SYM_MIN) {
    const size_t nt = (size_t)(tl + KT - 1) / KT;
    d.kpart = ar.take<double>(nt * nt * KT);
  }
  d.part = ar.take<double>((size_t)NPART * gather_blocks);
  d.hist = ar.take<double>((size_t)5 * SOS_HIST);
  d.asvec = ar.take<double>(an.npsd);
  d.mats = ar.take<double>((size_t)an.mat_total);
  d.tmp = ar.take<double>(std::max<size_t>(n, 1));
  d.st = ar.take<DevState>(1);
  d.is = ar.take<IterScal>(1);
  d.blk_col = ar.take<long long>(an.nblk);
  d.blk_mat = ar.take<long long>(an.nblk);
  d.blk_N = ar.take<int>(an.nblk);
  d.cta_blk = ar.take<int>(an.cta_blk.size());
  d.cta_q0 = ar.take<long long>(an.cta_q0.size());
  d.small_blk = ar.take<int>(an.small_blk.size());
  d.colown = ar.take<int>(n);
  d.jvp = ar.take<double>((size_t)std::max<long long>(an.vp_total, 1));
  d.blk_vp = ar.take<long long>(an.nblk);
  d.shbuf = ar.take<double>(2 * (2 * m + 3));  // peer mode alternates two buffers by epoch parity
  d.pflags = ar.take<unsigned long long>(PEER_MAXW);
  d.pepoch = ar.take<unsigned long long>(1);
  d.ppeer_buf = ar.take<double*>(PEER_MAXW);
  d.ppeer_flags = ar.take<unsigned long long*>(PEER_MAXW);
  d.pred3 = ar.take<double>(3);
  d.shpart = ar.take<double>(3 * (size_t)std::max(gather_blocks, low_blocks(an)));
}

size_t total_bytes(const Analysis& an) {
  Arena ar;
  DevPtrs d;
  const int gb = std::max(1, (an.m + GATHER_NT - 1) / GATHER_NT);
  carve(an, ar, d, gb);
  ar.used += large_eig_bytes(an.blk_N, an.large_blk) + kAlign;
  if (an.tl > 256) ar.used += spdinv_scratch_bytes(an.tl) + kAlign;  // setup-time scratch of the K inverse
  return ar.used + kAlign;
}

template <class T>
cudaError_t h2d(T* dst, const std::vector<T>& src, cudaStream_t s) {
  if (src.empty()) return cudaSuccess;
  return cudaMemcpyAsync(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s);
}

// z_t = K^{-1} y_t: one warp per row while K^{-1} is L2-sized, else the lower-triangle tile apply
// (half the HBM bytes; affine.cuh k_kinv_tiles / k_kinv_sum)
void launch_kinv(const AffineArgs& a, cudaStream_t s) {
  if (a.tl >= KINV_SYM_MIN) {
    const int nt = (a.tl + KT - 1) / KT;
    k_kinv_tiles<<<nt * (nt + 1) / 2, 256, 0, s>>>(a);
    k_kinv_sum<<<nt, 256, 0, s>>>(a);
  } else {
    k_kinv<<<std::max(1, (a.tl * 32 + 255) / 256), 256, 0, s>>>(a);
  }
}

// y_t = A_low^T x, z_t = K^{-1} y_t, then the single-CTA tau phase; for small t' the tau phase does all three
void launch_low_tphase(const AffineArgs& a, cudaStream_t s, int mode) {
  if (!a.fuse_low) {
    k_lowT<<<std::max(1, (a.tl * 32 + 255) / 256), 256, 0, s>>>(a);
    launch_kinv(a, s);
  }
  k_tphase<<<1, TP_NT, 0, s>>>(a, mode);
}

void launch_rowupdate(const AffineArgs& a, cudaStream_t s, int write_state) {
  if (a.row_lanes == 8)
    k_rowupdate8<<<(int)(((long long)a.m * 8 + 255) / 256), 256, 0, s>>>(a, write_state);
  else
    k_rowupdate<<<(a.m + 255) / 256, 256, 0, s>>>(a, write_state);
}

// phase (sharded mode only): 0 = the whole iteration with the NCCL allreduce inside; 1 = up to the
// collective (the 2m + 3 partial sums in sh.buf); 2 = from the completed sums on.  Phases 1 / 2 are the
// one-GPU emulation of several ranks (sosadmm_debug_group_iterate), which sums sh.buf itself.
sosadmm_err launch_iteration(sosadmm_ctx* c, int mode_full, cudaEvent_t* ev, int phase = 0) {
  AffineArgs& a = c->aa;
  cudaStream_t s = c->stream;
  if (ev) cudaEventRecord(ev[0], s);
  // graph path: the warm blocks' predictor (k_warm_pred + one GEMM; inputs = what the previous iteration left)
  // forks here and runs beside the affine chain; large_block_warm_begin joins it.  Its kernels read the
  // done / proceed flags k_tphase is about to write: at worst the predictor of the stopping iteration runs
  // (it touches only the warm start buffers, and nothing runs after the stop).
  cudaEvent_t pred_done[8] = {};
  bool any_pred = false;
  {
    cudaStreamCaptureStatus cap0 = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap0);
    if (mode_full && !ev && phase == 0 && !c->sp.emulated && c->early_pred && c->aux_ok && cap0 == cudaStreamCaptureStatusActive) {
      for (size_t b = 0; b < c->le.blocks.size() && b < 8; ++b) any_pred |= c->le.blocks[b].warm && c->le.blocks[b].wa.predict;
      if (any_pred) {
        cudaEventRecord(c->ev_pre0, s);
        for (size_t b = 0; b < c->le.blocks.size() && b < 8; ++b) {
          LargeBlock& lb = c->le.blocks[b];
          if (!(lb.warm && lb.wa.predict)) continue;
          cudaStreamWaitEvent(c->pre[b], c->ev_pre0, 0);
          large_block_warm_pred(c->le, lb, c->pre[b]);
          cudaEventRecord(c->ev_pre[b], c->pre[b]);
          pred_done[b] = c->ev_pre[b];
        }
      }
    }
  }
  if (c->sp.sharded) {
    if (c->sp.emulated && phase == 0) {
      c->err = SOSADMM_E_ARG;
      c->msg = "an emulated sharded context iterates only through sosadmm_debug_group_iterate";
      return c->err;
    }
    if (phase != 2) {
      k_lowdual_part<<<c->nb_low, SH_NT, 0, s>>>(a, c->sh);
      k_gather_part<<<c->gather_blocks, SH_NT, 0, s>>>(a, c->sh);
      k_shard_scalars<<<1, SH_NT, 0, s>>>(a, c->sh, c->gather_blocks, c->nb_low);
      if (c->sp.peer) k_peer_signal<<<1, 1, 0, s>>>(a, c->sh);
      if (phase == 1) return SOSADMM_OK;
    }
    if (c->sp.peer) {  // the reduction over peer memory, fused into the consumer (no NCCL call)
      k_gather_fin_peer<<<c->gather_blocks, GATHER_NT, 0, s>>>(a, c->sh);
    } else {
      if (phase != 2) {
        const ncclResult_t nr = nccl().allReduce(c->sh.buf, c->sh.buf, 2 * (size_t)a.m + 3, ncclFloat64, ncclSum,
                                                 c->comm, s);
        if (nr != ncclSuccess) {
          c->err = SOSADMM_E_NCCL;
          c->msg = std::string("ncclAllReduce: ") + nccl().getErrorString(nr);
          return c->err;
        }
      }
      k_gather_fin<<<c->gather_blocks, GATHER_NT, 0, s>>>(a, c->sh);
    }
  } else {
    k_gather<<<c->gather_blocks, GATHER_NT, 0, s>>>(a);
  }
  launch_low_tphase(a, s, mode_full ? 0 : 1);
  if (!mode_full) return SOSADMM_OK;
  launch_rowupdate(a, s, 1);
  if (ev) cudaEventRecord(ev[1], s);
  if (a.pos_ctas > 0) k_scatter<<<a.pos_ctas, POS_NT, 0, s>>>(a, 0);
  if (ev) cudaEventRecord(ev[2], s);
  const bool has_small = !c->an.small_blk.empty(), has_large = !c->an.large_blk.empty();
  cudaStreamCaptureStatus capst = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &capst);
  if (!ev && has_large && c->aux_ok && capst == cudaStreamCaptureStatusActive) {
    // graph path: Jacobi blocks, every large block's chain and its WY factors on parallel branches
    cudaEventRecord(c->ev_fork, s);
    if (has_small) {
      cudaStreamWaitEvent(c->aux[0], c->ev_fork, 0);
      jacobi_kernel(c->an.max_small_N, c->ja.blocked)<<<(int)c->an.small_blk.size(), jacobi_threads(c->an.max_small_N), jacobi_smem_bytes(c->an.max_small_N),
                                         c->aux[0]>>>(c->ja);
      cudaEventRecord(c->ev_join, c->aux[0]);
    }
    const cudaError_t ge = large_eig_launch_concurrent(c->le, s, true, c->ev_fork, c->aux + 1, c->ev_blk, c->body,
                                                       c->nest_ok ? c->nest : nullptr, any_pred ? pred_done : nullptr);
    if (ge != cudaSuccess) {
      c->err = SOSADMM_E_CUDA;
      c->msg = std::string("large-block projection capture: ") + cudaGetErrorString(ge);
      return c->err;
    }
    if (has_small) cudaStreamWaitEvent(s, c->ev_join, 0);
  } else {
    if (has_small)
      jacobi_kernel(c->an.max_small_N, c->ja.blocked)<<<(int)c->an.small_blk.size(), jacobi_threads(c->an.max_small_N), jacobi_smem_bytes(c->an.max_small_N),
                                         s>>>(c->ja);
    if (ev) cudaEventRecord(ev[3], s);
    if (has_large) {
      large_eig_launch(c->le, s, true, ev ? ev + 4 : nullptr);
    } else if (ev) {
      for (int q = 4; q < 7; ++q) cudaEventRecord(ev[q], s);
    }
  }
  if (a.pos_ctas > 0) k_pack<<<a.pos_ctas, POS_NT, 0, s>>>(a, nullptr, 1);
  else k_commit<<<1, 1, 0, s>>>(a);
  if (ev) cudaEventRecord(ev[7], s);
  return SOSADMM_OK;
}

int64_t count_launches(const sosadmm_ctx* c) {
  int64_t k = c->sp.sharded ? 9 : 6;  // gather (sharded: 4 kernels + allreduce), lowT, kinv, tphase, rowupdate, pack
  if (c->an.tl >= KINV_SYM_MIN) k += 1;  // symmetric K^{-1} apply: tiles + fixed-order sum
  if (c->aa.fuse_low) k -= 2;            // k_tphase does k_lowT's and k_kinv's work
  if (c->aa.pos_ctas > 0) k += 1;
  if (!c->an.small_blk.empty()) k += 1;
  if (!c->an.large_blk.empty()) k += large_eig_launches(c->le);
  return k;
}

sosadmm_err check_async(sosadmm_ctx* c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    c->err = SOSADMM_E_CUDA;
    c->msg = std::string("kernel launch: ") + cudaGetErrorString(e);
  }
  return c->err;
}

sosadmm_err read_info(sosadmm_ctx* c, sosadmm_info* out) {
  DevState st;
  CK_CTX(c, cudaMemcpyAsync(&st, c->aa.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  if (st.nonfinite) {
    c->err = SOSADMM_E_NONFINITE;
    c->msg = "non-finite iterate at iteration " + std::to_string(st.nonfinite_iter);
  }
  if (out) {
    out->iter = st.iter;
    out->status = st.status;
    out->res_pri = st.res_pri;
    out->res_dual = st.res_dual;
    out->res_gap = st.res_gap;
    out->pobj = st.pobj;
    out->dobj = st.dobj;
    out->tau = st.tau;
    out->kappa = st.kappa;
    out->pinf = st.pinf;
    out->dinf = st.dinf;
  }
  return c->err;
}

// Peer mode (f4): every rank's partial buffers and flag slots, device pointers in rank order
// (own entries included), installed into the context; the round counter and the flags start at 0.
sosadmm_err peer_wire(sosadmm_ctx* c, const std::vector<double*>& bufs, const std::vector<unsigned long long*>& flags) {
  const int W = c->sp.world;
  if (W > PEER_MAXW || (int)bufs.size() != W || (int)flags.size() != W) {
    c->err = SOSADMM_E_ARG;
    c->msg = "peer mode supports at most 8 ranks";
    return c->err;
  }
  DevPtrs& d = c->dp;
  cudaStream_t s = c->stream;
  CK_CTX(c, cudaMemcpyAsync(d.ppeer_buf, bufs.data(), sizeof(double*) * W, cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemcpyAsync(d.ppeer_flags, flags.data(), sizeof(unsigned long long*) * W, cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemsetAsync(d.pflags, 0, sizeof(unsigned long long) * PEER_MAXW, s));
  CK_CTX(c, cudaMemsetAsync(d.pepoch, 0, sizeof(unsigned long long), s));
  CK_CTX(c, cudaStreamSynchronize(s));
  c->sp.peer = true;
  c->sh.epoch = d.pepoch;
  c->sh.flags = d.pflags;
  c->sh.peer_buf = d.ppeer_buf;
  c->sh.peer_flags = d.ppeer_flags;
  c->sh.red3 = d.pred3;
  c->aa.shard_scal = d.pred3;
  return SOSADMM_OK;
}

// Real multi-GPU peer mode: exchange CUDA IPC handles of every rank's workspace allocation (one
// ncclAllGather at setup) and open the peers' buffers (NVLink peer mappings).
struct PeerRec {
  cudaIpcMemHandle_t h;
  unsigned long long off_buf, off_flags;
};
sosadmm_err peer_setup_ipc(sosadmm_ctx* c) {
  typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK_CTX(c, cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &qr));
  if (!fn || qr != cudaDriverEntryPointSuccess || !nccl().allGather) {
    c->err = SOSADMM_E_CUDA;
    c->msg = "peer mode: cuMemGetAddressRange / ncclAllGather unavailable";
    return c->err;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (((GetRange)fn)(&base, &size, (CUdeviceptr)c->dp.shbuf) != CUDA_SUCCESS) {
    c->err = SOSADMM_E_CUDA;
    c->msg = "peer mode: cuMemGetAddressRange failed";
    return c->err;
  }
  PeerRec me{};
  CK_CTX(c, cudaIpcGetMemHandle(&me.h, (void*)base));
  me.off_buf = (unsigned long long)((CUdeviceptr)c->dp.shbuf - base);
  me.off_flags = (unsigned long long)((CUdeviceptr)c->dp.pflags - base);
  const int W = c->sp.world;
  char* dsend = (char*)c->d_tmp;  // scratch (>= (W + 1) * sizeof(PeerRec) bytes: checked by the caller)
  char* drecv = dsend + sizeof(PeerRec);
  CK_CTX(c, cudaMemcpyAsync(dsend, &me, sizeof(me), cudaMemcpyHostToDevice, c->stream));
  const ncclResult_t nr = nccl().allGather(dsend, drecv, sizeof(PeerRec), ncclUint8, c->comm, c->stream);
  if (nr != ncclSuccess) {
    c->err = SOSADMM_E_NCCL;
    c->msg = std::string("ncclAllGather: ") + nccl().getErrorString(nr);
    return c->err;
  }
  std::vector<PeerRec> all(W);
  CK_CTX(c, cudaMemcpyAsync(all.data(), drecv, sizeof(PeerRec) * W, cudaMemcpyDeviceToHost, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  std::vector<double*> bufs(W);
  std::vector<unsigned long long*> flags(W);
  for (int q = 0; q < W; ++q) {
    if (q == c->sp.rank) {
      bufs[q] = c->dp.shbuf;
      flags[q] = c->dp.pflags;
      continue;
    }
    void* pb = nullptr;
    CK_CTX(c, cudaIpcOpenMemHandle(&pb, all[q].h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_open.push_back(pb);
    bufs[q] = (double*)((char*)pb + all[q].off_buf);
    flags[q] = (unsigned long long*)((char*)pb + all[q].off_flags);
  }
  return peer_wire(c, bufs, flags);
}

}  // namespace

extern "C" {

size_t sosadmm_workspace_size(const sosadmm_problem* prob) {
  Analysis an;
  std::string msg;
  if (analyse(prob, an, msg) != SOSADMM_OK) return 0;
  return total_bytes(an);
}

static sosadmm_err setup_impl(const sosadmm_problem* prob, const sosadmm_settings* settings, const ShardSpec& sp,
                              const void* nccl_id, sosadmm_ctx** out) {
  if (!out) return SOSADMM_E_ARG;
  *out = nullptr;
  sosadmm_ctx* c = new sosadmm_ctx();
  *out = c;
  c->sp = sp;
  Analysis& an = c->an;
  c->err = analyse(prob, an, c->msg, sp);
  if (c->err != SOSADMM_OK) return c->err;
  if (settings) {
    c->tol = settings->tol > 0 ? settings->tol : 1e-4;
    c->max_iters = settings->max_iters > 0 ? settings->max_iters : 2000;
    c->device = settings->device;
  }
  CK_CTX(c, cudaSetDevice(c->device));
  if (sp.sharded && !sp.emulated) {
    if (!nccl().ok) {
      c->err = SOSADMM_E_NCCL;
      c->msg = "libnccl.so.2 could not be loaded";
      return c->err;
    }
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    const ncclResult_t nr = nccl().commInitRank(&c->comm, sp.world, id, sp.rank);
    if (nr != ncclSuccess) {
      c->err = SOSADMM_E_NCCL;
      c->msg = std::string("ncclCommInitRank: ") + nccl().getErrorString(nr);
      return c->err;
    }
  }
  if (settings && settings->stream) {
    c->stream = (cudaStream_t)settings->stream;
  } else {
    CK_CTX(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  const size_t need = total_bytes(an);
  if (!settings || !settings->workspace) {  // the caller owns all device memory (SURVEY §8(b) ownership)
    c->err = SOSADMM_E_ARG;
    c->msg = "settings.workspace is required (sosadmm_workspace_size bytes of device memory)";
    return c->err;
  }
  if (settings->workspace_bytes < need) {
    c->err = SOSADMM_E_OOM;
    c->msg = "workspace too small: need " + std::to_string(need) + " bytes";
    return c->err;
  }
  c->ws = (char*)settings->workspace;
  c->ws_bytes = settings->workspace_bytes;
  c->gather_blocks = std::max(1, (an.m + GATHER_NT - 1) / GATHER_NT);
  Arena ar;
  ar.base = (char*)(((uintptr_t)c->ws + kAlign - 1) / kAlign * kAlign);
  DevPtrs d;
  carve(an, ar, d, c->gather_blocks);
  char* large_base = ar.take<char>(large_eig_bytes(an.blk_N, an.large_blk));
  char* spd_scratch = an.tl > 256 ? ar.take<char>(spdinv_scratch_bytes(an.tl)) : nullptr;

  // ---- cache (row a0): K = I + A_low^T P^{-1} A_low, K^{-1}, h = M^{-1} zeta, denom --------
  const int tl = an.tl, m = an.m;
  std::vector<double> K((size_t)tl * tl, 0.0);
  for (int j = 0; j < tl; ++j) K[(size_t)j * tl + j] = 1.0;
  for (int r = 0; r < m; ++r) {
    const double pi = an.Pinv[r];
    for (int e = an.lr_ptr[r]; e < an.lr_ptr[r + 1]; ++e)
      for (int f = an.lr_ptr[r]; f < an.lr_ptr[r + 1]; ++f)
        K[(size_t)an.lr_idx[e] * tl + an.lr_idx[f]] += an.lr_val[e] * pi * an.lr_val[f];
  }
  bool spd_ok;
  if (tl <= 256) {
    spd_ok = spd_inverse(K, tl);
  } else {  // large t' (weighted SOS, config 3): blocked Cholesky + inverse on the DMMA GEMM
    CK_CTX(c, cudaMemcpyAsync(d.Kinv, K.data(), sizeof(double) * K.size(), cudaMemcpyHostToDevice, c->stream));
    const int rc = gpu_spd_inverse(d.Kinv, tl, c->stream, spd_scratch);
    if (rc == 2) {
      c->err = SOSADMM_E_CUDA;
      c->msg = "GPU inverse of I + A_low^T P^{-1} A_low failed";
      return c->err;
    }
    spd_ok = rc == 0;
    CK_CTX(c, cudaMemcpyAsync(K.data(), d.Kinv, sizeof(double) * K.size(), cudaMemcpyDeviceToHost, c->stream));
    CK_CTX(c, cudaStreamSynchronize(c->stream));
  }
  if (!spd_ok) {
    c->err = SOSADMM_E_FACTOR;
    c->msg = "I + A_low^T P^{-1} A_low is not numerically positive definite";
    return c->err;
  }
  std::vector<double> c_low(tl), beta_low(tl, 0.0), h1_low(tl), h2(m);
  for (int j = 0; j < tl; ++j) c_low[j] = an.c[an.low_col[j]];
  // M^{-1} zeta with zeta = (c, -b):  r1 = c, r2 = -b;  A r1 = A_low c_low (c = 0 on orth cols)
  {
    std::vector<double> x(m), yt(tl, 0.0), zt(tl, 0.0);
    for (int r = 0; r < m; ++r) {
      double g = 0.0;
      for (int e = an.lr_ptr[r]; e < an.lr_ptr[r + 1]; ++e) g += an.lr_val[e] * c_low[an.lr_idx[e]];
      x[r] = (-an.b[r] - g) * an.Pinv[r];
    }
    for (int j = 0; j < tl; ++j) {
      double s = 0.0, sb = 0.0;
      for (int e = an.lc_ptr[j]; e < an.lc_ptr[j + 1]; ++e) {
        s += an.lc_val[e] * x[an.lc_row[e]];
        sb += an.lc_val[e] * an.Pinv[an.lc_row[e]] * an.b[an.lc_row[e]];
      }
      yt[j] = s;
      beta_low[j] = sb;
    }
    for (int i = 0; i < tl; ++i) {
      double s = 0.0;
      for (int j = 0; j < tl; ++j) s += K[(size_t)i * tl + j] * yt[j];
      zt[i] = s;
    }
    for (int r = 0; r < m; ++r) {
      double v = 0.0;
      for (int e = an.lr_ptr[r]; e < an.lr_ptr[r + 1]; ++e) v += an.lr_val[e] * zt[an.lr_idx[e]];
      h2[r] = x[r] - an.Pinv[r] * v;
    }
    for (int j = 0; j < tl; ++j) {
      double s = 0.0;
      for (int e = an.lc_ptr[j]; e < an.lc_ptr[j + 1]; ++e) s += an.lc_val[e] * h2[an.lc_row[e]];
      h1_low[j] = c_low[j] + s;
    }
  }
  // 1 + zeta^T M^{-1} zeta, accumulated in extended precision (it divides u_hat_3, reading C15)
  long double ch = 0.0L, bhl = 0.0L, nbl = 0.0L, ncl = 0.0L;
  for (int j = 0; j < tl; ++j) ch += (long double)c_low[j] * h1_low[j];
  for (int r = 0; r < m; ++r) {
    bhl += (long double)an.b[r] * h2[r];
    nbl += (long double)an.b[r] * an.b[r];
  }
  for (int j = 0; j < an.n; ++j) ncl += (long double)an.c[j] * an.c[j];
  const double denom = (double)(1.0L + ch - bhl);
  const double bh = (double)bhl, nb = (double)nbl, nc = (double)ncl;

  // ---- upload -----------------------------------------------------------------------------
  cudaStream_t s = c->stream;
  {
    const std::vector<double> h0((size_t)5 * SOS_HIST, -1.0);  // empty history slots
    CK_CTX(c, h2d(d.hist, h0, s));
  }
  CK_CTX(c, h2d(d.seg_ptr, an.seg_ptr, s));
  CK_CTX(c, h2d(d.seg_col, an.seg_col, s));
  CK_CTX(c, h2d(d.segpos, an.segpos, s));
  CK_CTX(c, h2d(d.seg_val, an.seg_val, s));
  CK_CTX(c, h2d(d.low_col, an.low_col, s));
  CK_CTX(c, h2d(d.lr_ptr, an.lr_ptr, s));
  CK_CTX(c, h2d(d.lr_idx, an.lr_idx, s));
  CK_CTX(c, h2d(d.lr_col, an.lr_col, s));
  CK_CTX(c, h2d(d.lr_val, an.lr_val, s));
  CK_CTX(c, h2d(d.lc_ptr, an.lc_ptr, s));
  CK_CTX(c, h2d(d.lc_row, an.lc_row, s));
  CK_CTX(c, h2d(d.lc_val, an.lc_val, s));
  CK_CTX(c, h2d(d.c_low, c_low, s));
  CK_CTX(c, h2d(d.h1_low, h1_low, s));
  CK_CTX(c, h2d(d.beta_low, beta_low, s));
  {  // K^{-1} rows at an even pitch (16-byte aligned column pairs); the padding column is never read
    const size_t ldk = (size_t)tl + (tl & 1);
    CK_CTX(c, cudaMemcpy2DAsync(d.Kinv, ldk * sizeof(double), K.data(), (size_t)tl * sizeof(double),
                                (size_t)tl * sizeof(double), (size_t)tl, cudaMemcpyHostToDevice, s));
  }
  CK_CTX(c, h2d(d.empty_cols, an.empty_cols, s));
  CK_CTX(c, h2d(d.b, an.b, s));
  CK_CTX(c, h2d(d.Pinv, an.Pinv, s));
  CK_CTX(c, h2d(d.h2, h2, s));
  CK_CTX(c, h2d(d.code, an.code, s));
  CK_CTX(c, h2d(d.aval, an.aval, s));
  CK_CTX(c, h2d(d.blk_col, an.blk_col, s));
  CK_CTX(c, h2d(d.blk_mat, an.blk_mat, s));
  CK_CTX(c, h2d(d.blk_N, an.blk_N, s));
  CK_CTX(c, h2d(d.cta_blk, an.cta_blk, s));
  CK_CTX(c, h2d(d.cta_q0, an.cta_q0, s));
  CK_CTX(c, h2d(d.small_blk, an.small_blk, s));
  CK_CTX(c, h2d(d.colown, an.colown, s));
  CK_CTX(c, h2d(d.blk_vp, an.blk_vp, s));
  if (an.vp_total > 0) {  // warm-start eigenvectors start as identities (the first solve is cold)
    std::vector<double> eye((size_t)an.vp_total, 0.0);
    for (int b : an.small_blk) {
      const int N = an.blk_N[b];
      for (int i = 0; i < N; ++i) eye[(size_t)an.blk_vp[b] + (size_t)i * N + i] = 1.0;
    }
    CK_CTX(c, cudaMemcpyAsync(d.jvp, eye.data(), sizeof(double) * eye.size(), cudaMemcpyHostToDevice, s));
    CK_CTX(c, cudaStreamSynchronize(s));  // `eye` leaves scope
  }
  CK_CTX(c, cudaMemsetAsync(d.shbuf, 0, sizeof(double) * (2 * (size_t)an.m + 3), s));
  CK_CTX(c, cudaMemsetAsync(d.xi, 0, sizeof(double) * an.n, s));
  CK_CTX(c, cudaMemsetAsync(d.z, 0, sizeof(double) * an.n, s));
  CK_CTX(c, cudaMemsetAsync(d.xis, 0, sizeof(double) * std::max<size_t>(an.seg_col.size(), 1), s));
  CK_CTX(c, cudaMemsetAsync(d.zs, 0, sizeof(double) * std::max<size_t>(an.seg_col.size(), 1), s));
  CK_CTX(c, cudaMemsetAsync(d.y, 0, sizeof(double) * an.m, s));
  CK_CTX(c, cudaMemsetAsync(d.s, 0, sizeof(double) * an.m, s));
  CK_CTX(c, cudaMemsetAsync(d.mats, 0, sizeof(double) * std::max<long long>(an.mat_total, 1), s));
  DevState st0{};
  st0.tau = 1.0;  // reading C7: u0 = (0, 0, 1), v0 = 0
  st0.kappa = 0.0;
  st0.max_iters = c->max_iters;
  st0.tol = c->tol;
  st0.res_pri = st0.res_dual = st0.res_gap = INFINITY;
  CK_CTX(c, cudaMemcpyAsync(d.st, &st0, sizeof(DevState), cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemsetAsync(d.is, 0, sizeof(IterScal), s));

  AffineArgs& a = c->aa;
  a.m = an.m; a.n = an.n; a.t_free = an.t; a.tl = an.tl; a.npsd = an.npsd;
  a.seg_ptr = d.seg_ptr; a.seg_col = d.seg_col; a.seg_val = d.seg_val;
  a.segpos = d.segpos; a.xis = d.xis; a.zs = d.zs;
  a.low_col = d.low_col; a.lr_ptr = d.lr_ptr; a.lr_idx = d.lr_idx; a.lr_col = d.lr_col; a.lr_val = d.lr_val;
  {
    int mx = 0;
    for (int r = 0; r < an.m; ++r) mx = std::max(mx, an.lr_ptr[r + 1] - an.lr_ptr[r]);
    a.row_lanes = mx >= 16 ? 8 : 1;
    a.fuse_low = (an.tl <= FUSE_LOW_TL && an.lr_ptr[an.m] <= FUSE_LOW_NNZ && !getenv("SOSADMM_NO_FUSE_LOW")) ? 1 : 0;
  }
  a.lc_ptr = d.lc_ptr; a.lc_row = d.lc_row; a.lc_val = d.lc_val;
  a.c_low = d.c_low; a.h1_low = d.h1_low; a.beta_low = d.beta_low; a.Kinv = d.Kinv;
  a.ldk = an.tl + (an.tl & 1);
  a.empty_cols = d.empty_cols; a.n_empty = (int)an.empty_cols.size();
  a.b = d.b; a.Pinv = d.Pinv; a.h2 = d.h2;
  a.denom = denom; a.bh2 = bh; a.nb = std::sqrt(nb); a.nc = std::sqrt(nc);
  a.code = d.code; a.aval = d.aval;
  a.xi = d.xi; a.z = d.z; a.y = d.y; a.s = d.s; a.st = d.st; a.is = d.is;
  a.x = d.x; a.uhat2 = d.uhat2; a.yt = d.yt; a.zt = d.zt; a.ulow = d.ulow; a.aty = d.aty; a.kpart = d.kpart;
  a.part = d.part; a.gather_blocks = c->gather_blocks; a.asvec = d.asvec;
  a.hist = d.hist;
  a.nblk = an.nblk; a.blk_col = d.blk_col; a.blk_N = d.blk_N; a.blk_mat = d.blk_mat; a.mats = d.mats;
  a.cta_blk = d.cta_blk; a.cta_q0 = d.cta_q0; a.pos_ctas = (int)an.cta_blk.size();
  c->d_tmp = d.tmp;
  a.side = nullptr;
  a.shard_scal = sp.sharded ? d.shbuf + 2 * (size_t)an.m : nullptr;
  c->nb_low = low_blocks(an);
  c->sh.colown = d.colown;
  c->sh.buf = d.shbuf;
  c->sh.part = d.shpart;
  c->sh.nparts = std::max(c->gather_blocks, c->nb_low);
  c->sh.world = sp.world;
  c->sh.rank = sp.rank;
  c->dp = d;  // kept for the peer-mode wiring (sosadmm_debug_group_link_peers, IPC exchange)
  JacobiArgs& ja = c->ja;
  ja.mats = d.mats; ja.blk_mat = d.blk_mat; ja.blk_N = d.blk_N; ja.small_blk = d.small_blk;
  ja.st = d.st; ja.is = d.is; ja.check_state = 1;
  ja.vp = d.jvp; ja.blk_vp = d.blk_vp; ja.warm = 1;
  ja.blocked = 1;  // SOSADMM_JACOBI_BLOCKED=0: the elementwise round update (A/B runs)
  if (const char* jb = getenv("SOSADMM_JACOBI_BLOCKED")) ja.blocked = atoi(jb) != 0;
  if (!an.small_blk.empty()) {
    // the attribute is per kernel and process-wide: set the template's bound, never a per-context
    // size (a later context with smaller blocks would otherwise shrink it under an earlier one)
    CK_CTX(c, cudaFuncSetAttribute(jacobi_kernel(an.max_small_N, c->ja.blocked), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)jacobi_smem_bytes(an.max_small_N <= 32 ? 32 : JAC_MAXN)));
  }
  {
    std::string lmsg;
    if (large_eig_init(c->le, an.blk_N, an.blk_mat, an.large_blk, d.mats, large_base, d.st, d.is, s, lmsg,
                       warm_enabled()) != 0) {
      c->err = SOSADMM_E_CUDA;
      c->msg = "large-block eigensolver setup: " + lmsg;
      return c->err;
    }
  }
  c->aa.side = c->le.side;
  // host mirror of the structure
  c->row_of.assign(an.n, -2);
  for (int j = an.t; j < an.n; ++j)
    if (an.code[j] >= -1) c->row_of[j] = an.code[j];
  if (!an.large_blk.empty() && an.large_blk.size() <= 8) {
    const int naux = 1 + 3 * (int)an.large_blk.size();
    for (int q = 0; q < naux; ++q) CK_CTX(c, cudaStreamCreateWithFlags(&c->aux[q], cudaStreamNonBlocking));
    for (size_t q = 0; q < an.large_blk.size(); ++q) {
      CK_CTX(c, cudaStreamCreateWithFlags(&c->body[q], cudaStreamNonBlocking));
      CK_CTX(c, cudaStreamCreateWithFlags(&c->nest[q], cudaStreamNonBlocking));
      CK_CTX(c, cudaStreamCreateWithFlags(&c->pre[q], cudaStreamNonBlocking));
      CK_CTX(c, cudaEventCreateWithFlags(&c->ev_pre[q], cudaEventDisableTiming));
    }
    CK_CTX(c, cudaEventCreateWithFlags(&c->ev_pre0, cudaEventDisableTiming));
    if (const char* ep = getenv("SOSADMM_EARLY_PRED")) c->no_early_pred_env = atoi(ep) == 0;
    c->early_pred = !c->no_early_pred_env;
    CK_CTX(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK_CTX(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    for (int q = 0; q < 8 * (int)an.large_blk.size(); ++q)
      CK_CTX(c, cudaEventCreateWithFlags(&c->ev_blk[q], cudaEventDisableTiming));
    c->aux_ok = true;
  }
  c->launches = count_launches(c);
  CK_CTX(c, cudaStreamSynchronize(s));
  {  // f4 peer mode on real ranks (opt-in: SOSADMM_ALLREDUCE=peer; NCCL otherwise)
    const char* env = getenv("SOSADMM_ALLREDUCE");
    if (sp.sharded && !sp.emulated && env && std::string(env) == "peer") {
      if ((size_t)an.n * sizeof(double) < (sp.world + 1) * sizeof(PeerRec)) {
        c->err = SOSADMM_E_ARG;
        c->msg = "peer mode: problem too small for the handle exchange scratch";
        return c->err;
      }
      if (peer_setup_ipc(c)) return c->err;
      c->launches = count_launches(c);
    }
  }
  return SOSADMM_OK;
}

sosadmm_err sosadmm_setup(const sosadmm_problem* prob, const sosadmm_settings* settings, sosadmm_ctx** out) {
  return setup_impl(prob, settings, ShardSpec(), nullptr, out);
}

sosadmm_err sosadmm_nccl_unique_id(void* id) {
  if (!id) return SOSADMM_E_ARG;
  if (!nccl().ok) return SOSADMM_E_NCCL;
  ncclUniqueId u;
  if (nccl().getUniqueId(&u) != ncclSuccess) return SOSADMM_E_NCCL;
  std::memcpy(id, &u, sizeof(u));
  return SOSADMM_OK;
}

sosadmm_err sosadmm_setup_sharded(const sosadmm_problem* prob, const sosadmm_settings* settings, const void* nccl_id,
                                  int32_t rank, int32_t world, const int32_t* block_owner, sosadmm_ctx** out) {
  if (!out) return SOSADMM_E_ARG;
  if (!nccl_id || world < 1 || rank < 0 || rank >= world || !block_owner) {
    *out = nullptr;
    return SOSADMM_E_ARG;
  }
  ShardSpec sp;
  sp.rank = rank;
  sp.world = world;
  sp.block_owner = block_owner;
  sp.sharded = true;
  return setup_impl(prob, settings, sp, nccl_id, out);
}

static sosadmm_err build_graph(sosadmm_ctx* c) {
  if (c->graph) return SOSADMM_OK;
  for (int attempt = 0; attempt < 3; ++attempt) {
    CK_CTX(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const sosadmm_err le = launch_iteration(c, 1, nullptr);
    cudaGraph_t g = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(c->stream, &g);
    cudaError_t ie = cudaErrorUnknown;
    if (le == SOSADMM_OK && ee == cudaSuccess) {
      ie = cudaGraphInstantiate(&c->graph, g, 0);
      if (ie == cudaSuccess) {
        c->graph_raw = g;
        return SOSADMM_OK;
      }
      c->graph = nullptr;
    }
    if (g) cudaGraphDestroy(g);  // a failed capture (e.g. ncclAllReduce) is never instantiated
    bool warm = false;
    for (auto& lb : c->le.blocks) warm |= lb.warm;
    if (attempt == 0 && warm && c->nest_ok && !(le != SOSADMM_OK && c->err == SOSADMM_E_NCCL)) {
      // nested conditional nodes rejected here: capture again with the cluster kernels unconditional
      c->nest_ok = false;
      c->msg = std::string("nested conditional nodes disabled (graph capture: ") +
               cudaGetErrorString(ee != cudaSuccess ? ee : ie) + ")";
      c->err = SOSADMM_OK;
      (void)cudaGetLastError();
      continue;
    }
    if (attempt <= 1 && warm && !(le != SOSADMM_OK && c->err == SOSADMM_E_NCCL)) {
      // the warm mode's conditional nodes could not be captured / instantiated here: cold path every
      // iteration (still correct: the D&C root then forms every eigenvector), recorded in the message
      for (auto& lb : c->le.blocks) lb.warm = false;
      c->msg = std::string("warm start disabled (graph capture: ") + cudaGetErrorString(ee != cudaSuccess ? ee : ie) + ")";
      c->err = SOSADMM_OK;
      (void)cudaGetLastError();
      c->launches = count_launches(c);
      continue;
    }
    if (le != SOSADMM_OK) return c->err = le;
    c->err = SOSADMM_E_CUDA;
    c->msg = std::string("graph capture: ") + cudaGetErrorString(ee != cudaSuccess ? ee : ie);
    return c->err;
  }
  return c->err;
}

// Enqueue up to k graph replays in chunks (8, 16, ... 128).  After each chunk the device state is copied
// to pinned host memory behind an event; the host keeps two chunks in flight, and once a finished chunk
// shows the latched `done` (or a non-finite iterate) it stops enqueueing.  Replays after termination are
// no-ops on the device (every kernel early-exits), so the iterates are exactly those of k plain replays;
// this only bounds the no-op tail to two chunks instead of k − k_stop replays (≈ 40 µs each).  The stop
// decision depends only on the device's replicated state at chunk boundaries, so every rank of a sharded
// run enqueues the same replays (and the same in-graph allreduces).
static sosadmm_err enqueue_replays(sosadmm_ctx* c, int64_t k) {
  if (!c->h_poll) {
    CK_CTX(c, cudaHostAlloc(reinterpret_cast<void**>(&c->h_poll), 2 * sizeof(DevState), cudaHostAllocDefault));
    for (auto& e : c->ev_poll) CK_CTX(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  int64_t done = 0, chunk = 8;
  int j = 0;  // chunks enqueued
  while (done < k) {
    const int64_t n = std::min(chunk, k - done);
    for (int64_t i = 0; i < n; ++i) CK_CTX(c, cudaGraphLaunch(c->graph, c->stream));
    done += n;
    chunk = std::min<int64_t>(chunk * 2, 128);
    if (done >= k) break;
    const int slot = j & 1;
    CK_CTX(c, cudaMemcpyAsync(&c->h_poll[slot], c->aa.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    CK_CTX(c, cudaEventRecord(c->ev_poll[slot], c->stream));
    if (j >= 1) {  // wait for the previous chunk (the current one keeps the GPU busy meanwhile)
      CK_CTX(c, cudaEventSynchronize(c->ev_poll[slot ^ 1]));
      const DevState& st = c->h_poll[slot ^ 1];
      if (st.done || st.nonfinite) break;
    }
    ++j;
  }
  return check_async(c);
}

sosadmm_err sosadmm_iterate(sosadmm_ctx* c, int64_t k, sosadmm_info* out) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  if (k < 0) return SOSADMM_E_ARG;
  CK_CTX(c, cudaSetDevice(c->device));
  if (build_graph(c)) return c->err;
  if (enqueue_replays(c, k)) return c->err;
  launch_iteration(c, 0, nullptr);  // residual check of the final iterate
  if (check_async(c)) return c->err;
  return read_info(c, out);
}

sosadmm_err sosadmm_iterate_async(sosadmm_ctx* c, int64_t k) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  if (k < 0) return SOSADMM_E_ARG;
  CK_CTX(c, cudaSetDevice(c->device));
  if (build_graph(c)) return c->err;
  for (int64_t i = 0; i < k; ++i) CK_CTX(c, cudaGraphLaunch(c->graph, c->stream));
  return check_async(c);
}

sosadmm_err sosadmm_set_shared_gpu(sosadmm_ctx* c, int shared) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  const bool want = shared == 0 && !c->no_early_pred_env;
  if (want == c->early_pred) return SOSADMM_OK;
  CK_CTX(c, cudaSetDevice(c->device));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  c->early_pred = want;
  if (c->graph) {  // rebuilt by the next iterate call
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
    if (c->graph_raw) cudaGraphDestroy(c->graph_raw);
    c->graph_raw = nullptr;
  }
  return SOSADMM_OK;
}

sosadmm_err sosadmm_iterate_profiled(sosadmm_ctx* c, int64_t k, sosadmm_info* out, double* ms_phase) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  CK_CTX(c, cudaSetDevice(c->device));
  constexpr int NE = SOSADMM_NPHASE + 1;
  std::vector<cudaEvent_t> ev((size_t)NE * std::max<int64_t>(k, 1));
  for (auto& e : ev) CK_CTX(c, cudaEventCreate(&e));
  for (int64_t i = 0; i < k; ++i)
    if (launch_iteration(c, 1, &ev[NE * i])) return c->err;
  launch_iteration(c, 0, nullptr);
  if (check_async(c)) return c->err;
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  double acc[SOSADMM_NPHASE] = {};
  for (int64_t i = 0; i < k; ++i)
    for (int p = 0; p < SOSADMM_NPHASE; ++p) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[NE * i + p], ev[NE * i + p + 1]);
      acc[p] += ms;
    }
  for (auto& e : ev) cudaEventDestroy(e);
  if (ms_phase)
    for (int p = 0; p < SOSADMM_NPHASE; ++p) ms_phase[p] += acc[p];
  return read_info(c, out);
}

sosadmm_err sosadmm_get_info(sosadmm_ctx* c, sosadmm_info* out) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  CK_CTX(c, cudaSetDevice(c->device));
  launch_iteration(c, 0, nullptr);
  if (check_async(c)) return c->err;
  return read_info(c, out);
}

sosadmm_err sosadmm_get_iterate(sosadmm_ctx* c, double* xi, double* y, double* z, double* s, double* tau,
                                double* kappa, int64_t* iter) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  CK_CTX(c, cudaSetDevice(c->device));
  const AffineArgs& a = c->aa;
  if (c->sp.sharded) {  // collective: assemble the owned entries of every rank (exact: x + 0 = x)
    for (int v = 0; v < 2; ++v) {
      double* host = v == 0 ? xi : z;
      const double* src = v == 0 ? a.xi : a.z;
      k_mask_owned<<<(a.n + 255) / 256, 256, 0, c->stream>>>(src, c->sh.colown, c->d_tmp, a.n);
      const ncclResult_t nr = nccl().allReduce(c->d_tmp, c->d_tmp, (size_t)a.n, ncclFloat64, ncclSum, c->comm,
                                               c->stream);
      if (nr != ncclSuccess) {
        c->err = SOSADMM_E_NCCL;
        c->msg = std::string("ncclAllReduce: ") + nccl().getErrorString(nr);
        return c->err;
      }
      if (host) CK_CTX(c, cudaMemcpyAsync(host, c->d_tmp, sizeof(double) * a.n, cudaMemcpyDeviceToHost, c->stream));
      CK_CTX(c, cudaStreamSynchronize(c->stream));
    }
    xi = nullptr;
    z = nullptr;
  }
  if (xi) CK_CTX(c, cudaMemcpyAsync(xi, a.xi, sizeof(double) * a.n, cudaMemcpyDeviceToHost, c->stream));
  if (z) CK_CTX(c, cudaMemcpyAsync(z, a.z, sizeof(double) * a.n, cudaMemcpyDeviceToHost, c->stream));
  if (y) CK_CTX(c, cudaMemcpyAsync(y, a.y, sizeof(double) * a.m, cudaMemcpyDeviceToHost, c->stream));
  if (s) CK_CTX(c, cudaMemcpyAsync(s, a.s, sizeof(double) * a.m, cudaMemcpyDeviceToHost, c->stream));
  DevState st;
  CK_CTX(c, cudaMemcpyAsync(&st, a.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  if (tau) *tau = st.tau;
  if (kappa) *kappa = st.kappa;
  if (iter) *iter = st.iter;
  return SOSADMM_OK;
}

sosadmm_err sosadmm_set_iterate(sosadmm_ctx* c, const double* xi, const double* y, const double* z,
                                const double* s, double tau, double kappa, int64_t iter) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  if (!xi || !y || !z) return SOSADMM_E_ARG;
  CK_CTX(c, cudaSetDevice(c->device));
  const AffineArgs& a = c->aa;
  CK_CTX(c, cudaMemcpyAsync(a.xi, xi, sizeof(double) * a.n, cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaMemcpyAsync(a.z, z, sizeof(double) * a.n, cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaMemcpyAsync(a.y, y, sizeof(double) * a.m, cudaMemcpyHostToDevice, c->stream));
  if (s) CK_CTX(c, cudaMemcpyAsync(a.s, s, sizeof(double) * a.m, cudaMemcpyHostToDevice, c->stream));
  else CK_CTX(c, cudaMemsetAsync(a.s, 0, sizeof(double) * a.m, c->stream));
  const int nseg = (int)c->an.seg_col.size();
  if (nseg > 0) k_seg_copy<<<(nseg + 255) / 256, 256, 0, c->stream>>>(a);
  DevState st{};
  st.tau = tau;
  st.kappa = kappa;
  st.iter = iter;
  st.max_iters = c->max_iters;
  st.tol = c->tol;
  st.res_pri = st.res_dual = st.res_gap = INFINITY;
  CK_CTX(c, cudaMemcpyAsync(a.st, &st, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  return SOSADMM_OK;
}

sosadmm_err sosadmm_get_structure(sosadmm_ctx* c, int32_t* row_of, double* D, int64_t* t_low) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  if (row_of) std::memcpy(row_of, c->row_of.data(), sizeof(int32_t) * c->an.n);
  if (D) std::memcpy(D, c->an.D.data(), sizeof(double) * c->an.m);
  if (t_low) *t_low = c->an.tl;
  return SOSADMM_OK;
}

// Unit entry point: u_hat = (I + Q)^{-1} w through the production kernels (mode 2 of k_tphase).
sosadmm_err sosadmm_project_affine(sosadmm_ctx* c, const double* w1, const double* w2, double w3, double* u1,
                                   double* u2, double* u3) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  if (c->sp.sharded) return SOSADMM_E_ARG;  // unit entry points are single-GPU only
  CK_CTX(c, cudaSetDevice(c->device));
  const AffineArgs& a = c->aa;
  const int n = a.n, m = a.m;
  // save the iterate, load (xi, y, tau) = w and (z, s, kappa) = 0
  std::vector<double> sxi(n), sz(n), sy(m), ss(m);
  double stau, skap;
  int64_t sit;
  if (sosadmm_get_iterate(c, sxi.data(), sy.data(), sz.data(), ss.data(), &stau, &skap, &sit)) return c->err;
  // the whole device state (termination latch, status, residuals) is restored afterwards, not rebuilt
  DevState sst;
  IterScal sis;
  CK_CTX(c, cudaMemcpyAsync(&sst, a.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  CK_CTX(c, cudaMemcpyAsync(&sis, a.is, sizeof(IterScal), cudaMemcpyDeviceToHost, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  std::vector<double> zero_n(n, 0.0), zero_m(m, 0.0);
  if (sosadmm_set_iterate(c, w1, w2, zero_n.data(), zero_m.data(), w3, 0.0, 0)) return c->err;
  cudaStream_t s = c->stream;
  k_gather<<<c->gather_blocks, GATHER_NT, 0, s>>>(a);
  launch_low_tphase(a, s, 2);
  launch_rowupdate(a, s, 0);
  if (a.pos_ctas > 0) k_scatter<<<a.pos_ctas, POS_NT, 0, s>>>(a, 1);
  if (check_async(c)) return c->err;
  std::vector<double> asv(std::max(a.npsd, 1)), ulow(std::max(a.tl, 1));
  IterScal is;
  CK_CTX(c, cudaMemcpyAsync(u2, a.uhat2, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
  if (a.npsd) CK_CTX(c, cudaMemcpyAsync(asv.data(), a.asvec, sizeof(double) * a.npsd, cudaMemcpyDeviceToHost, s));
  if (a.tl) CK_CTX(c, cudaMemcpyAsync(ulow.data(), a.ulow, sizeof(double) * a.tl, cudaMemcpyDeviceToHost, s));
  CK_CTX(c, cudaMemcpyAsync(&is, a.is, sizeof(IterScal), cudaMemcpyDeviceToHost, s));
  CK_CTX(c, cudaStreamSynchronize(s));
  for (int j = 0; j < c->an.t; ++j) u1[j] = 0.0;
  for (int j = c->an.t; j < n; ++j) u1[j] = asv[j - c->an.t];
  for (int jl = 0; jl < a.tl; ++jl) u1[c->an.low_col[jl]] = ulow[jl];
  *u3 = is.u3;
  CK_CTX(c, cudaMemcpyAsync(a.xi, sxi.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemcpyAsync(a.z, sz.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  if (!c->an.seg_col.empty()) k_seg_copy<<<((int)c->an.seg_col.size() + 255) / 256, 256, 0, s>>>(a);
  CK_CTX(c, cudaMemcpyAsync(a.y, sy.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemcpyAsync(a.s, ss.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemcpyAsync(a.st, &sst, sizeof(DevState), cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemcpyAsync(a.is, &sis, sizeof(IterScal), cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaStreamSynchronize(s));
  return SOSADMM_OK;
}

// Unit entry point: Pi_{S+} of one block given in svec coordinates.
sosadmm_err sosadmm_project_psd(sosadmm_ctx* c, int32_t block, const double* a_svec, double* out_svec) {
  if (!c) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  if (c->sp.sharded) return SOSADMM_E_ARG;  // unit entry points are single-GPU only
  if (block < 0 || block >= c->an.nblk) return SOSADMM_E_ARG;
  CK_CTX(c, cudaSetDevice(c->device));
  const AffineArgs& a = c->aa;
  const int N = c->an.blk_N[block];
  const long long L = (long long)N * (N + 1) / 2;
  const long long off = c->an.blk_col[block] - c->an.t;
  cudaStream_t s = c->stream;
  DevState sst;
  IterScal sis;
  CK_CTX(c, cudaMemcpyAsync(&sst, a.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CK_CTX(c, cudaMemcpyAsync(&sis, a.is, sizeof(IterScal), cudaMemcpyDeviceToHost, s));
  CK_CTX(c, cudaStreamSynchronize(s));
  DevState st = sst;
  st.done = 0;
  IterScal is = sis;
  is.proceed = 1;
  CK_CTX(c, cudaMemcpyAsync(a.st, &st, sizeof(DevState), cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemcpyAsync(a.is, &is, sizeof(IterScal), cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemcpyAsync(c->d_tmp + off, a_svec, sizeof(double) * L, cudaMemcpyHostToDevice, s));
  k_unpack_block<<<(int)((L + 255) / 256), 256, 0, s>>>(a, block, c->d_tmp + off);
  if (!c->an.small_blk.empty())
    jacobi_kernel(c->an.max_small_N, c->ja.blocked)<<<(int)c->an.small_blk.size(), jacobi_threads(c->an.max_small_N), jacobi_smem_bytes(c->an.max_small_N),
                                         s>>>(c->ja);
  if (!c->an.large_blk.empty()) large_eig_launch(c->le, s, true);
  if (a.pos_ctas > 0) k_pack<<<a.pos_ctas, POS_NT, 0, s>>>(a, c->d_tmp, 0);
  if (check_async(c)) return c->err;
  CK_CTX(c, cudaMemcpyAsync(out_svec, c->d_tmp + off, sizeof(double) * L, cudaMemcpyDeviceToHost, s));
  CK_CTX(c, cudaMemcpyAsync(a.st, &sst, sizeof(DevState), cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaMemcpyAsync(a.is, &sis, sizeof(IterScal), cudaMemcpyHostToDevice, s));
  CK_CTX(c, cudaStreamSynchronize(s));
  return SOSADMM_OK;
}

int64_t sosadmm_launches_per_iter(const sosadmm_ctx* c) { return c ? c->launches : 0; }

sosadmm_err sosadmm_psd_work(sosadmm_ctx* c, double* work, int32_t* nblocks) {
  if (!c || !nblocks) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  CK_CTX(c, cudaSetDevice(c->device));
  const int nb = (int)c->le.blocks.size();
  if (work)
    for (int b = 0; b < std::min(nb, *nblocks); ++b)
      if (large_block_work(c->le.blocks[b], c->stream, work + 6 * b)) {
        c->err = SOSADMM_E_CUDA;
        c->msg = "sosadmm_psd_work: device read failed";
        return c->err;
      }
  *nblocks = nb;
  return SOSADMM_OK;
}

sosadmm_err sosadmm_residual_history(sosadmm_ctx* c, double* out, int32_t* count) {
  if (!c || !out || !count) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  CK_CTX(c, cudaSetDevice(c->device));
  const int n = std::min<int>(*count, SOS_HIST);
  std::vector<double> h((size_t)5 * SOS_HIST);
  CK_CTX(c, cudaMemcpyAsync(h.data(), c->dp.hist, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c->stream));
  CK_CTX(c, cudaStreamSynchronize(c->stream));
  // newest first: u^{k-1} was checked during iteration k (k = the device's iteration count), walking back
  DevState hs{};
  CK_CTX(c, cudaMemcpy(&hs, c->aa.st, sizeof(hs), cudaMemcpyDeviceToHost));
  const long long best = hs.iter - 1;
  const int slot = best >= 0 ? (int)(best % SOS_HIST) : 0;
  int k = 0;
  for (; k < n && best >= 0; ++k) {
    const int q = ((slot - k) % SOS_HIST + SOS_HIST) % SOS_HIST;
    if (h[5 * q] < 0 || (long long)h[5 * q] != best - k) break;
    for (int f = 0; f < 5; ++f) out[5 * k + f] = h[5 * q + f];
  }
  *count = k;
  return SOSADMM_OK;
}

sosadmm_err sosadmm_warm_stats(sosadmm_ctx* c, int64_t* stats, int32_t* nblocks) {
  if (!c || !nblocks) return SOSADMM_E_ARG;
  if (c->err) return c->err;
  CK_CTX(c, cudaSetDevice(c->device));
  const int nb = (int)c->le.blocks.size();
  if (stats)
    for (int b = 0; b < std::min(nb, *nblocks); ++b) {
      const LargeBlock& lb = c->le.blocks[b];
      WarmState h{};
      int sel[3] = {0, 0, 0};
      CK_CTX(c, cudaMemcpyAsync(&h, lb.wa.ws, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
      CK_CTX(c, cudaMemcpyAsync(sel, lb.warm ? lb.wa.sel : lb.sel, sizeof(sel), cudaMemcpyDeviceToHost, c->stream));
      CK_CTX(c, cudaStreamSynchronize(c->stream));
      int64_t* o = stats + 10 * b;
      o[0] = h.n_warm;
      o[1] = h.n_cold;
      o[2] = h.n_steps;
      o[3] = h.n_fail;
      o[4] = lb.warm ? 1 : 0;
      o[5] = sel[0];
      o[6] = lb.N;
      o[7] = h.step;
      o[8] = h.n_seed;
      o[9] = h.why;
    }
  *nblocks = nb;
  return SOSADMM_OK;
}

void sosadmm_destroy(sosadmm_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->graph_raw) cudaGraphDestroy(c->graph_raw);
  large_eig_free(c->le);
  if (c->comm) nccl().commDestroy(c->comm);
  for (auto& a : c->aux)
    if (a) cudaStreamDestroy(a);
  for (auto& a : c->body)
    if (a) cudaStreamDestroy(a);
  for (auto& a : c->nest)
    if (a) cudaStreamDestroy(a);
  for (auto& a : c->pre)
    if (a) cudaStreamDestroy(a);
  for (auto& e : c->ev_pre)
    if (e) cudaEventDestroy(e);
  if (c->ev_pre0) cudaEventDestroy(c->ev_pre0);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (auto& e : c->ev_poll)
    if (e) cudaEventDestroy(e);
  if (c->h_poll) cudaFreeHost(c->h_poll);
  for (auto& e : c->ev_blk)
    if (e) cudaEventDestroy(e);
  for (void* pb : c->ipc_open) cudaIpcCloseMemHandle(pb);
  if (c->own_mem) cudaFree(c->own_mem);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* sosadmm_strerror(sosadmm_err e) {
  switch (e) {
    case SOSADMM_OK: return "ok";
    case SOSADMM_E_ARG: return "invalid argument";
    case SOSADMM_E_STRUCT: return "unsupported structure";
    case SOSADMM_E_FACTOR: return "factorisation failed";
    case SOSADMM_E_CUDA: return "CUDA error";
    case SOSADMM_E_NCCL: return "NCCL error";
    case SOSADMM_E_NONFINITE: return "non-finite iterate";
    case SOSADMM_E_OOM: return "out of memory";
  }
  return "unknown error";
}

const char* sosadmm_last_error_message(const sosadmm_ctx* c) { return c ? c->msg.c_str() : "null context"; }

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// Stage-level debug entry points (include/sosadmm_debug.h).
#include "../../include/sosadmm_debug.h"

namespace {
struct DebugLarge {
  LargeEig le;
  DevState* st = nullptr;
  IterScal* is = nullptr;
  double* mats = nullptr;
  char* base = nullptr;
  cudaStream_t s = nullptr;
  int init(int N, bool warm = false) {
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) return -4;
    std::vector<int> blk_N{N}, large{0};
    std::vector<long long> blk_mat{0};
    const size_t bytes = large_eig_bytes(blk_N, large);
    if (cudaMalloc(&base, bytes + 1024)) return -7;
    if (cudaMalloc(&mats, sizeof(double) * N * N)) return -7;
    if (cudaMalloc(&st, sizeof(DevState))) return -7;
    if (cudaMalloc(&is, sizeof(IterScal))) return -7;
    cudaMemset(st, 0, sizeof(DevState));
    IterScal h{};
    h.proceed = 1;
    cudaMemcpy(is, &h, sizeof(h), cudaMemcpyHostToDevice);
    std::string msg;
    if (large_eig_init(le, blk_N, blk_mat, large, mats, base, st, is, s, msg, warm)) return -4;
    return cudaStreamSynchronize(s) ? -4 : 0;
  }
  ~DebugLarge() {
    if (s) cudaStreamSynchronize(s);
    cudaFree(base);
    cudaFree(mats);
    cudaFree(st);
    cudaFree(is);
    if (s) cudaStreamDestroy(s);
  }
};
}  // namespace

extern "C" int sosadmm_debug_gemm(int M, int N, int K, const double* A, const double* B, int transB, double* C) {
  double *dA, *dB, *dC;
  GemmDesc* dg;
  if (cudaMalloc(&dA, 8ull * M * std::max(K, 1)) || cudaMalloc(&dB, 8ull * N * std::max(K, 1)) ||
      cudaMalloc(&dC, 8ull * M * N) || cudaMalloc(&dg, sizeof(GemmDesc)))
    return -7;
  cudaMemcpy(dA, A, 8ull * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B, 8ull * N * K, cudaMemcpyHostToDevice);
  GemmDesc g{};
  g.A = dA; g.lda = M; g.B = dB; g.ldb = transB ? N : K; g.transB = transB;
  g.C = dC; g.ldc = M; g.M = M; g.N = N; g.K = K; g.alpha = 1.0; g.beta = 0.0;
  cudaMemcpy(dg, &g, sizeof(g), cudaMemcpyHostToDevice);
  dim3 gr((M + GM_BM - 1) / GM_BM, (N + GM_BN - 1) / GM_BN, 1);
  k_gemm_f64<<<gr, GM_NT>>>(dg, nullptr, nullptr, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) cudaMemcpy(C, dC, 8ull * M * N, cudaMemcpyDeviceToHost);
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dg);
  return e == cudaSuccess ? 0 : -4;
}

// C (M x N) = op(A) B with the warm-path DMMA GEMM (dgemm.cuh): A is M x K (transA = 0) or K x M
// (transA = 1), B is K x N, all column-major host arrays; upper = 1 fills only the tiles meeting the upper
// triangle (the other entries of C are left 0).  reps > 0: *ms = mean CUDA-event time of reps launches.
extern "C" int sosadmm_debug_dgemm(int M, int N, int K, const double* A, int transA, int upper, const double* B,
                                   double* C, int variant, int reps, float* ms) {
  if (variant < 0) variant = DG_DEFAULT;
  if (variant >= DG_NVAR) return -1;
  const int ar = transA ? K : M, ac = transA ? M : K;  // stored A: ar x ac
  const int lda = (ar + 1) & ~1, ldb = (K + 1) & ~1, ldc = (M + 1) & ~1;
  double *dA, *dB, *dC;
  DgemmDesc* dg;
  if (cudaMalloc(&dA, 8ull * lda * std::max(ac, 1)) || cudaMalloc(&dB, 8ull * ldb * std::max(N, 1)) ||
      cudaMalloc(&dC, 8ull * ldc * std::max(N, 1)) || cudaMalloc(&dg, sizeof(DgemmDesc)))
    return -7;
  cudaMemset(dA, 0, 8ull * lda * std::max(ac, 1));
  cudaMemset(dB, 0, 8ull * ldb * std::max(N, 1));
  cudaMemset(dC, 0, 8ull * ldc * std::max(N, 1));
  cudaMemcpy2D(dA, 8ull * lda, A, 8ull * ar, 8ull * ar, ac, cudaMemcpyHostToDevice);
  cudaMemcpy2D(dB, 8ull * ldb, B, 8ull * K, 8ull * K, N, cudaMemcpyHostToDevice);
  DgemmDesc g{};
  g.A = dA; g.lda = lda; g.B = dB; g.ldb = ldb; g.C = dC; g.ldc = ldc;
  g.M = M; g.N = N; g.K = K; g.transA = transA; g.upper = upper; g.alpha = 1.0; g.beta = 0.0;
  cudaMemcpy(dg, &g, sizeof(g), cudaMemcpyHostToDevice);
  dgemm_prepare();
  dgemm_launch(variant, dg, 1, M, N, nullptr, nullptr, nullptr, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess && reps > 0 && ms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) dgemm_launch(variant, dg, 1, M, N, nullptr, nullptr, nullptr, 0);
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    *ms = t / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (e == cudaSuccess) e = cudaMemcpy2D(C, 8ull * M, dC, 8ull * ldc, 8ull * M, N, cudaMemcpyDeviceToHost);
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dg);
  return e == cudaSuccess ? 0 : -4;
}

// Warm-started projection of one block (tests/test_gpu_warm.py): a0 through the cold path (which seeds the
// eigenvectors), then a1 through the warm refinement (cold fallback if it does not converge).  out0 / out1:
// Pi_{S+}(a0), Pi_{S+}(a1), full N x N column-major; stats = [status of the a1 projection (1 warm, 2 cold),
// S evaluations, clusters of the last step, r, side, refinement updates].
extern "C" int sosadmm_debug_warm_project(int N, const double* a0, const double* a1, double* out0, double* out1,
                                          int* stats) {
  if (N <= 64 || N > 1280) return -1;
  DebugLarge dl;
  int rc = dl.init(N, true);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  for (int pass = 0; pass < 2; ++pass) {
    const double* a = pass ? a1 : a0;
    double* out = pass ? out1 : out0;
    cudaMemcpyAsync(dl.mats, a, 8ull * N * N, cudaMemcpyHostToDevice, dl.s);
    if (large_block_warm_ungraphed(dl.le, lb, dl.s, nullptr) != cudaSuccess) return -4;
    std::vector<double> M((size_t)N * N);
    int side = 0;
    cudaMemcpyAsync(M.data(), dl.mats, 8ull * N * N, cudaMemcpyDeviceToHost, dl.s);
    cudaMemcpyAsync(&side, dl.le.side, 4, cudaMemcpyDeviceToHost, dl.s);
    WarmState h{};
    int sel[3] = {0, 0, 0};
    cudaMemcpyAsync(&h, lb.wa.ws, sizeof(h), cudaMemcpyDeviceToHost, dl.s);
    cudaMemcpyAsync(sel, h.status == 1 ? lb.wa.sel : lb.sel, sizeof(sel), cudaMemcpyDeviceToHost, dl.s);
    if (cudaStreamSynchronize(dl.s) != cudaSuccess) return -4;
    // the block holds the upper triangle of Pi(a) (side 0) or Pi(-a) (side 1: Pi(a) = a + Pi(-a))
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i) {
        const double m = i <= j ? M[(size_t)j * N + i] : M[(size_t)i * N + j];
        out[(size_t)j * N + i] = side ? a[(size_t)j * N + i] + m : m;
      }
    if (pass == 1 && stats) {
      stats[0] = h.status;
      stats[1] = h.step;
      stats[2] = h.ncl;
      stats[3] = sel[0];
      stats[4] = side;
      stats[5] = (int)h.n_steps;
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

// Diagnostics: the warm refinement's per-evaluation trace of the last iteration of large block b
// (out: 4 x WM_MAXS + 8 doubles = coupling / ||a||_F, projected side's orthonormality defect / N, Gershgorin
// bound / ||a||_F, [evaluations, clusters at step 0, predicted start, status, why, backoff, fails, largest
// cluster], the other side's orthonormality defect / N);
// -1 for a bad block index.
extern "C" int sosadmm_debug_warm_trace(sosadmm_ctx* c, int b, double* out) {
  if (!c || !out || b < 0 || b >= (int)c->le.blocks.size()) return -1;
  const LargeBlock& lb = c->le.blocks[b];
  WarmState h{};
  if (cudaMemcpyAsync(&h, lb.wa.ws, sizeof(h), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return -4;
  for (int j = 0; j < WM_MAXS; ++j) {
    out[j] = h.tr_eta[j];
    out[WM_MAXS + j] = h.tr_rn[j];
    out[2 * WM_MAXS + j] = h.tr_g[j];
  }
  const double tail[8] = {(double)h.step, (double)h.cl0, (double)h.pred, (double)h.status, (double)h.why,
                          (double)h.backoff, (double)h.fails, (double)h.maxcl};
  for (int j = 0; j < 8; ++j) out[3 * WM_MAXS + j] = tail[j];
  for (int j = 0; j < WM_MAXS; ++j) out[3 * WM_MAXS + 8 + j] = h.tr_ro[j];
  return 0;
}

extern "C" int sosadmm_debug_tridiag(int N, const double* A, double* d, double* e, double* tau, double* V) {
  if (N < 3) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  lb.two = false;  // the one-cluster BLAS-2 kernel (k_tridiag)
  cudaMemcpyAsync(lb.M, A, 8ull * N * N, cudaMemcpyHostToDevice, dl.s);
  cudaMemsetAsync(lb.V, 0, 8ull * N * N, dl.s);
  large_block_tridiag(dl.le, lb, dl.s, false);
  cudaError_t err = cudaStreamSynchronize(dl.s);
  if (err != cudaSuccess) return -4;
  cudaMemcpy(d, lb.d, 8ull * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(e, lb.e, 8ull * (N - 1), cudaMemcpyDeviceToHost);
  cudaMemcpy(tau, lb.tau, 8ull * (N - 1), cudaMemcpyDeviceToHost);
  cudaMemcpy(V, lb.V, 8ull * N * N, cudaMemcpyDeviceToHost);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

extern "C" int sosadmm_debug_stedc(int N, const double* d, const double* e, double* lam, double* Z) {
  if (N < 2) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  cudaMemcpyAsync(lb.d, d, 8ull * N, cudaMemcpyHostToDevice, dl.s);
  cudaMemcpyAsync(lb.e, e, 8ull * (N - 1), cudaMemcpyHostToDevice, dl.s);
  lb.dc.topsel_on = 0;  // the stage test checks every eigenvector
  large_block_dc(dl.le, lb, dl.s, false);
  cudaError_t err = cudaStreamSynchronize(dl.s);
  if (err != cudaSuccess) return -4;
  const int fb = lb.D & 1;
  cudaMemcpy(lam, lb.dc.lam[fb], 8ull * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(Z, lb.dc.Q[fb], 8ull * N * N, cudaMemcpyDeviceToHost);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

extern "C" int sosadmm_debug_spdinv(int t, double* K) {
  double* dK;
  cudaStream_t s;
  if (cudaStreamCreate(&s)) return -4;
  char* scr;
  if (cudaMalloc(&dK, 8ull * t * t)) return -7;
  if (cudaMalloc(&scr, spdinv_scratch_bytes(t))) {
    cudaFree(dK);
    return -7;
  }
  cudaMemcpy(dK, K, 8ull * t * t, cudaMemcpyHostToDevice);
  const int rc = gpu_spd_inverse(dK, t, s, scr);
  cudaMemcpy(K, dK, 8ull * t * t, cudaMemcpyDeviceToHost);
  cudaFree(dK);
  cudaFree(scr);
  cudaStreamDestroy(s);
  return rc == 0 ? 0 : (rc == 1 ? -3 : -4);
}

// Timing probe of the cluster tridiagonalisation: prof receives 16 clock64 stamp slots per step of
// CTA 0 ((N - 2) x 16), ms the CUDA-event time of one launch (after a warm-up launch).
extern "C" int sosadmm_debug_tridiag_prof(int N, const double* A, long long* prof, float* ms) {
  if (N < 3) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  long long* dprof;
  if (cudaMalloc(&dprof, sizeof(long long) * 16 * N)) return -7;
  cudaMemsetAsync(dprof, 0, sizeof(long long) * 16 * N, dl.s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpyAsync(lb.M, A, 8ull * N * N, cudaMemcpyHostToDevice, dl.s);
    lb.ta.prof = rep ? dprof : nullptr;
    if (rep) cudaEventRecord(e0, dl.s);
    large_block_tridiag(dl.le, lb, dl.s, false);
    if (rep) cudaEventRecord(e1, dl.s);
  }
  lb.ta.prof = nullptr;
  cudaError_t err = cudaStreamSynchronize(dl.s);
  if (err == cudaSuccess) {
    cudaEventElapsedTime(ms, e0, e1);
    cudaMemcpy(prof, dprof, sizeof(long long) * 16 * (N - 2), cudaMemcpyDeviceToHost);
  }
  cudaFree(dprof);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return err == cudaSuccess ? 0 : -4;
}

// ---- two-stage tridiagonalisation stages (sy2sb.cuh, sb2st.cuh, bt2.cuh) ----
// The stage entry points run the two-stage path whatever SOSADMM_TRIDIAG says (when N is inside its envelope).
static bool ts_force(LargeBlock& lb) {
  const bool fits = lb.sy_smem <= (size_t)DYN_SMEM_MAX && lb.st_smem <= (size_t)DYN_SMEM_MAX && lb.sa.maxrb <= 4;
  if (!fits) return false;
  lb.two = true;
  lb.nref = lb.sa.P * lb.BW;
  return true;
}
extern "C" int sosadmm_debug_sy2sb(int N, const double* A, double* band, double* V1, double* tau1, int* bw,
                                   int* nref) {
  if (N < 3) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  if (!ts_force(lb)) return -2;
  cudaMemcpyAsync(lb.M, A, 8ull * N * N, cudaMemcpyHostToDevice, dl.s);
  cudaMemsetAsync(lb.V, 0, 8ull * N * N, dl.s);
  cudaMemsetAsync(lb.tau, 0, 8ull * N, dl.s);
  cudaMemsetAsync(lb.Bg, 0, 8ull * N * 2 * lb.BW, dl.s);
  lb.sa.check_state = 0;
  cudaMemsetAsync(lb.cnt, 0, 16, dl.s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(lb.sa.NW + 1, 1, 1);
  cfg.blockDim = dim3(SB_NT, 1, 1);
  cfg.dynamicSmemBytes = lb.sy_smem;
  cfg.stream = dl.s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, sy2sb_kernel(lb.BW), lb.sa) != cudaSuccess) return -4;
  if (cudaStreamSynchronize(dl.s) != cudaSuccess) return -4;
  cudaMemcpy(band, lb.Bg, 8ull * N * 2 * lb.BW, cudaMemcpyDeviceToHost);
  cudaMemcpy(V1, lb.V, 8ull * N * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(tau1, lb.tau, 8ull * N, cudaMemcpyDeviceToHost);
  *bw = lb.BW;
  *nref = lb.nref;
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

extern "C" int sosadmm_debug_sb2st(int N, int BW, const double* band, double* d, double* e, double* V2,
                                   double* tau2, int* kmax) {
  if (N < 3) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  if (!ts_force(lb) || lb.BW != BW) return -2;
  cudaMemcpyAsync(lb.Bg, band, 8ull * N * 2 * BW, cudaMemcpyHostToDevice, dl.s);
  sb2st_kernel(BW)<<<1, ST_NT, lb.st_smem, dl.s>>>(lb.Bg, N, lb.d, lb.e, lb.V2, lb.tau2, lb.sa.st, lb.sa.is, 0,
                                                   nullptr);
  if (cudaStreamSynchronize(dl.s) != cudaSuccess) return -4;
  cudaMemcpy(d, lb.d, 8ull * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(e, lb.e, 8ull * (N - 1), cudaMemcpyDeviceToHost);
  cudaMemcpy(V2, lb.V2, 8ull * N * lb.KMAX * BW, cudaMemcpyDeviceToHost);
  cudaMemcpy(tau2, lb.tau2, 8ull * N * lb.KMAX, cudaMemcpyDeviceToHost);
  *kmax = lb.KMAX;
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

extern "C" int sosadmm_debug_bt2(int N, int BW, const double* V2, const double* tau2, int r, double* Z) {
  if (N < 3 || r < 0 || r > N) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  if (!ts_force(lb) || lb.BW != BW) return -2;
  const int fb = lb.D & 1;
  cudaMemcpyAsync(lb.V2, V2, 8ull * N * lb.KMAX * BW, cudaMemcpyHostToDevice, dl.s);
  cudaMemcpyAsync(lb.tau2, tau2, 8ull * N * lb.KMAX, cudaMemcpyHostToDevice, dl.s);
  cudaMemcpyAsync(lb.dc.Q[fb], Z, 8ull * N * r, cudaMemcpyHostToDevice, dl.s);
  const int sel[3] = {r, 0, 0};
  cudaMemcpyAsync(lb.sel, sel, sizeof(sel), cudaMemcpyHostToDevice, dl.s);
  bt2_kernel(BW)<<<(r + BT2_NC - 1) / BT2_NC + 1, BT2_NT, lb.bt2_smem_b, dl.s>>>(
      lb.dc.Q[fb], lb.sel, lb.V2, lb.tau2, N, lb.KMAX, lb.sa.st, lb.sa.is, 0);
  if (cudaStreamSynchronize(dl.s) != cudaSuccess) return -4;
  cudaMemcpy(Z, lb.dc.Q[fb], 8ull * N * r, cudaMemcpyDeviceToHost);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

extern "C" int sosadmm_debug_tridiag2(int N, const double* A, double* d, double* e, float* ms) {
  if (N < 3) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  if (!ts_force(lb)) return -2;
  cudaMemcpyAsync(lb.M, A, 8ull * N * N, cudaMemcpyHostToDevice, dl.s);
  large_block_tridiag(dl.le, lb, dl.s, false);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, dl.s);
  large_block_tridiag(dl.le, lb, dl.s, false);
  cudaEventRecord(e1, dl.s);
  if (cudaStreamSynchronize(dl.s) != cudaSuccess) return -4;
  if (ms) cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaMemcpy(d, lb.d, 8ull * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(e, lb.e, 8ull * (N - 1), cudaMemcpyDeviceToHost);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

// ---- one-GPU emulation of a block-sharded solve (tests of the world >= 2 arithmetic) ----
__global__ void k_group_sum(GroupBufs g, int len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  double s = 0.0;
  for (int r = 0; r < g.world; ++r) s += g.buf[r][i];  // rank order (NCCL's order may differ)
  for (int r = 0; r < g.world; ++r) g.buf[r][i] = s;
}

extern "C" int sosadmm_debug_setup_emulated(const sosadmm_problem* prob, const sosadmm_settings* settings,
                                            int32_t rank, int32_t world, const int32_t* block_owner,
                                            sosadmm_ctx** out) {
  if (!out) return SOSADMM_E_ARG;
  if (world < 1 || world > 8 || rank < 0 || rank >= world || !block_owner) {
    *out = nullptr;
    return SOSADMM_E_ARG;
  }
  ShardSpec sp;
  sp.rank = rank;
  sp.world = world;
  sp.block_owner = block_owner;
  sp.sharded = true;
  sp.emulated = true;
  return setup_impl(prob, settings, sp, nullptr, out);
}

// Switch an emulated group to the peer-memory reduction (f4): every rank's k_gather_fin_peer reads the
// other ranks' partial buffers directly (same device here, NVLink peer mappings on real ranks).
extern "C" int sosadmm_debug_group_link_peers(sosadmm_ctx* const* ctx, int world) {
  if (!ctx || world < 1 || world > PEER_MAXW) return SOSADMM_E_ARG;
  std::vector<double*> bufs(world);
  std::vector<unsigned long long*> flags(world);
  for (int r = 0; r < world; ++r) {
    if (!ctx[r] || ctx[r]->err || !ctx[r]->sp.emulated || ctx[r]->sp.world != world || ctx[r]->sp.rank != r)
      return SOSADMM_E_ARG;
    bufs[r] = ctx[r]->dp.shbuf;
    flags[r] = ctx[r]->dp.pflags;
  }
  for (int r = 0; r < world; ++r)
    if (peer_wire(ctx[r], bufs, flags)) return ctx[r]->err;
  return SOSADMM_OK;
}

extern "C" int sosadmm_debug_group_iterate(sosadmm_ctx* const* ctx, int world, int64_t k) {
  if (!ctx || world < 1 || world > 8) return SOSADMM_E_ARG;
  for (int r = 0; r < world; ++r)
    if (!ctx[r] || ctx[r]->err || !ctx[r]->sp.emulated || ctx[r]->sp.world != world || ctx[r]->sp.rank != r)
      return SOSADMM_E_ARG;
  if (ctx[0]->sp.peer) {  // every rank publishes its round, then every rank reduces over the peers' buffers
    for (int64_t it = 0; it < k; ++it) {
      for (int r = 0; r < world; ++r)
        if (launch_iteration(ctx[r], 1, nullptr, 1)) return ctx[r]->err;
      for (int r = 0; r < world; ++r)
        if (cudaStreamSynchronize(ctx[r]->stream) != cudaSuccess) return SOSADMM_E_CUDA;
      for (int r = 0; r < world; ++r)
        if (launch_iteration(ctx[r], 1, nullptr, 2)) return ctx[r]->err;
      for (int r = 0; r < world; ++r)
        if (cudaStreamSynchronize(ctx[r]->stream) != cudaSuccess) return SOSADMM_E_CUDA;
    }
    return SOSADMM_OK;
  }
  GroupBufs g{};
  g.world = world;
  for (int r = 0; r < world; ++r) g.buf[r] = ctx[r]->sh.buf;
  const int len = 2 * ctx[0]->aa.m + 3;
  for (int64_t it = 0; it < k; ++it) {
    for (int r = 0; r < world; ++r)
      if (launch_iteration(ctx[r], 1, nullptr, 1)) return ctx[r]->err;
    for (int r = 0; r < world; ++r)
      if (cudaStreamSynchronize(ctx[r]->stream) != cudaSuccess) return SOSADMM_E_CUDA;
    k_group_sum<<<(len + 255) / 256, 256, 0, ctx[0]->stream>>>(g, len);
    if (cudaStreamSynchronize(ctx[0]->stream) != cudaSuccess) return SOSADMM_E_CUDA;
    for (int r = 0; r < world; ++r)
      if (launch_iteration(ctx[r], 1, nullptr, 2)) return ctx[r]->err;
    for (int r = 0; r < world; ++r)
      if (cudaStreamSynchronize(ctx[r]->stream) != cudaSuccess) return SOSADMM_E_CUDA;
  }
  return SOSADMM_OK;
}

// Full iterate of an emulated group: each column from its owner rank (free columns: rank 0), the
// replicated m-vectors and scalars from rank 0.
extern "C" int sosadmm_debug_group_get_iterate(sosadmm_ctx* const* ctx, int world, double* xi, double* y, double* z,
                                               double* s, double* tau, double* kappa, int64_t* iter) {
  if (!ctx || world < 1 || world > 8) return SOSADMM_E_ARG;
  const int n = ctx[0]->aa.n, m = ctx[0]->aa.m;
  std::vector<double> lx(n), lz(n);
  std::vector<int> own(n);
  for (int r = 0; r < world; ++r) {
    sosadmm_ctx* c = ctx[r];
    if (cudaMemcpy(lx.data(), c->aa.xi, sizeof(double) * n, cudaMemcpyDeviceToHost) ||
        cudaMemcpy(lz.data(), c->aa.z, sizeof(double) * n, cudaMemcpyDeviceToHost) ||
        cudaMemcpy(own.data(), c->sh.colown, sizeof(int) * n, cudaMemcpyDeviceToHost))
      return SOSADMM_E_CUDA;
    for (int j = 0; j < n; ++j)
      if (own[j]) {
        if (xi) xi[j] = lx[j];
        if (z) z[j] = lz[j];
      }
  }
  sosadmm_ctx* c = ctx[0];
  if (y && cudaMemcpy(y, c->aa.y, sizeof(double) * m, cudaMemcpyDeviceToHost)) return SOSADMM_E_CUDA;
  if (s && cudaMemcpy(s, c->aa.s, sizeof(double) * m, cudaMemcpyDeviceToHost)) return SOSADMM_E_CUDA;
  DevState st;
  if (cudaMemcpy(&st, c->aa.st, sizeof(DevState), cudaMemcpyDeviceToHost)) return SOSADMM_E_CUDA;
  if (tau) *tau = st.tau;
  if (kappa) *kappa = st.kappa;
  if (iter) *iter = st.iter;
  return SOSADMM_OK;
}

// Per-stage timing of the two-stage reduction (CUDA events, second of two runs): stage 1, stage 2.
extern "C" int sosadmm_debug_ts_timing(int N, const double* A, float* ms1, float* ms2, long long* prof1,
                                       long long* prof2) {
  if (N < 3) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  if (!ts_force(lb)) return -2;
  long long *dp1 = nullptr, *dp2 = nullptr;
  const size_t n1 = 16 * (size_t)(lb.sa.P + 1), n2 = 4 * (size_t)lb.KMAX;
  if (prof1 && cudaMalloc(&dp1, 8 * n1)) return -7;
  if (prof2 && cudaMalloc(&dp2, 8 * n2)) return -7;
  if (dp1) cudaMemset(dp1, 0, 8 * n1);
  lb.sa.prof = dp1;
  cudaMemcpyAsync(lb.M, A, 8ull * N * N, cudaMemcpyHostToDevice, dl.s);
  cudaEvent_t e[3];
  for (auto& x : e) cudaEventCreate(&x);
  for (int rep = 0; rep < 2; ++rep) {
    lb.sa.check_state = 0;
    cudaMemsetAsync(lb.cnt, 0, 16, dl.s);
    cudaEventRecord(e[0], dl.s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(lb.sa.NW + 1, 1, 1);
    cfg.blockDim = dim3(SB_NT, 1, 1);
    cfg.dynamicSmemBytes = lb.sy_smem;
    cfg.stream = dl.s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, sy2sb_kernel(lb.BW), lb.sa);
    cudaEventRecord(e[1], dl.s);
    sb2st_kernel(lb.BW)<<<1, ST_NT, lb.st_smem, dl.s>>>(lb.Bg, N, lb.d, lb.e, lb.V2, lb.tau2, lb.sa.st, lb.sa.is, 0,
                                                       dp2);
    cudaEventRecord(e[2], dl.s);
  }
  if (cudaStreamSynchronize(dl.s) != cudaSuccess) return -4;
  if (dp1) cudaMemcpy(prof1, dp1, 8 * n1, cudaMemcpyDeviceToHost);
  if (dp2) cudaMemcpy(prof2, dp2, 8 * n2, cudaMemcpyDeviceToHost);
  cudaFree(dp1);
  cudaFree(dp2);
  lb.sa.prof = nullptr;
  cudaEventElapsedTime(ms1, e[0], e[1]);
  cudaEventElapsedTime(ms2, e[1], e[2]);
  for (auto& x : e) cudaEventDestroy(x);
  return 0;
}

// Intermediate results of one large-block projection of A (debugging aid): d, e of the tridiagonal,
// the D&C eigenvalues (ascending) and sel = [r, c0, side].
extern "C" int sosadmm_debug_psd_stages(int N, const double* A, double* d, double* e, double* lam, int* sel) {
  if (N < 3) return -1;
  DebugLarge dl;
  int rc = dl.init(N);
  if (rc) return rc;
  LargeBlock& lb = dl.le.blocks[0];
  cudaMemcpyAsync(lb.M, A, 8ull * N * N, cudaMemcpyHostToDevice, dl.s);
  large_block_tridiag(dl.le, lb, dl.s, false);
  large_block_dc(dl.le, lb, dl.s, false);
  large_block_recon(dl.le, lb, dl.s, false);
  if (cudaStreamSynchronize(dl.s) != cudaSuccess) return -4;
  const int fb = lb.D & 1;
  cudaMemcpy(d, lb.d, 8ull * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(e, lb.e, 8ull * (N - 1), cudaMemcpyDeviceToHost);
  cudaMemcpy(lam, lb.dc.lam[fb], 8ull * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(sel, lb.sel, 12, cudaMemcpyDeviceToHost);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}
