// PSD projection of large Gram blocks (N > 64): placeholder, replaced by the tridiagonal
// path (Householder tridiagonalisation in a thread-block cluster, divide-and-conquer, DMMA
// back-transform and reconstruction).
#pragma once
#include <string>
#include <vector>
#include "common.cuh"

struct LargeEig {
  int nlarge = 0;
};

inline size_t large_eig_bytes(const std::vector<int>& blk_N, const std::vector<int>& large) { return 0; }
inline int large_eig_init(LargeEig& le, const std::vector<int>& blk_N, const std::vector<long long>& blk_mat,
                          const std::vector<int>& large, double* mats, char* base, DevState* st, IterScal* is,
                          cudaStream_t s, std::string& msg) {
  le.nlarge = (int)large.size();
  if (le.nlarge) {
    msg = "blocks with N > 64 are not supported yet";
    return 1;
  }
  return 0;
}
inline void large_eig_launch(LargeEig& le, cudaStream_t s, bool check) {}
inline int large_eig_launches(const LargeEig& le) { return 0; }
inline void large_eig_free(LargeEig& le) {}
