#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "grow.cuh"

namespace aiwc_b200 {

// 16-byte node for inference: threshold (internal) or leaf value (leaf), split
// column (-1 = leaf), left child (right = left + 1, BFS numbering forest.hpp:310-311)
struct alignas(16) PredNode {
  double thr;
  int32_t feature;
  int32_t left;
};

// 8-byte node of a binned tree chunk: split column (0xffff = leaf), threshold bin j,
// chunk-relative left child (right = left + 1) or leaf-value index
struct BinNode {
  uint16_t feat;
  uint16_t j;
  uint32_t child;
};

// field layout of packed 4-byte predict nodes: column in bits [0, cb) (cmask = leaf),
// threshold bin in [cb, cb+bb), chunk-relative child / leaf index from bit sh = cb+bb
struct PredFmt {
  uint32_t cb, bb, sh, cmask, bmask;
};
// 32-bit words of the warp-transposed bins of q queries x p columns
inline uint64_t bin_words(uint64_t q, uint32_t p, uint32_t bin_bytes) {
  const uint64_t e = 4 / bin_bytes;
  return (q + 31) / 32 * ((p + e - 1) / e) * 32;
}

#ifndef AIWC_PRED_NT
#define AIWC_PRED_NT 1024
#endif
#ifndef AIWC_PRED_Q
#define AIWC_PRED_Q 1
#endif
constexpr int kPredictThreads = AIWC_PRED_NT;  // predict CTA size (one CTA per SM)
constexpr int kPredictQ = AIWC_PRED_Q;         // queries per thread (2 measured slower: the
                                               // warp waits for the deepest of 64 paths)

// binned shared-memory predict (kernels live in forest_kernels.cu and are launched there)
cudaError_t launch_bin_queries(int bin_bytes, const double* rows, uint64_t q, uint32_t p,
                               const double* thr, const uint32_t* thr_off, void* bins,
                               cudaStream_t s);
// node_bytes 8: BinNode; 4: packed (column | bin << 7 | child << 15, column 127 = leaf)
cudaError_t launch_predict_chunk(int bin_bytes, int node_bytes, const void* nodes,
                                 uint32_t nnodes, const double* leaves, uint32_t nleaves,
                                 const uint32_t* roots, uint32_t ntrees, const void* bins,
                                 uint64_t q, uint32_t p, double* sum, int first, int last,
                                 double total_trees, double* out, unsigned grid, size_t smem,
                                 size_t smem_max, PredFmt fmt, cudaStream_t s);

// device presort of a dataset (presort.cu): per column (value, row) argsort into
// d_sorted (p x n), dense ranks into d_rank (p x n), distinct values into d_vals
// (column c at c*n), distinct counts into d_counts (p)
cudaError_t gpu_presort(const double* d_col, uint64_t n, uint32_t p, cudaStream_t s,
                        uint32_t* d_sorted, uint32_t* d_rank, double* d_vals,
                        uint32_t* d_counts, uint64_t* launches);
cudaError_t narrow_ranks(const uint32_t* d_in, uint64_t count, uint16_t* d_out, cudaStream_t s);
cudaError_t count_nonfinite(const double* d_v, uint64_t count, unsigned long long* d_bad,
                            cudaStream_t s);

// batched multi-kernel grower for one batch of trees (grow_wide.cuh)
cudaError_t run_wide(int rank_bytes, const WideArgs& a, cudaStream_t st, int sms,
                     uint32_t* h_active, uint64_t* launches);

cudaError_t launch_grow(int nt, int rank_bytes, const GrowArgs& a, int slots, size_t smem,
                        cudaStream_t st, int* blocks_per_sm);

__global__ void compact_kernel(const int32_t* pf, const double* pt, const int32_t* pl,
                               const double* pv, const uint64_t* src_off,
                               const uint64_t* dst_off, int32_t* f, double* thr,
                               int32_t* left, double* val, PredNode* packed);
__global__ void oob_reduce_kernel(const uint32_t* oobleaf, const uint64_t* off,
                                  const double* value, uint32_t T, uint64_t n, double* sum,
                                  uint32_t* count);
__global__ void oob_prefix_kernel(const uint32_t* oobleaf, const uint64_t* off,
                                  const double* value, const uint32_t* cps, uint32_t k,
                                  uint64_t n, double* sums, uint32_t* counts);
__global__ void right_child_kernel(const int32_t* left, uint64_t N, int32_t* right);
__global__ void max_feature_kernel(const int32_t* feature, uint64_t N, int32_t* out);
__global__ void expand_rows_kernel(const double* feats, uint64_t nq, uint32_t nfeat,
                                   uint32_t ndev, double* rows);
__global__ void rank_best_kernel(const double* resp, uint64_t q, uint32_t ndev, uint32_t* best,
                                 uint8_t* near_tie);
__global__ void pack_check_kernel(const uint64_t* off, uint32_t T, const int32_t* feature,
                                  const double* thr, const int32_t* left, const double* val,
                                  PredNode* packed, uint32_t* bad);
__global__ void inbag_flags_kernel(const uint32_t* inbag, uint32_t t0, uint64_t n,
                                   uint8_t* flags);
__global__ void oob_walk_kernel(const PredNode* nodes, const uint64_t* off,
                                const uint8_t* flags, const double* col, uint64_t n, uint32_t t0,
                                uint32_t* oobleaf);
__global__ void make_queries_kernel(const double* rows, uint64_t n, uint32_t p, uint64_t q,
                                    uint64_t seed, uint64_t tag, double* out);
__global__ void predict_small_kernel(const PredNode* nodes, const uint64_t* off, uint32_t T,
                                     const double* rows, uint64_t q, uint32_t p, double* out);
__global__ void predict_kernel(const PredNode* nodes, const uint64_t* off, uint32_t T,
                               const double* rows, uint64_t q, uint32_t p, double* out);

}  // namespace aiwc_b200
