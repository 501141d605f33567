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

cudaError_t launch_grow(int nt, int rank_bytes, const GrowArgs& a, int slots, size_t smem,
                        cudaStream_t st, int* blocks_per_sm);

__global__ void compact_kernel(const int32_t* pf, const double* pt, const int32_t* pl,
                               const double* pv, const uint64_t* src_off,
                               const uint64_t* dst_off, int32_t* f, double* thr,
                               int32_t* left, double* val, PredNode* packed);
__global__ void oob_reduce_kernel(const double* oobval, uint32_t T, uint64_t n, double* sum,
                                  uint32_t* count);
__global__ void inbag_flags_kernel(const uint32_t* inbag, uint32_t T, uint64_t n,
                                   uint8_t* flags);
__global__ void oob_walk_kernel(const PredNode* nodes, const uint64_t* off,
                                const uint8_t* flags, const double* col, uint64_t n,
                                double* oobval);
__global__ void make_queries_kernel(const double* rows, uint64_t n, uint32_t p, uint64_t q,
                                    uint64_t seed, uint64_t tag, double* out);
__global__ void predict_kernel(const PredNode* nodes, const uint64_t* off, uint32_t T,
                               const double* rows, uint64_t q, uint32_t p, double* out);

}  // namespace aiwc_b200
