// Device-side helpers shared by the forest kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace aiwc_b200 {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;
constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kInBag = 0xffffffffu;  // OOB leaf index of an in-bag row

// splitmix64 finaliser (rng.hpp:13-18)
__device__ __forceinline__ uint64_t dmix64(uint64_t x) {
  x += kGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// draw `k` (1-based counter) of the stream keyed by `key`, bounded to [0, n)
// (Rng::next_u64 + Rng::bounded, rng.hpp:45, 56-59)
__device__ __forceinline__ uint64_t draw_bounded(uint64_t key, uint64_t k, uint64_t n) {
  return __umul64hi(dmix64(key + k * kGamma), n);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(kFull, v, o);
    if (static_cast<int>(lane_id()) >= o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Block-wide exclusive scan of one uint32 per thread.  `sh` needs NT/32 + 1 words.
// Returns the exclusive prefix; *total receives the block sum.  Contains three
// __syncthreads(); every thread must call it.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sh,
                                                    uint32_t* total) {
  constexpr int NW = NT / 32;
  __syncthreads();  // `sh` may still be read by a previous call
  const uint32_t inc = warp_incl_scan(v);
  if (lane_id() == 31) sh[warp_id()] = inc;
  __syncthreads();
  if (warp_id() == 0) {
    uint32_t w = lane_id() < NW ? sh[lane_id()] : 0u;
    const uint32_t wi = warp_incl_scan(w);
    if (lane_id() < NW) sh[lane_id()] = wi - w;
    if (lane_id() == NW - 1) sh[NW] = wi;
  }
  __syncthreads();
  const uint32_t r = sh[warp_id()] + inc - v;
  *total = sh[NW];
  return r;
}

// Block-wide exclusive scan of one uint64 per thread (used with 4 packed 16-bit
// counters: one scan serves four tile rows).  `sh` needs 2*(NT/32) + 2 words.
template <int NT>
__device__ __forceinline__ uint64_t block_excl_scan64(uint64_t v, uint64_t* sh,
                                                      uint64_t* total) {
  constexpr int NW = NT / 32;
  __syncthreads();
  const uint64_t inc = warp_incl_scan(v);
  if (lane_id() == 31) sh[warp_id()] = inc;
  __syncthreads();
  if (warp_id() == 0) {
    const uint64_t w = lane_id() < NW ? sh[lane_id()] : 0ull;
    const uint64_t wi = warp_incl_scan(w);
    if (lane_id() < NW) sh[lane_id()] = wi - w;
    if (lane_id() == NW - 1) sh[NW] = wi;
  }
  __syncthreads();
  const uint64_t r = sh[warp_id()] + inc - v;
  *total = sh[NW];
  return r;
}

}  // namespace aiwc_b200
