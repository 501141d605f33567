// Device presort of a PreparedDataset (FitContext, forest.hpp:140-160): per column the
// (value asc, row asc) argsort, the dense value rank of every row and the distinct
// values -- the reference's std::sort over (value, row) restated as a stable LSD radix
// sort of order-preserving 64-bit keys carrying the row index (CUB, library code like
// cuBLAS).  -0.0 and +0.0 compare equal in the reference, so both map to one key; a
// distinct value is stored as the first row's original value in sorted order, exactly
// as the reference's `distinct.push_back(v[o[k]])`.
#include <cub/cub.cuh>

#include "forest_kernels.cuh"

namespace aiwc_b200 {

namespace {

__device__ __forceinline__ uint64_t order_key(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 == +0.0 (forest.hpp:154-158 compares with <)
  const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void key_kernel(const double* __restrict__ v, uint64_t n, uint64_t* __restrict__ keys,
                           uint32_t* __restrict__ rows) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n;
       i += uint64_t{gridDim.x} * blockDim.x) {
    keys[i] = order_key(v[i]);
    rows[i] = static_cast<uint32_t>(i);
  }
}

__global__ void flag_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                            uint32_t* __restrict__ flags) {
  for (uint64_t k = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; k < n;
       k += uint64_t{gridDim.x} * blockDim.x)
    flags[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1u : 0u;
}

// inc[k] = 1-based index of the distinct value at sorted position k
__global__ void rank_kernel(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ inc,
                            const double* __restrict__ v, uint64_t n,
                            uint32_t* __restrict__ rank, double* __restrict__ vals) {
  for (uint64_t k = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; k < n;
       k += uint64_t{gridDim.x} * blockDim.x) {
    const uint32_t r = inc[k] - 1u, row = rows[k];
    rank[row] = r;
    if (k == 0 || inc[k - 1] != inc[k]) vals[r] = v[row];
  }
}

__global__ void nonfinite_kernel(const double* __restrict__ v, uint64_t count,
                                 unsigned long long* __restrict__ bad) {
  uint32_t b = 0;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < count;
       i += uint64_t{gridDim.x} * blockDim.x)
    b += isfinite(v[i]) ? 0u : 1u;
  if (b) atomicAdd(bad, static_cast<unsigned long long>(b));
}

unsigned grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 65536 ? (b ? b : 1) : 65536);
}

}  // namespace

__global__ void narrow_kernel(const uint32_t* __restrict__ in, uint64_t count,
                              uint16_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < count;
       i += uint64_t{gridDim.x} * blockDim.x)
    out[i] = static_cast<uint16_t>(in[i]);
}

cudaError_t narrow_ranks(const uint32_t* d_in, uint64_t count, uint16_t* d_out, cudaStream_t s) {
  narrow_kernel<<<grid_for(count), 256, 0, s>>>(d_in, count, d_out);
  return cudaGetLastError();
}

cudaError_t count_nonfinite(const double* d_v, uint64_t count, unsigned long long* d_bad,
                            cudaStream_t s) {
  nonfinite_kernel<<<grid_for(count), 256, 0, s>>>(d_v, count, d_bad);
  return cudaGetLastError();
}

cudaError_t gpu_presort(const double* d_col, uint64_t n, uint32_t p, cudaStream_t s,
                        uint32_t* d_sorted, uint32_t* d_rank, double* d_vals,
                        uint32_t* d_counts, uint64_t* launches) {
  uint64_t *keys_in = nullptr, *keys_out = nullptr;
  uint32_t *rows_in = nullptr, *flags = nullptr, *inc = nullptr;
  void* temp = nullptr;
  size_t sort_bytes = 0, scan_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys_in, keys_out, rows_in,
                                                  d_sorted, static_cast<int>(n), 0, 64, s);
  if (e == cudaSuccess)
    e = cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, flags, inc, static_cast<int>(n), s);
  const size_t temp_bytes = sort_bytes > scan_bytes ? sort_bytes : scan_bytes;
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&keys_in), n * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&keys_out), n * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&rows_in), n * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&flags), n * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&inc), n * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&temp, temp_bytes, s);
  for (uint32_t c = 0; c < p && e == cudaSuccess; ++c) {
    const double* v = d_col + size_t{c} * n;
    uint32_t* sorted = d_sorted + size_t{c} * n;
    key_kernel<<<grid_for(n), 256, 0, s>>>(v, n, keys_in, rows_in);
    size_t tb = temp_bytes;
    e = cub::DeviceRadixSort::SortPairs(temp, tb, keys_in, keys_out, rows_in, sorted,
                                        static_cast<int>(n), 0, 64, s);
    if (e != cudaSuccess) break;
    flag_kernel<<<grid_for(n), 256, 0, s>>>(keys_out, n, flags);
    tb = temp_bytes;
    e = cub::DeviceScan::InclusiveSum(temp, tb, flags, inc, static_cast<int>(n), s);
    if (e != cudaSuccess) break;
    rank_kernel<<<grid_for(n), 256, 0, s>>>(sorted, inc, v, n, d_rank + size_t{c} * n,
                                            d_vals + size_t{c} * n);
    e = cudaMemcpyAsync(d_counts + c, inc + (n - 1), 4, cudaMemcpyDeviceToDevice, s);
    *launches += 5;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaFreeAsync(keys_in, s);
  cudaFreeAsync(keys_out, s);
  cudaFreeAsync(rows_in, s);
  cudaFreeAsync(flags, s);
  cudaFreeAsync(inc, s);
  cudaFreeAsync(temp, s);
  return e;
}

}  // namespace aiwc_b200
