// Forest-level kernels: pool compaction into tree order, out-of-bag reduction,
// out-of-bag walks for imported forests, and batched predict.
#include <cmath>

#include "device_common.cuh"
#include "forest_kernels.cuh"

namespace aiwc_b200 {

// one CTA per tree: pool (completion order) -> forest arrays (tree order); packed
// predict nodes only when asked for (a fitted forest builds them lazily, ensure_packed)
__global__ void compact_kernel(const int32_t* __restrict__ pf, const double* __restrict__ pt,
                               const int32_t* __restrict__ pl, const double* __restrict__ pv,
                               const uint64_t* __restrict__ src_off,
                               const uint64_t* __restrict__ dst_off, int32_t* __restrict__ f,
                               double* __restrict__ thr, int32_t* __restrict__ left,
                               double* __restrict__ val, PredNode* __restrict__ packed) {
  const uint32_t t = blockIdx.x;
  const uint64_t s = src_off[t], o = dst_off[t], cnt = dst_off[t + 1] - o;
  for (uint64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int32_t fi = pf[s + i];
    const double th = pt[s + i];
    const int32_t le = pl[s + i];
    const double v = pv[s + i];
    f[o + i] = fi;
    thr[o + i] = th;
    left[o + i] = le;
    val[o + i] = v;
    if (packed) packed[o + i] = PredNode{fi >= 0 ? th : v, fi, le};
  }
}

// per row, tree-ordered sum of OOB leaf values (forest.hpp:418-435).  oobleaf[t*n + i]
// is the tree-local index of the leaf tree t sends OOB row i to (0xffffffff = in bag);
// the value is read from the forest's node arrays (off = per-tree node offsets).
// Continues from (sum, count) so chained partial forests reproduce the order.
__global__ void oob_reduce_kernel(const uint32_t* __restrict__ oobleaf,
                                  const uint64_t* __restrict__ off,
                                  const double* __restrict__ value, uint32_t T, uint64_t n,
                                  double* __restrict__ sum, uint32_t* __restrict__ count) {
  const uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  double s = sum[i];
  uint32_t c = count[i];
  for (uint32_t t = 0; t < T; ++t) {
    const uint32_t l = __ldg(oobleaf + t * n + i);
    if (l != kInBag) {
      s = __dadd_rn(s, __ldg(value + __ldg(off + t) + l));
      ++c;
    }
  }
  sum[i] = s;
  count[i] = c;
}

// Per-row OOB (sum, count) after each of k ascending tree-count checkpoints, summed in
// tree order: the OOB statistics of every tree prefix of one fit at once (a T-tree fit is
// the first T trees of a longer fit with the same seed, forest.hpp:182, 477-479).
__global__ void oob_prefix_kernel(const uint32_t* __restrict__ oobleaf,
                                  const uint64_t* __restrict__ off,
                                  const double* __restrict__ value,
                                  const uint32_t* __restrict__ cps, uint32_t k, uint64_t n,
                                  double* __restrict__ sums, uint32_t* __restrict__ counts) {
  const uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  uint32_t c = 0, t = 0;
  for (uint32_t j = 0; j < k; ++j) {
    for (const uint32_t te = cps[j]; t < te; ++t) {
      const uint32_t l = __ldg(oobleaf + t * n + i);
      if (l != kInBag) {
        s = __dadd_rn(s, __ldg(value + __ldg(off + t) + l));
        ++c;
      }
    }
    sums[j * n + i] = s;
    counts[j * n + i] = c;
  }
}

// right child of every node (left + 1, BFS numbering forest.hpp:310-311; -1 for leaves)
__global__ void right_child_kernel(const int32_t* __restrict__ left, uint64_t N,
                                   int32_t* __restrict__ right) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < N;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const int32_t l = left[i];
    right[i] = l < 0 ? -1 : l + 1;
  }
}

// Forest built from device SoA (a gathered forest, aiwc_forest_import_device): CTA per
// tree packs the predict nodes and checks the canonical BFS layout the host import checks
// (split nodes' children after them and inside the tree, forest.hpp:310-311); *bad = 1 + tree on failure
__global__ void pack_check_kernel(const uint64_t* __restrict__ off, uint32_t T,
                                  const int32_t* __restrict__ feature,
                                  const double* __restrict__ thr,
                                  const int32_t* __restrict__ left,
                                  const double* __restrict__ val, PredNode* __restrict__ packed,
                                  uint32_t* __restrict__ bad) {
  for (uint32_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint64_t b = off[t], e = off[t + 1];
    if (e <= b) {
      if (threadIdx.x == 0) atomicCAS(bad, 0u, t + 1u);
      continue;
    }
    const int64_t cnt = static_cast<int64_t>(e - b);
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      const int32_t f = feature[i], l = left[i];
      // children after their parent (no back edges: walks terminate) and inside the tree
      if (f >= 0 && (l <= static_cast<int64_t>(i - b) || l + 1 >= cnt)) atomicCAS(bad, 0u, t + 1u);
      packed[i] = PredNode{f >= 0 ? thr[i] : val[i], f, l};
    }
  }
}

// OOB leaves of an imported forest: in-bag flags from the draws, then a walk over the
// column store with the stored f64 thresholds (Tree::predict semantics).  Trees
// [t0, t0 + gridDim.y) -- the host loops over chunks of <= 65,535 trees.
__global__ void inbag_flags_kernel(const uint32_t* __restrict__ inbag, uint32_t t0, uint64_t n,
                                   uint8_t* __restrict__ flags) {
  const uint64_t j = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x;
  const uint64_t t = t0 + blockIdx.y;
  if (j < n) flags[t * n + inbag[t * n + j]] = 1;
}

__global__ void oob_walk_kernel(const PredNode* __restrict__ nodes,
                                const uint64_t* __restrict__ off, const uint8_t* __restrict__ flags,
                                const double* __restrict__ col, uint64_t n, uint32_t t0,
                                uint32_t* __restrict__ oobleaf) {
  const uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x;
  const uint64_t t = t0 + blockIdx.y;
  if (i >= n) return;
  uint32_t leaf = kInBag;
  if (!flags[t * n + i]) {
    const PredNode* nd = nodes + off[t];
    int32_t k = 0;
    PredNode x = nd[0];
    while (x.feature >= 0) {
      k = col[static_cast<uint64_t>(x.feature) * n + i] <= x.thr ? x.left : x.left + 1;
      x = nd[k];
    }
    leaf = static_cast<uint32_t>(k);
  }
  oobleaf[t * n + i] = leaf;
}

// predict_response for q row-major rows: mean over trees, summed in tree order
// (forest.hpp:77-81).  One query per thread; nodes stream from L2.
__global__ void predict_kernel(const PredNode* __restrict__ nodes,
                               const uint64_t* __restrict__ off, uint32_t T,
                               const double* __restrict__ rows, uint64_t q, uint32_t p,
                               double* __restrict__ out) {
  const uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x;
  if (i >= q) return;
  const double* x = rows + i * p;
  double s = 0.0;
  for (uint32_t t = 0; t < T; ++t) {
    const PredNode* nd = nodes + __ldg(off + t);
    PredNode v = nd[0];
    while (v.feature >= 0) {
      const int32_t k = __ldg(x + v.feature) <= v.thr ? v.left : v.left + 1;
      v = nd[k];
    }
    s = __dadd_rn(s, v.thr);
  }
  out[i] = __ddiv_rn(s, static_cast<double>(T));
}

// Few queries (e.g. the 60 held-out rows of an evaluate fold): one warp per query, the
// lanes walk 32 trees at a time from L2, and the warp adds the 32 leaf values in tree
// order (forest.hpp:77-81) -- no binned copy of the forest is built for them.
__global__ void __launch_bounds__(256) predict_small_kernel(const PredNode* __restrict__ nodes,
                                                            const uint64_t* __restrict__ off,
                                                            uint32_t T,
                                                            const double* __restrict__ rows,
                                                            uint64_t q, uint32_t p,
                                                            double* __restrict__ out) {
  __shared__ double st[8][32];
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint64_t i = blockIdx.x * uint64_t{8} + w;
  if (i >= q) return;  // warp-uniform
  const double* x = rows + i * p;
  double s = 0.0;
  for (uint32_t t0 = 0; t0 < T; t0 += 32) {
    const uint32_t t = t0 + lane;
    double leaf = 0.0;
    if (t < T) {
      const PredNode* nd = nodes + __ldg(off + t);
      PredNode v = nd[0];
      while (v.feature >= 0) {
        const int32_t k = __ldg(x + v.feature) <= v.thr ? v.left : v.left + 1;
        v = nd[k];
      }
      leaf = v.thr;
    }
    st[w][lane] = leaf;
    __syncwarp();
    const uint32_t cnt = T - t0 < 32 ? T - t0 : 32;
    for (uint32_t j = 0; j < cnt; ++j) s = __dadd_rn(s, st[w][j]);
    __syncwarp();
  }
  if (lane == 0) out[i] = __ddiv_rn(s, static_cast<double>(T));
}

// Largest split column of a forest (-1 if all leaves): the schema-width check of predict
__global__ void max_feature_kernel(const int32_t* __restrict__ feature, uint64_t N,
                                   int32_t* __restrict__ out) {
  int32_t m = -1;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < N;
       i += uint64_t{gridDim.x} * blockDim.x)
    m = max(m, feature[i]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31u) == 0) atomicMax(out, m);
}

// ---- device ranking (cmd_rank, tools/main.cpp:338-349) ------------------------------
// Rows of nq queries x ndev devices, each Forest::make_row(features_i, device d)
// (forest.hpp:98-115): the nfeat feature values, then a one-hot over the device columns.
// Expanded chunk-wise in HBM so the binned predict path scores them.
__global__ void expand_rows_kernel(const double* __restrict__ feats, uint64_t nq,
                                   uint32_t nfeat, uint32_t ndev, double* __restrict__ rows) {
  const uint32_t p = nfeat + ndev;
  const uint64_t total = nq * ndev * p;
  for (uint64_t g = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; g < total;
       g += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t r = g / p;
    const uint32_t c = static_cast<uint32_t>(g - r * p);
    const uint64_t i = r / ndev;
    const uint32_t d = static_cast<uint32_t>(r - i * ndev);
    rows[g] = c < nfeat ? feats[i * nfeat + c] : (c - nfeat == d ? 1.0 : 0.0);
  }
}

// Thread per query: the first-ranked device = smallest response, lowest device column on
// ties (ranking sorts (seconds, device name) and device columns are in name order,
// dataset.hpp:121-126).  seconds = 10^r is monotone but may merge distinct responses a few
// ulps apart, so a runner-up within 1e-12 relative flags the query for the exact host
// tie-break (std::pow, as Forest::predict_time, forest.hpp:84-86).
__global__ void rank_best_kernel(const double* __restrict__ resp, uint64_t q, uint32_t ndev,
                                 uint32_t* __restrict__ best, uint8_t* __restrict__ near_tie) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < q;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const double* r = resp + i * ndev;
    uint32_t b = 0;
    double rb = r[0];
    for (uint32_t d = 1; d < ndev; ++d)
      if (r[d] < rb) {
        rb = r[d];
        b = d;
      }
    uint8_t tie = 0;
    const double tol = 1e-12 * fmax(1.0, fabs(rb));
    for (uint32_t d = 0; d < ndev; ++d)
      if (d != b && r[d] - rb <= tol) tie = 1;
    best[i] = b;
    near_tie[i] = tie;
  }
}

// ---- shared-memory predict over binned queries ------------------------------------
// Threshold binning: with T_c the sorted distinct thresholds the forest uses on column
// c and thr = T_c[j],  x <= thr  <=>  #{t in T_c : t < x} <= j.  NaN goes to the
// largest bin (every comparison false -> right child, as in Tree::predict).
//
// Bins are stored warp-transposed: per group of 32 queries, word k of query l (bins
// k*E .. k*E+E-1, E = 4 / sizeof(BinT)) at group*W*32 + k*32 + l.  A warp's 32 queries
// then read their bins from 32 different banks whatever columns they test -- no shared-
// memory bank conflicts in the tree walks (row-major bins cost 2.15 wavefronts/load).
template <typename BinT>
__global__ void bin_queries_kernel(const double* __restrict__ rows, uint64_t q, uint32_t p,
                                   const double* __restrict__ thr,
                                   const uint32_t* __restrict__ thr_off,
                                   uint32_t* __restrict__ bins) {
  constexpr uint32_t E = 4 / sizeof(BinT);
  const uint32_t W = (p + E - 1) / E;
  const uint64_t groups = (q + 31) / 32, total = groups * W * 32;
  for (uint64_t g = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; g < total;
       g += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t grp = g / (uint64_t{W} * 32);
    const uint32_t rem = static_cast<uint32_t>(g - grp * W * 32), k = rem / 32, l = rem % 32;
    const uint64_t qi = grp * 32 + l;
    uint32_t word = 0;
    for (uint32_t e = 0; e < E; ++e) {
      const uint32_t c = k * E + e;
      if (c >= p || qi >= q) break;
      const double x = rows[qi * p + c];
      const double* t = thr + thr_off[c];
      uint32_t lo = 0, hi = thr_off[c + 1] - thr_off[c];
      if (x != x) {
        lo = sizeof(BinT) == 1 ? 0xffu : 0xffffu;
      } else {
        while (lo < hi) {  // first index with t >= x == count of thresholds < x
          const uint32_t mid = (lo + hi) >> 1;
          if (t[mid] < x) lo = mid + 1; else hi = mid;
        }
      }
      word |= lo << (8 * sizeof(BinT) * e);
    }
    bins[g] = word;
  }
}

// Node accessors.  A split node names its column by the BYTE OFFSET of that column's bin
// inside a query's transposed bin words (column c: word c/E at +128 bytes each, byte
// (c%E)*sizeof(BinT)), so a visit reads its bin with one shared-memory load at
// thread_base + off -- no column arithmetic.  8-byte BinNode {off, j, child}, or the
// packed 4-byte form: off in the low 12 bits (0xfff = leaf), threshold bin in the next bb
// bits, chunk-relative left child (right = left + 1) or leaf index above (PredFmt) --
// half the node wavefronts per visit and twice the trees per chunk.
struct Node8 {
  using T = BinNode;
  static __device__ __forceinline__ bool leaf(const BinNode& v, PredFmt) { return v.feat == 0xffffu; }
  static __device__ __forceinline__ uint32_t off(const BinNode& v, PredFmt) { return v.feat; }
  static __device__ __forceinline__ uint32_t j(const BinNode& v, PredFmt) { return v.j; }
  static __device__ __forceinline__ uint32_t child(const BinNode& v, PredFmt) { return v.child; }
};
struct Node4 {
  using T = uint32_t;
  static __device__ __forceinline__ bool leaf(uint32_t v, PredFmt) { return (v & 0xfffu) == 0xfffu; }
  static __device__ __forceinline__ uint32_t off(uint32_t v, PredFmt) { return v & 0xfffu; }
  static __device__ __forceinline__ uint32_t j(uint32_t v, PredFmt f) { return (v >> 12) & f.bmask; }
  static __device__ __forceinline__ uint32_t child(uint32_t v, PredFmt f) { return v >> f.sh; }
};

// One launch per tree chunk: the chunk's nodes and leaf values sit in shared memory,
// every query walks the chunk's trees in order, continuing its running sum from the
// previous chunk (so the per-query sum keeps the reference's tree order exactly).
// A tile holds Q*NT queries (whole 32-query groups of the transposed bins); thread t
// walks queries t, t+NT, ... of it as Q independent node chains.
template <typename BinT, typename NA, int NT, int Q>
__global__ void __launch_bounds__(NT, 1)
    predict_chunk_kernel(const typename NA::T* __restrict__ nodes, uint32_t nnodes,
                         const double* __restrict__ leaves, uint32_t nleaves,
                         const uint32_t* __restrict__ roots, uint32_t ntrees,
                         const uint32_t* __restrict__ bins, uint64_t q, uint32_t p,
                         double* __restrict__ sum, int first, int last, double total_trees,
                         double* __restrict__ out, PredFmt fmt) {
  using NodeT = typename NA::T;
  constexpr uint32_t TQ = NT * Q;
  constexpr uint32_t E = 4 / sizeof(BinT);
  const uint32_t W = (p + E - 1) / E;  // bin words per query
  extern __shared__ __align__(16) unsigned char smem[];
  NodeT* sn = reinterpret_cast<NodeT*>(smem);
  double* sl = reinterpret_cast<double*>(smem + ((nnodes * sizeof(NodeT) + 15) & ~size_t{15}));
  uint32_t* sb = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(sl) +
                                             ((size_t{nleaves} * 8 + 15) & ~size_t{15}));
  for (uint32_t i = threadIdx.x; i < nnodes; i += NT) sn[i] = nodes[i];
  for (uint32_t i = threadIdx.x; i < nleaves; i += NT) sl[i] = leaves[i];
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t tile = uint64_t{blockIdx.x} * TQ; tile < q; tile += uint64_t{gridDim.x} * TQ) {
    __syncthreads();
    const uint64_t rem = q - tile;
    const uint32_t cnt = rem < TQ ? static_cast<uint32_t>(rem) : TQ;
    {  // stage the tile's groups of transposed bins: 16-byte copies, 4 in flight
      const size_t n16 = size_t{(cnt + 31) / 32} * W * 32 / 4;
      const uint4* s4 = reinterpret_cast<const uint4*>(bins + (tile / 32) * W * 32);
      uint4* d4 = reinterpret_cast<uint4*>(sb);
      size_t i = threadIdx.x;
      for (; i + 3 * NT < n16; i += 4 * NT) {
        const uint4 a0 = __ldg(s4 + i), a1 = __ldg(s4 + i + NT), a2 = __ldg(s4 + i + 2 * NT),
                    a3 = __ldg(s4 + i + 3 * NT);
        d4[i] = a0;
        d4[i + NT] = a1;
        d4[i + 2 * NT] = a2;
        d4[i + 3 * NT] = a3;
      }
      for (; i < n16; i += NT) d4[i] = __ldg(s4 + i);
    }
    __syncthreads();
    if (threadIdx.x >= cnt) continue;
    const unsigned char* bq[Q];
    double s[Q];
#pragma unroll
    for (int u = 0; u < Q; ++u) {
      // a query slot past the tile's end re-walks query threadIdx.x (result dropped)
      const uint32_t qi = threadIdx.x + u * NT < cnt ? threadIdx.x + u * NT : threadIdx.x;
      bq[u] = reinterpret_cast<const unsigned char*>(sb + (qi / 32) * W * 32 + lane);
      s[u] = first ? 0.0 : sum[tile + qi];
    }
    for (uint32_t t = 0; t < ntrees; ++t) {
      const uint32_t r = roots[t];
      uint32_t idx[Q];
      NodeT v[Q];
      bool done = true;
#pragma unroll
      for (int u = 0; u < Q; ++u) {
        idx[u] = r;
        v[u] = sn[r];
        done = done && NA::leaf(v[u], fmt);
      }
      while (!done) {
        done = true;
#pragma unroll
        for (int u = 0; u < Q; ++u) {
          const bool lf = NA::leaf(v[u], fmt);
          const uint32_t bin = *reinterpret_cast<const BinT*>(bq[u] + (lf ? 0u : NA::off(v[u], fmt)));
          idx[u] = lf ? idx[u] : NA::child(v[u], fmt) + (bin <= NA::j(v[u], fmt) ? 0u : 1u);
        }
#pragma unroll
        for (int u = 0; u < Q; ++u) {
          v[u] = sn[idx[u]];
          done = done && NA::leaf(v[u], fmt);
        }
      }
#pragma unroll
      for (int u = 0; u < Q; ++u) s[u] = __dadd_rn(s[u], sl[NA::child(v[u], fmt)]);
    }
#pragma unroll
    for (int u = 0; u < Q; ++u) {
      if (threadIdx.x + u * NT >= cnt) continue;
      const uint64_t qi = tile + threadIdx.x + u * NT;
      if (last)
        out[qi] = __ddiv_rn(s[u], total_trees);
      else
        sum[qi] = s[u];
    }
  }
}

// host-side launchers (kernels are launched from the TU that defines them)
namespace {
template <typename BinT>
cudaError_t bin_t(const double* rows, uint64_t q, uint32_t p, const double* thr,
                  const uint32_t* thr_off, void* bins, cudaStream_t s) {
  const uint64_t words = bin_words(q, p, sizeof(BinT));
  const uint64_t blocks = (words + 255) / 256;
  bin_queries_kernel<BinT><<<static_cast<unsigned>(blocks < 524288 ? blocks : 524288), 256, 0,
                             s>>>(rows, q, p, thr, thr_off, static_cast<uint32_t*>(bins));
  return cudaGetLastError();
}
template <typename BinT, typename NA>
cudaError_t chunk_t(const void* nodes, uint32_t nnodes, const double* leaves, uint32_t nleaves,
                    const uint32_t* roots, uint32_t ntrees, const void* bins, uint64_t q,
                    uint32_t p, double* sum, int first, int last, double total_trees, double* out,
                    unsigned grid, size_t smem, size_t smem_max, PredFmt fmt, cudaStream_t s) {
  auto k = predict_chunk_kernel<BinT, NA, kPredictThreads, kPredictQ>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_max));
  if (e != cudaSuccess) return e;
  k<<<grid, kPredictThreads, smem, s>>>(static_cast<const typename NA::T*>(nodes), nnodes,
                                        leaves, nleaves, roots, ntrees,
                                        static_cast<const uint32_t*>(bins), q, p, sum, first,
                                        last, total_trees, out, fmt);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_bin_queries(int bin_bytes, const double* rows, uint64_t q, uint32_t p,
                               const double* thr, const uint32_t* thr_off, void* bins,
                               cudaStream_t s) {
  return bin_bytes == 1 ? bin_t<uint8_t>(rows, q, p, thr, thr_off, bins, s)
                        : bin_t<uint16_t>(rows, q, p, thr, thr_off, bins, s);
}

cudaError_t launch_predict_chunk(int bin_bytes, int node_bytes, const void* nodes,
                                 uint32_t nnodes, const double* leaves, uint32_t nleaves,
                                 const uint32_t* roots, uint32_t ntrees, const void* bins,
                                 uint64_t q, uint32_t p, double* sum, int first, int last,
                                 double total_trees, double* out, unsigned grid, size_t smem,
                                 size_t smem_max, PredFmt fmt, cudaStream_t s) {
  if (node_bytes == 4)
    return bin_bytes == 1
               ? chunk_t<uint8_t, Node4>(nodes, nnodes, leaves, nleaves, roots, ntrees, bins, q,
                                         p, sum, first, last, total_trees, out, grid, smem,
                                         smem_max, fmt, s)
               : chunk_t<uint16_t, Node4>(nodes, nnodes, leaves, nleaves, roots, ntrees, bins, q,
                                          p, sum, first, last, total_trees, out, grid, smem,
                                          smem_max, fmt, s);
  return bin_bytes == 1
             ? chunk_t<uint8_t, Node8>(nodes, nnodes, leaves, nleaves, roots, ntrees, bins, q, p,
                                       sum, first, last, total_trees, out, grid, smem, smem_max,
                                       fmt, s)
             : chunk_t<uint16_t, Node8>(nodes, nnodes, leaves, nleaves, roots, ntrees, bins, q, p,
                                        sum, first, last, total_trees, out, grid, smem, smem_max,
                                        fmt, s);
}

// C5 query generator: query i copies table row Rng(derive_seed(seed,"query",i)).bounded(n)
// (first draw of that stream; rng.hpp:32-59)
__global__ void make_queries_kernel(const double* __restrict__ rows, uint64_t n, uint32_t p,
                                    uint64_t q, uint64_t seed, uint64_t tag,
                                    double* __restrict__ out) {
  const uint64_t total = q * p;
  for (uint64_t g = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; g < total;
       g += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t i = g / p, c = g - i * p;
    const uint64_t key = dmix64(seed ^ tag ^ dmix64(i));
    const uint64_t r = draw_bounded(key, 1, n);
    out[g] = rows[r * p + c];
  }
}

}  // namespace aiwc_b200
