// Layout shared by the forest grower kernel (grow.cu) and its host driver (capi.cu).
#pragma once

#include <cstddef>
#include <cstdint>

namespace aiwc_b200 {

// One frontier node: its compacted range [b, e) in the level's payload / list
// order, its BFS node id and its (weight, sum, sumsq) -- NodeWork, forest.hpp:211-215.
struct NodeWork {
  uint32_t b, e, id, pad;
  double w, s, q;
};

// Per in-bag row of a tree, in node-grouped row order: global row, bootstrap
// multiplicity, weighted response mult*y (forest.hpp:194-195).
struct Payload {
  uint32_t row, mult;
  double wy;
};

struct ChainRes {
  double gain;
  uint32_t pos;
  uint32_t pad;
};

struct SplitInfo {
  uint32_t f;         // frontier index of the split node
  uint32_t c;         // chosen column
  uint32_t thr_rank;  // largest global value rank <= threshold
  uint32_t cnt;       // rows of the node
  uint32_t nl;        // rows going left (route result)
  uint32_t base;      // compacted start of the children
  uint32_t pad0, pad1;
};

// per segment (frontier node) partition offsets; offL == INT32_MIN => leaf (drop)
struct SegTab {
  int32_t offL, offR;
  uint32_t child;  // next-frontier index of the left child
  uint32_t pad;
};

// Device view of a PreparedDataset (forest.hpp:134-161): column store, responses,
// per-column (value,row) argsort, dense value ranks and the distinct values.
// Columns with <= 2 distinct values ("two-level" columns, e.g. the one-hot device
// columns) keep no sorted list: their (value,row) order is the row order of the
// value-0 rows followed by the value-1 rows, which the grower reads off the
// row-ordered payload directly.
struct DevData {
  uint64_t n;
  uint32_t p;
  uint32_t rank_bytes;      // 2 or 4
  uint32_t nlisted;         // columns with >= 3 distinct values
  uint32_t order_stride;    // padded row stride of `order` (multiple of 4)
  const double* col;        // p x n
  const double* y;          // n
  const uint32_t* order;    // nlisted x order_stride, listed columns only
  const void* rank;         // p x n (uint16 or uint32)
  const double* vals;       // concatenated distinct sorted values per column
  const uint64_t* vals_off; // p+1
  const int32_t* list_of;   // p: list slot of column c, or -1
  const uint32_t* listed;   // nlisted: column of list slot i
};

struct SlotLayout {
  uint32_t stride;  // max in-bag rows per tree (payload / list length)
  uint32_t fmax;    // max frontier width
  uint32_t emax;    // max eligible nodes per level
  uint32_t nodes_cap;
  size_t off_mult, off_pay0, off_pay1, off_list0, off_list1, off_seg0,
      off_seg1, off_front0, off_front1, off_segtab, off_e2f, off_samp, off_res, off_split,
      off_nf, off_nthr, off_nleft, off_nval, off_nrank, off_chunk, off_off2, off_gbits, off_gpref,
      off_ecls, off_wsplit;
  size_t bytes;
};

struct GrowArgs {
  DevData d;
  uint32_t mtry, mns;
  // several forests in one launch (grid cells, batched concurrent fits): local tree tl
  // belongs to forest tree_cell[tl], grows with that forest's mtry / min.node.size /
  // seed, and is tree tree_t[tl] of its forest (its RNG key).  Null: one forest.
  const uint32_t* tree_cell;
  const uint32_t* tree_t;
  const uint32_t* cell_mtry;
  const uint32_t* cell_mns;
  const uint64_t* cell_seed;
  // hold-out folds (evaluate, experiments.hpp:393-397): forest c trains on
  // cell_nrows[c] rows of the table, its local row i being table row
  // cell_rows[cell_rows_off[c] + i] (ascending).  Null: every forest trains on all n rows.
  const uint32_t* cell_nrows;
  const uint32_t* cell_rows;
  const uint64_t* cell_rows_off;
  uint64_t seed;
  uint64_t tag_tree;  // fnv1a64("tree")
  uint32_t tree_begin, tree_end;
  uint32_t* queue;    // dynamic tree counter
  char* scratch;      // slots x layout.bytes
  SlotLayout L;
  int bits_in_smem;
  // outputs (indexed by local tree t - tree_begin)
  uint32_t* inbag;    // T x n, may be null
  uint32_t* oobleaf;  // T x n tree-local OOB leaf index (kInBag = in bag), may be null
  int32_t* pool_feature;
  double* pool_thr;
  int32_t* pool_left;
  double* pool_value;
  uint32_t* pool_rank;
  unsigned long long* pool_used;
  uint64_t pool_cap;
  uint64_t* tree_off;
  uint32_t* tree_cnt;
  unsigned long long* split_rows;  // sum over split nodes of their in-bag distinct rows
  unsigned long long* prof;  // optional: kPhases per-phase cycle totals (all CTAs)
  int* err;  // 1 = pool overflow, 2 = in-bag rows exceed stride, 3 = frontier overflow
};

// per-tree level state of the wide (batched) grower
struct TreeState {
  uint32_t A, F, E, S;
  uint32_t nodes, done, totL, A_next;
  uint32_t E0, E1, E2;  // eligible nodes by size class: small (lane chains), mid (lane
                        // groups), big (warp per chain)
  uint32_t Sbig;        // split nodes routed by a CTA (column 0 listed, >= coop_min rows)
  uint32_t Swarp;       // split nodes routed by a warp (the rest of those >= kLaneMax rows)
  unsigned long long elig_base, split_rows;
};

struct WideArgs {
  GrowArgs g;
  TreeState* ts;     // [B]
  uint32_t B;        // trees in this batch (slots 0..B-1)
  uint32_t t0;       // local index of the batch's first tree
  uint32_t cur;      // buffer parity of the current level
  uint32_t big_min;  // nodes with >= big_min rows run one warp per chain (else lane groups)
  uint32_t coop_min; // split nodes with >= coop_min rows are routed by one CTA each
  uint32_t pair_big; // lanes per chain for big nodes: 32 (warp), 16 or 8 (lane groups)
  uint32_t lane_max; // nodes below this many rows run one lane per chain
  uint32_t* off[5];  // [B+1] prefixes: chain tasks, splits, positions, list chunks, warp routes
  uint32_t* active;  // trees still splitting after this level's decide
  uint32_t* task_ctr;  // dynamic task counters of this level's chain kernels (zeroed by w_prefix)
};

// bitmap words + prefix words the grower keeps in shared memory (or global)
__host__ __device__ inline size_t grow_bits_words(uint64_t n, uint32_t stride) {
  const size_t a = (n + 31) / 32, b = (stride + 31) / 32;
  return (((a > b ? a : b) + 2) + 1) & ~size_t{1};
}
__host__ __device__ inline size_t grow_pref_words(uint64_t n, uint32_t stride) {
  const size_t a = (n + 63) / 64, b = (stride + 31) / 32;
  return (a > b ? a : b) + 2;
}

SlotLayout make_layout(uint64_t n, uint32_t p, uint32_t nlisted, uint32_t mtry, uint32_t mns,
                       bool gbits);

}  // namespace aiwc_b200
