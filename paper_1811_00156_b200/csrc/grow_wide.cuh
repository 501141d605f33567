// "Wide" forest grower for large tables -- included at the end of grow.cu (it uses
// that file's device helpers).
//
// Same algorithm and the same bit-exact results as grow_kernel, but the batch of trees
// advances level-synchronously and every phase of a level is its own grid-wide kernel
// over ALL trees of the batch: per-tree bookkeeping (leaf tests, numbering scans,
// segment tables) runs one CTA per tree, while the heavy passes (split chains, routing,
// payload and list partitions) are flattened over (tree, task) and spread over the
// whole GPU at full occupancy.  A tree's long sequential FP64 chain on a huge node no
// longer idles the rest of its CTA: other trees' tasks fill the SMs.
#pragma once

namespace aiwc_b200 {

// Pointers of slot b for the current level (cur) and the next one (suffix _n).  The
// double buffers are resolved here, with selects, so no kernel indexes a pointer array
// dynamically (that would put the whole struct in local memory).
struct SlotPtrs {
  uint32_t* mult;
  Payload *pay, *pay_n;
  uint32_t *lists, *lists_n;
  uint32_t *seg, *seg_n;
  NodeWork *front, *front_n;
  SegTab* segtab;
  uint32_t* e2f;
  uint32_t* ecls;
  uint32_t* wsplit;
  uint16_t* samp;
  ChainRes* res;
  SplitInfo* spl;
  int32_t* nf;
  double* nthr;
  int32_t* nleft;
  double* nval;
  uint32_t* nrank;
  uint32_t* chunk;
  int2* off2;
  uint32_t* bits;
  uint32_t* pref;
};

__device__ __forceinline__ SlotPtrs slot_ptrs(const WideArgs& a, uint32_t b) {
  const SlotLayout& L = a.g.L;
  char* s = a.g.scratch + static_cast<size_t>(b) * L.bytes;
  const bool c = a.cur != 0u;
  SlotPtrs p;
  p.mult = reinterpret_cast<uint32_t*>(s + L.off_mult);
  p.pay = reinterpret_cast<Payload*>(s + (c ? L.off_pay1 : L.off_pay0));
  p.pay_n = reinterpret_cast<Payload*>(s + (c ? L.off_pay0 : L.off_pay1));
  p.lists = reinterpret_cast<uint32_t*>(s + (c ? L.off_list1 : L.off_list0));
  p.lists_n = reinterpret_cast<uint32_t*>(s + (c ? L.off_list0 : L.off_list1));
  p.seg = reinterpret_cast<uint32_t*>(s + (c ? L.off_seg1 : L.off_seg0));
  p.seg_n = reinterpret_cast<uint32_t*>(s + (c ? L.off_seg0 : L.off_seg1));
  p.front = reinterpret_cast<NodeWork*>(s + (c ? L.off_front1 : L.off_front0));
  p.front_n = reinterpret_cast<NodeWork*>(s + (c ? L.off_front0 : L.off_front1));
  p.segtab = reinterpret_cast<SegTab*>(s + L.off_segtab);
  p.e2f = reinterpret_cast<uint32_t*>(s + L.off_e2f);
  p.ecls = reinterpret_cast<uint32_t*>(s + L.off_ecls);
  p.wsplit = reinterpret_cast<uint32_t*>(s + L.off_wsplit);
  p.samp = reinterpret_cast<uint16_t*>(s + L.off_samp);
  p.res = reinterpret_cast<ChainRes*>(s + L.off_res);
  p.spl = reinterpret_cast<SplitInfo*>(s + L.off_split);
  p.nf = reinterpret_cast<int32_t*>(s + L.off_nf);
  p.nthr = reinterpret_cast<double*>(s + L.off_nthr);
  p.nleft = reinterpret_cast<int32_t*>(s + L.off_nleft);
  p.nval = reinterpret_cast<double*>(s + L.off_nval);
  p.nrank = reinterpret_cast<uint32_t*>(s + L.off_nrank);
  p.chunk = reinterpret_cast<uint32_t*>(s + L.off_chunk);
  p.off2 = reinterpret_cast<int2*>(s + L.off_off2);
  p.bits = reinterpret_cast<uint32_t*>(s + L.off_gbits);
  p.pref = reinterpret_cast<uint32_t*>(s + L.off_gpref);
  return p;
}

// tree index b of flattened item t given exclusive prefix off[0..B] (off[B] = total)
__device__ __forceinline__ uint32_t owner(const uint32_t* off, uint32_t B, uint32_t t) {
  uint32_t lo = 0, hi = B;  // off[lo] <= t < off[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// lane-group width of the mid-size chain kernel: the widest power of two that still
// fits all m sampled columns of a node in one warp (G = 32 / pow2ceil(m)), but at least
// kGrpMin lanes per chain -- a node with more columns than 32 / kGrpMin then takes
// several warps (grp_tpn)
#ifndef AIWC_GRP_MIN
#define AIWC_GRP_MIN 1
#endif
constexpr uint32_t kGrpMin = AIWC_GRP_MIN;
__host__ __device__ inline uint32_t grp_width(uint32_t m) {
  uint32_t c = 1;
  while (c < m && c < 32) c <<= 1;
  return 32u / c > kGrpMin ? 32u / c : kGrpMin;
}

// Per-tree parameters: with several forests (GrowArgs::tree_cell) the batch's tree b is
// tree tree_t[t0+b] of forest tree_cell[t0+b], which has its own mtry / mns / seed.
__device__ __forceinline__ uint32_t tree_m(const WideArgs& a, uint32_t b) {
  return a.g.tree_cell ? a.g.cell_mtry[a.g.tree_cell[a.t0 + b]] : a.g.mtry;
}
__device__ __forceinline__ uint32_t tree_mns(const WideArgs& a, uint32_t b) {
  return a.g.tree_cell ? a.g.cell_mns[a.g.tree_cell[a.t0 + b]] : a.g.mns;
}
// training rows of the batch's tree b: its fold's row count, or the whole table
__device__ __forceinline__ uint32_t tree_n(const WideArgs& a, uint32_t b) {
  return a.g.cell_nrows ? a.g.cell_nrows[a.g.tree_cell[a.t0 + b]]
                        : static_cast<uint32_t>(a.g.d.n);
}
__device__ __forceinline__ uint64_t tree_key(const WideArgs& a, uint32_t b) {
  const uint32_t tl = a.t0 + b;
  if (a.g.tree_cell)
    return dmix64(a.g.cell_seed[a.g.tree_cell[tl]] ^ a.g.tag_tree ^ dmix64(uint64_t{a.g.tree_t[tl]}));
  return dmix64(a.g.seed ^ a.g.tag_tree ^ dmix64(uint64_t{a.g.tree_begin} + tl));
}
// lane-group tasks of a node with m sampled columns when the group kernel was launched
// for the batch's widest mtry (lane groups of grp_width(mmax))
__host__ __device__ inline uint32_t grp_tpn(uint32_t m, uint32_t mmax) {
  const uint32_t ng = 32u / grp_width(mmax);
  return (m + ng - 1) / ng;
}

__device__ __forceinline__ uint32_t nchunks_of(uint32_t A, uint32_t nl) {
  const uint32_t A16 = (A + 15u) & ~15u;
  return (nl * A16 + kChunk - 1) / kChunk;
}

// true when list-pass chunk [cb, ce) lies inside one list and one segment; then `u`
// holds that segment's (offL, offR) and the chunk needs no per-position offsets
__device__ __forceinline__ bool chunk_uniform(uint32_t cb, uint32_t ce, uint32_t A16, uint32_t A,
                                              const uint32_t* seg, const int2* off2, int2& u) {
  const uint32_t li = cb / A16;
  if ((ce - 1) / A16 != li) return false;
  const uint32_t k0 = cb - li * A16;
  if (k0 >= A) return false;
  const uint32_t k1 = min(ce - 1 - li * A16, A - 1);
  if (seg[k0] != seg[k1]) return false;
  u = off2[k0];
  return true;
}

// ---- batch initialisation ---------------------------------------------------------
__global__ void w_zero(const WideArgs a) {
  const SlotPtrs P = slot_ptrs(a, blockIdx.y);
  const uint32_t n = static_cast<uint32_t>(a.g.d.n);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    P.mult[i] = 0u;
}

// bootstrap draws (forest.hpp:184-195)
__global__ void w_boot(const WideArgs a) {
  const uint32_t b = blockIdx.y, tl = a.t0 + b;
  const SlotPtrs P = slot_ptrs(a, b);
  const uint32_t n = static_cast<uint32_t>(a.g.d.n);
  const uint64_t key = tree_key(a, b);
  // a hold-out fold draws local rows of its training subset (forest.hpp:184-190 on the
  // fold's own dataset) and maps them to table rows
  const uint32_t nk = tree_n(a, b);
  const uint32_t* map =
      a.g.cell_rows ? a.g.cell_rows + a.g.cell_rows_off[a.g.tree_cell[tl]] : nullptr;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nk; j += gridDim.x * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(draw_bounded(key, uint64_t{j} + 1u, nk));
    if (a.g.inbag) a.g.inbag[static_cast<size_t>(tl) * n + j] = r;
    atomicAdd(P.mult + (map ? map[r] : r), 1u);
  }
}

// in-bag bitmap + 64-row prefix counts + A0 (CTA per tree)
template <int NT>
__global__ void __launch_bounds__(NT) w_bits(const WideArgs a) {
  constexpr int NW = NT / 32;
  __shared__ uint32_t sh[NW + 2];
  const uint32_t b = blockIdx.x;
  const SlotPtrs P = slot_ptrs(a, b);
  const uint32_t n = static_cast<uint32_t>(a.g.d.n);
  const uint32_t nwords = (n + 31u) / 32u, nblk64 = (n + 63u) / 64u;
  for (uint32_t w = warp_id(); w < nwords; w += NW) {
    const uint32_t r = w * 32u + lane_id();
    const unsigned bl = __ballot_sync(kFull, r < n && P.mult[r] > 0u);
    if (lane_id() == 0) P.bits[w] = bl;
  }
  __syncthreads();
  uint32_t carry = 0;
  for (uint32_t base = 0; base < nblk64; base += NT) {
    const uint32_t i = base + threadIdx.x;
    uint32_t v = 0;
    if (i < nblk64)
      v = __popc(P.bits[2 * i]) + (2 * i + 1 < nwords ? __popc(P.bits[2 * i + 1]) : 0u);
    uint32_t tot;
    const uint32_t ex = block_excl_scan<NT>(v, sh, &tot);
    if (i < nblk64) P.pref[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    TreeState& s = a.ts[b];
    s.A = carry;
    s.F = 1;
    s.nodes = 1;
    s.done = 0;
    s.E = 0;
    s.S = 0;
    s.elig_base = 0;
    s.split_rows = 0;
    if (carry > a.g.L.stride) {
      s.done = 1;
      atomicExch(a.g.err, 2);
    }
  }
}

// payload in row order (forest.hpp:194-195)
__global__ void w_payload(const WideArgs a) {
  const uint32_t b = blockIdx.y;
  const SlotPtrs P = slot_ptrs(a, b);
  const uint32_t n = static_cast<uint32_t>(a.g.d.n);
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (!get_bit(P.bits, r)) continue;
    const uint32_t pos = inbag_pos(P.bits, P.pref, r);
    const uint32_t mu = P.mult[r];
    const double yr = __ldg(a.g.d.y + r);
    const double wy = __dmul_rn(static_cast<double>(mu), yr);
    P.pay[pos] = Payload{r, mu, wy};
    P.seg[pos] = 0u;
  }
}

// per listed column: stable in-bag filter of the presort.  Items = (tree, chunk of the
// flat (list, presort position) space); counts, then a per-tree scan, then scatter.
__global__ void w_l0count(const WideArgs a) {
  const uint32_t nl = a.g.d.nlisted, os = a.g.d.order_stride;
  const uint32_t per = (nl * os + kChunk - 1) / kChunk;
  const uint32_t total = per * a.B;
  const uint32_t n = static_cast<uint32_t>(a.g.d.n);
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = gw; it < total; it += nw) {
    const uint32_t b = it / per, c = it - b * per;
    const SlotPtrs P = slot_ptrs(a, b);
    const uint32_t ce = min(nl * os, (c + 1) * kChunk);
    uint32_t cnt = 0;
    for (uint32_t s = c * kChunk; s < ce; s += 128) {
      const uint32_t g0 = s + lane_id() * 4;
      if (g0 < ce) {
        const uint32_t k0 = g0 % os;
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(a.g.d.order + g0));
        const uint32_t r4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) cnt += (k0 + j < n) ? get_bit(P.bits, r4[j]) : 0u;
      }
    }
    cnt = warp_sum(cnt);
    if (lane_id() == 0) P.chunk[c] = cnt;
  }
}

// exclusive scan of each tree's chunk counts (CTA per tree); `which` selects the
// item space: 0 = list init, 1 = level list pass (also advances the tree's level state)
template <int NT>
__global__ void __launch_bounds__(NT) w_chunkscan(const WideArgs a, int which) {
  constexpr int NW = NT / 32;
  __shared__ uint32_t sh[NW + 2];
  const uint32_t b = blockIdx.x;
  TreeState& s = a.ts[b];
  const uint32_t nl = a.g.d.nlisted;
  if (which == 1 && s.done) return;
  const uint32_t per = which == 0 ? (nl * a.g.d.order_stride + kChunk - 1) / kChunk
                                  : nchunks_of(s.A, nl);
  const SlotPtrs P = slot_ptrs(a, b);
  uint32_t carry = 0;
  for (uint32_t base = 0; base < per; base += NT) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < per ? P.chunk[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<NT>(v, sh, &tot);
    if (i < per) P.chunk[i] = carry + ex;
    carry += tot;
  }
}

__global__ void w_l0scatter(const WideArgs a) {
  const uint32_t nl = a.g.d.nlisted, os = a.g.d.order_stride;
  const uint32_t per = (nl * os + kChunk - 1) / kChunk;
  const uint32_t total = per * a.B;
  const uint32_t n = static_cast<uint32_t>(a.g.d.n);
  const uint32_t stride = a.g.L.stride;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = gw; it < total; it += nw) {
    const uint32_t b = it / per, c = it - b * per;
    const SlotPtrs P = slot_ptrs(a, b);
    const uint32_t A0 = a.ts[b].A;
    const uint32_t ce = min(nl * os, (c + 1) * kChunk);
    uint32_t run = P.chunk[c];
    for (uint32_t s = c * kChunk; s < ce; s += 128) {
      const uint32_t g0 = s + lane_id() * 4;
      uint32_t in = 0, r4[4] = {0, 0, 0, 0}, li = 0;
      if (g0 < ce) {
        li = g0 / os;
        const uint32_t k0 = g0 - li * os;
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(a.g.d.order + g0));
        r4[0] = x.x; r4[1] = x.y; r4[2] = x.z; r4[3] = x.w;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (k0 + j < n && get_bit(P.bits, r4[j])) in |= 1u << j;
      }
      const uint32_t mine = __popc(in);
      const uint32_t inc = warp_incl_scan(mine);
      uint32_t o = run + inc - mine - li * A0;
      uint32_t* out = P.lists + static_cast<size_t>(li) * stride;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if ((in >> j) & 1u) out[o++] = inbag_pos(P.bits, P.pref, r4[j]);
      run += __shfl_sync(kFull, inc, 31);
    }
  }
}

// root sums in row order (forest.hpp:221-226), warp per tree
__global__ void w_root(const WideArgs a) {
  __shared__ double st[64];
  const uint32_t b = blockIdx.x;
  const SlotPtrs P = slot_ptrs(a, b);
  TreeState& s = a.ts[b];
  if (s.done) return;
  double sum, sq;
  root_sums_warp<4>(P.pay, a.g.d.y, s.A, sum, sq, st);
  if (lane_id() == 0) {
    P.front[0] = NodeWork{0u, s.A, 0u, 0u, static_cast<double>(tree_n(a, b)), sum, sq};
    P.nf[0] = -1;
    P.nthr[0] = 0.0;
    P.nleft[0] = -1;
    P.nval[0] = 0.0;
    P.nrank[0] = 0u;
  }
}

// ---- level kernels ----------------------------------------------------------------
// leaf tests, eligible compaction, mtry sampling, bitmap reset (CTA per tree)
template <int NT>
__global__ void __launch_bounds__(NT) w_front(const WideArgs a) {
  constexpr int NW = NT / 32;
  __shared__ uint32_t sh[NW + 2];
  const uint32_t b = blockIdx.x;
  TreeState& s = a.ts[b];
  if (s.done) return;
  const SlotPtrs P = slot_ptrs(a, b);
  const NodeWork* fr = P.front;
  const uint32_t F = s.F, A = s.A, m = tree_m(a, b), p = a.g.d.p;
  const uint32_t n = tree_n(a, b);  // mtry draws continue after the n bootstrap draws
  uint32_t carry = 0;
  for (uint32_t base = 0; base < F; base += NT) {
    const uint32_t f = base + threadIdx.x;
    uint32_t el = 0;
    if (f < F) {
      const NodeWork nw = fr[f];
      const double sse = __dsub_rn(nw.q, __ddiv_rn(__dmul_rn(nw.s, nw.s), nw.w));
      const bool too_small = nw.w < 2.0 * static_cast<double>(tree_mns(a, b));
      const bool pure = sse <= __dmul_rn(1e-12, nw.q > 1.0 ? nw.q : 1.0);
      if (too_small || pure)
        P.nval[nw.id] = __ddiv_rn(nw.s, nw.w);
      else
        el = 1;
      P.segtab[f].offL = INT_MIN;
    }
    uint32_t tot;
    const uint32_t ex = block_excl_scan<NT>(el, sh, &tot);
    if (el) P.e2f[carry + ex] = f;
    carry += tot;
  }
  const uint32_t E = carry;
  const uint64_t key = tree_key(a, b);
  for (uint32_t e = threadIdx.x; e < E; e += NT) {
    uint16_t pool[kMaxP];
    for (uint32_t c = 0; c < p; ++c) pool[c] = static_cast<uint16_t>(c);
    const uint64_t ctr = uint64_t{n} + (s.elig_base + e) * m;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t j = i + static_cast<uint32_t>(draw_bounded(key, ctr + i + 1, p - i));
      const uint16_t tmp = pool[i];
      pool[i] = pool[j];
      pool[j] = tmp;
    }
    for (uint32_t i = 1; i < m; ++i)
      for (uint32_t k = i; k > 0 && pool[k - 1] > pool[k]; --k) {
        const uint16_t tmp = pool[k];
        pool[k] = pool[k - 1];
        pool[k - 1] = tmp;
      }
    for (uint32_t i = 0; i < m; ++i) P.samp[static_cast<size_t>(e) * m + i] = pool[i];
  }
  // eligible nodes by size class, BFS order inside each: [0, E0) small (< kLaneMax
  // rows: lane per chain), [E0, E0+E1) mid (lane groups), then big (warp per chain)
  uint32_t base = 0, E0 = 0, E1 = 0, E2 = 0;
  for (uint32_t cls = 0; cls < 3; ++cls) {
    carry = 0;
    for (uint32_t b0 = 0; b0 < E; b0 += NT) {
      const uint32_t e = b0 + threadIdx.x;
      uint32_t in = 0;
      if (e < E) {
        const NodeWork& nw = fr[P.e2f[e]];
        const uint32_t R = nw.e - nw.b;
        const uint32_t c = R < a.lane_max ? 0u : (R < a.big_min ? 1u : 2u);
        in = c == cls;
      }
      uint32_t tot;
      const uint32_t ex = block_excl_scan<NT>(in, sh, &tot);
      if (in) P.ecls[base + carry + ex] = e;
      carry += tot;
    }
    if (cls == 0) E0 = carry;
    if (cls == 1) E1 = carry;
    if (cls == 2) E2 = carry;
    base += carry;
  }
  for (uint32_t w = threadIdx.x; w < (A + 31u) / 32u; w += NT) P.bits[w] = 0u;
  if (threadIdx.x == 0) {
    s.E = E;
    s.E0 = E0;
    s.E1 = E1;
    s.E2 = E2;
  }
}

// exclusive prefixes over trees of this level's work items (one CTA)
//   which 0: chain tasks (lane, group, warp);  which 1: CTA-routed splits, splits S,
//   positions A, list chunks
template <int NT>
__global__ void __launch_bounds__(NT) w_prefix(const WideArgs a, int which) {
  constexpr int NW = NT / 32;
  __shared__ uint32_t sh[NW + 2];
  uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
  for (uint32_t base = 0; base < a.B; base += NT) {
    const uint32_t b = base + threadIdx.x;
    uint32_t v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0;
    if (b < a.B && !a.ts[b].done) {
      const TreeState& s = a.ts[b];
      if (which == 0) {  // chain tasks: lane (small), group (mid), warp (big)
        const uint32_t m = tree_m(a, b);
        v0 = s.E0 * m;
        v1 = s.E1 * grp_tpn(m, a.g.mtry);
        v2 = s.E2 * m;
      } else {
        v0 = s.Sbig;
        v1 = s.S;
        v2 = s.A;
        v3 = nchunks_of(s.A, a.g.d.nlisted);
        v4 = s.Swarp;
      }
    }
    uint32_t t0, t1, t2, t3;
    const uint32_t e0 = block_excl_scan<NT>(v0, sh, &t0);
    const uint32_t e1 = block_excl_scan<NT>(v1, sh, &t1);
    const uint32_t e2 = block_excl_scan<NT>(v2, sh, &t2);
    const uint32_t e3 = block_excl_scan<NT>(v3, sh, &t3);
    uint32_t t4;
    const uint32_t e4 = block_excl_scan<NT>(v4, sh, &t4);
    if (b < a.B) {
      a.off[0][b] = c0 + e0;
      a.off[1][b] = c1 + e1;
      a.off[2][b] = c2 + e2;
      a.off[3][b] = c3 + e3;
      if (which == 1) a.off[4][b] = c4 + e4;
    }
    c0 += t0;
    c1 += t1;
    c2 += t2;
    c3 += t3;
    c4 += t4;
  }
  if (threadIdx.x == 0) {
    if (which == 1) {
      a.off[4][a.B] = c4;
      a.task_ctr[2] = 0u;
    }
    if (which == 0) a.task_ctr[0] = a.task_ctr[1] = a.task_ctr[3] = 0u;
    a.off[0][a.B] = c0;
    a.off[1][a.B] = c1;
    a.off[2][a.B] = c2;
    a.off[3][a.B] = c3;
  }
}

// split chains (forest.hpp:268-297), three kernels over the size classes of w_front:
// big nodes (>= big_min rows) run one warp per (node, column) ...
#ifndef AIWC_BIG_U
#define AIWC_BIG_U 4
#endif
#ifndef AIWC_ROUTE_G
#define AIWC_ROUTE_G 3
#endif
constexpr int kBigU = AIWC_BIG_U;     // positions per lane per round of the big-node chains
constexpr int kRouteG = AIWC_ROUTE_G;  // 32-position tiles per round of the warp route
#ifndef AIWC_GRP_U
#define AIWC_GRP_U 4
#endif
constexpr int kGrpU = AIWC_GRP_U;  // positions per lane per round of the mid-node chains
template <typename RankT, int GB>  // GB lanes per chain: 32 (warp_p) or 16 / 8 (lane groups)
__global__ void __launch_bounds__(256) w_chains_warp(const WideArgs a) {
  constexpr int UB = kBigU;  // positions per lane per round of the big-node lane groups
  __shared__ double stage[8][GB == 32 ? 64 : 32 * UB];
  const uint32_t total = a.off[2][a.B];
  const uint32_t n = static_cast<uint32_t>(a.g.d.n), stride = a.g.L.stride;
  const RankT* rank = static_cast<const RankT*>(a.g.d.rank);
  // tasks are claimed dynamically (chains differ in length by orders of magnitude)
  for (;;) {
    uint32_t t = 0;
    if (lane_id() == 0) t = atomicAdd(a.task_ctr, 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= total) break;
    const uint32_t b = owner(a.off[2], a.B, t), k = t - a.off[2][b];
    const uint32_t m = tree_m(a, b);
    const SlotPtrs P = slot_ptrs(a, b);
    const TreeState& st = a.ts[b];
    const uint32_t e = P.ecls[st.E0 + st.E1 + k / m];  // class 2
    const uint32_t slot = e * m + k % m;
    const NodeWork nw_ = P.front[P.e2f[e]];
    if (nw_.e - nw_.b >= a.coop_min) continue;  // w_chains_coop
    if (GB < 32) {  // 32/GB lane groups: sampled columns j .. j+32/GB-1 of the node
      constexpr uint32_t NG = 32 / GB;
      const uint32_t j = k % m;
      if (j % NG) continue;
      const uint32_t grp = lane_id() / GB, jj = j + grp;
      const bool act = jj < m;
      const uint32_t c = act ? P.samp[e * m + jj] : 0u;
      const int32_t li = a.g.d.list_of[c];
      double bg;
      uint32_t bp;
      chain_grp<RankT, (GB < 32 ? GB : 16), UB>(
          act, li >= 0, P.lists + static_cast<size_t>(li >= 0 ? li : 0) * stride, nw_.b,
          nw_.e, P.pay, rank + static_cast<size_t>(c) * n, nw_.w, nw_.s, bg, bp,
          stage[warp_id()] + grp * UB * GB);
      if (act && (lane_id() % GB) == 0) P.res[e * m + jj] = ChainRes{bg, bp, 0u};
      continue;
    }
    const uint32_t c = P.samp[slot];
    const int32_t li = a.g.d.list_of[c];
    const RankT* rk_c = rank + static_cast<size_t>(c) * n;
    double bg;
    uint32_t bp;
    chain_warp_p<RankT, 2>(li >= 0, P.lists + static_cast<size_t>(li >= 0 ? li : 0) * stride,
                           nw_.b, nw_.e, P.pay, rk_c, nw_.w, nw_.s, bg, bp, stage[warp_id()]);
    if (lane_id() == 0) P.res[slot] = ChainRes{bg, bp, 0u};
  }
}

// Huge split nodes (>= coop_min rows, column 0 listed) are routed by a whole CTA:
// three producer warps gather blocks of kCoopBlock positions while warp 0 sums.
// (The CTA-per-node kernels shorten each node's critical path but spend 4 warps per
// chain: they pay off only when a lane's batch is small; the host sets coop_min.)
constexpr int kCoopPerLane = 4;
constexpr uint32_t kCoopBlock = 3 * 32 * kCoopPerLane;  // positions per block

// ... and huge nodes (>= coop_min rows) one CTA per (node, column), with the chain's
// sequential FP64 adds alone on one warp: a chain step costs one DADD latency (8 cycles
// on B200) only if nothing else sits on that warp's critical path, so three producer
// warps gather each block of kCB positions (list -> payload -> rank) into shared memory,
// warp 0 runs the chain over the block writing the running value before every position,
// and the producers then derive the integer weight prefix, the value boundaries and the
// gains of that block from it.  Blocks flow through three shared-memory stages: while
// warp 0 chains block i, the producers fill block i+1 and score block i-1.
constexpr int kCoopW = 3;                                // producer warps
constexpr int kCoopE = 4;                                // positions per producer lane
constexpr uint32_t kCB = kCoopW * 32 * kCoopE;           // positions per block
struct CoopStage {
  double wy[kCB];   // addends (two-level chains: +0.0 for value-1 rows)
  double pre[kCB];  // running sum before each position (written by warp 0)
  uint32_t mu[kCB];
  uint32_t rk[kCB];
};

template <typename RankT>
__global__ void __launch_bounds__(128) w_chains_coop(const WideArgs a) {
  __shared__ CoopStage S[3];
  __shared__ uint32_t s_task, s_wsum[kCoopW], s_n0;
  __shared__ double s_sl, s_bg[kCoopW];
  __shared__ uint32_t s_w0;
  __shared__ uint32_t s_bp[kCoopW];
  const uint32_t total = a.off[2][a.B];
  const uint32_t n = static_cast<uint32_t>(a.g.d.n), stride = a.g.L.stride;
  const RankT* rank = static_cast<const RankT*>(a.g.d.rank);
  const unsigned lane = lane_id(), wid = warp_id();
  const uint32_t pt = threadIdx.x - 32;  // producer thread index (wid > 0)
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(a.task_ctr + 1, 1u);
    __syncthreads();
    const uint32_t t = s_task;
    __syncthreads();
    if (t >= total) break;
    const uint32_t b = owner(a.off[2], a.B, t), k = t - a.off[2][b];
    const uint32_t m = tree_m(a, b);
    const SlotPtrs P = slot_ptrs(a, b);
    const TreeState& ts = a.ts[b];
    const uint32_t e = P.ecls[ts.E0 + ts.E1 + k / m];
    const uint32_t slot = e * m + k % m;
    const NodeWork nw = P.front[P.e2f[e]];
    if (nw.e - nw.b < a.coop_min) continue;  // CTA-uniform: w_chains_warp's task
    const uint32_t c = P.samp[slot];
    const int32_t li = a.g.d.list_of[c];
    const bool listed = li >= 0;
    const uint32_t* list = P.lists + static_cast<size_t>(listed ? li : 0) * stride;
    const RankT* rk_c = rank + static_cast<size_t>(c) * n;
    const uint32_t R = nw.e - nw.b, nblk = (R + kCB - 1) / kCB;
    // producers: a register pipeline over blocks -- at step i a producer lane writes
    // block i+1 (ranks gathered at step i-1) into its stage, gathers the ranks of block
    // i+2, the payload of block i+3 and the list entries of block i+4
    uint32_t q4[kCoopE] = {}, row3[kCoopE] = {}, mu3[kCoopE] = {}, mu2[kCoopE] = {},
             rk2[kCoopE] = {}, mu1[kCoopE] = {}, rk1[kCoopE] = {};
    double wy3[kCoopE] = {}, wy2[kCoopE] = {}, wy1[kCoopE] = {};
    auto pos = [&](int64_t blk, int j) -> int64_t {
      return blk * kCB + (wid - 1) * 32 * kCoopE + j * 32 + lane;
    };
    auto step = [&](int64_t i) {
#pragma unroll
      for (int j = 0; j < kCoopE; ++j) {  // (mu1, wy1, rk1) <- block i+1 (ranks from step i-1)
        mu1[j] = mu2[j];
        wy1[j] = wy2[j];
        rk1[j] = rk2[j];
      }
      if (i + 1 >= 0 && i + 1 < nblk) {  // block i+1 -> shared memory
        CoopStage& st = S[(i + 1) % 3];
#pragma unroll
        for (int j = 0; j < kCoopE; ++j) {
          const int64_t x = pos(i + 1, j);
          uint32_t mu = x < R ? mu1[j] : 0u;
          double wy = x < R ? wy1[j] : 0.0;
          if (!listed && rk1[j] != 0u) {  // two-level: only value-0 rows enter the chain
            mu = 0u;
            wy = 0.0;
          }
          const uint32_t idx = static_cast<uint32_t>(x - (i + 1) * kCB);
          st.wy[idx] = wy;
          st.mu[idx] = mu;
          st.rk[idx] = rk1[j];
        }
      }
#pragma unroll
      for (int j = 0; j < kCoopE; ++j) {  // ranks of block i+2
        const int64_t x = pos(i + 2, j);
        mu2[j] = mu3[j];
        wy2[j] = wy3[j];
        rk2[j] = (x >= 0 && x < R) ? rank_of(rk_c, row3[j]) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kCoopE; ++j) {  // payload of block i+3
        const int64_t x = pos(i + 3, j);
        if (x >= 0 && x < R) {
          const Payload pv = P.pay[q4[j]];
          row3[j] = pv.row;
          mu3[j] = pv.mult;
          wy3[j] = pv.wy;
        } else {
          row3[j] = 0u;
          mu3[j] = 0u;
          wy3[j] = 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < kCoopE; ++j) {  // list entries of block i+4
        const int64_t x = pos(i + 4, j);
        q4[j] = (x >= 0 && x < R) ? (listed ? list[nw.b + x] : nw.b + static_cast<uint32_t>(x)) : 0u;
      }
    };
    // producer scoring state: weight prefix carry, last rank, best gain (first max)
    uint32_t wcarry = 0, last_rk = 0, n0 = 0;
    double bg = -INFINITY;
    uint32_t bp = 0xffffffffu;
    auto score = [&](uint32_t blk) {
      const CoopStage& st = S[blk % 3];
      const uint32_t i0 = blk * kCB + pt * kCoopE;  // kCoopE consecutive positions
      uint32_t mu[kCoopE], loc = 0;
#pragma unroll
      for (int j = 0; j < kCoopE; ++j) {
        mu[j] = i0 + j < R ? st.mu[pt * kCoopE + j] : 0u;
        loc += mu[j];
      }
      // exclusive prefix of the producer threads' sums (3 warps, producer-only barrier)
      const uint32_t inc = warp_incl_scan(loc);
      if (lane == 31) s_wsum[wid - 1] = inc;
      asm volatile("bar.sync 1, 96;" ::: "memory");
      uint32_t wpre = 0, btot = 0;
#pragma unroll
      for (int w = 0; w < kCoopW; ++w) {
        wpre += (w < static_cast<int>(wid) - 1) ? s_wsum[w] : 0u;
        btot += s_wsum[w];
      }
      uint32_t wb = wcarry + wpre + inc - loc;
      if (listed) {
        uint32_t prk = pt == 0 ? last_rk : st.rk[pt * kCoopE - 1];
#pragma unroll
        for (int j = 0; j < kCoopE; ++j) {
          const uint32_t i = i0 + j;
          if (i >= R) break;
          const uint32_t rk = st.rk[pt * kCoopE + j];
          if (i > 0 && rk != prk) {
            const double gn = gain_at(st.pre[pt * kCoopE + j], static_cast<double>(wb), nw.w, nw.s);
            if (gn > bg) {
              bg = gn;
              bp = nw.b + i;
            }
          }
          wb += mu[j];
          prk = rk;
        }
        const uint32_t nlast = min(kCB, R - blk * kCB);
        last_rk = st.rk[nlast - 1];
      } else {
#pragma unroll
        for (int j = 0; j < kCoopE; ++j)
          if (i0 + j < R && st.rk[pt * kCoopE + j] == 0u) ++n0;
      }
      wcarry += btot;
      asm volatile("bar.sync 1, 96;" ::: "memory");  // s_wsum reuse
    };
    if (wid > 0)
      for (int64_t i = -4; i < 0; ++i) step(i);
    __syncthreads();
    double r = 0.0;  // warp 0: the chain
    for (uint32_t i = 0; i <= nblk; ++i) {
      if (wid == 0) {
        if (i < nblk) {
          CoopStage& st = S[i % 3];
          constexpr int kW = 8;
          double buf[kW];
#pragma unroll
          for (int j = 0; j < kW; ++j) buf[j] = st.wy[j];
#pragma unroll 16
          for (uint32_t j = 0; j < kCB; ++j) {
            const double x = buf[j % kW];
            if (j + kW < kCB) buf[j % kW] = st.wy[j + kW];
            if (lane == 0) st.pre[j] = r;
            r = __dadd_rn(r, x);
          }
        }
      } else {
        step(i);
        if (i >= 1) score(i - 1);
      }
      __syncthreads();
    }
    // reduce the producers' best (first max: larger gain, then smaller position)
    if (wid > 0) {
      double g = bg;
      uint32_t q = bp;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double og = __shfl_xor_sync(kFull, g, o);
        const uint32_t op = __shfl_xor_sync(kFull, q, o);
        if (og > g || (og == g && op < q)) {
          g = og;
          q = op;
        }
        n0 += __shfl_xor_sync(kFull, n0, o);
      }
      if (lane == 0) {
        s_bg[wid - 1] = g;
        s_bp[wid - 1] = q;
        s_wsum[wid - 1] = n0;
      }
      if (pt == 0) s_w0 = wcarry;  // every producer carries the same weight total
    } else if (lane == 0) {
      s_sl = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double g = -INFINITY;
      uint32_t q = 0xffffffffu, z = 0;
      for (int w = 0; w < kCoopW; ++w) {
        if (s_bg[w] > g || (s_bg[w] == g && s_bp[w] < q)) {
          g = s_bg[w];
          q = s_bp[w];
        }
        z += s_wsum[w];
      }
      if (!listed) {
        if (z == 0 || z == R) {
          g = -INFINITY;
          q = 0xffffffffu;
        } else {
          g = gain_at(s_sl, static_cast<double>(s_w0), nw.w, nw.s);
          q = nw.b + z;
        }
      }
      P.res[slot] = ChainRes{g, q, 0u};
    }
    __syncthreads();
  }
}

// ... mid nodes run one warp per node (or per group of 32/G of its columns), G lanes
// per column (chain_grp) ...
template <typename RankT, int G, int U>
__global__ void __launch_bounds__(256) w_chains_grp(const WideArgs a) {
  __shared__ double stage[8][32 * U];
  const uint32_t total = a.off[1][a.B];
  const uint32_t n = static_cast<uint32_t>(a.g.d.n), stride = a.g.L.stride;
  const uint32_t grp = lane_id() / G;
  const RankT* rank = static_cast<const RankT*>(a.g.d.rank);
  for (;;) {  // tasks claimed dynamically
    uint32_t t = 0;
    if (lane_id() == 0) t = atomicAdd(a.task_ctr + 3, 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= total) break;
    const uint32_t b = owner(a.off[1], a.B, t), k = t - a.off[1][b];
    const uint32_t m = tree_m(a, b), tpn = grp_tpn(m, a.g.mtry);
    const SlotPtrs P = slot_ptrs(a, b);
    const TreeState& st = a.ts[b];
    const uint32_t e = P.ecls[st.E0 + k / tpn];
    const uint32_t j = (k % tpn) * (32 / G) + grp;  // sampled-column index of this group
    const bool act = j < m;
    const NodeWork nw_ = P.front[P.e2f[e]];
    const uint32_t c = act ? P.samp[e * m + j] : 0u;
    const int32_t li = a.g.d.list_of[c];
    const RankT* rk_c = rank + static_cast<size_t>(c) * n;
    const uint32_t* list = P.lists + static_cast<size_t>(li >= 0 ? li : 0) * stride;
    double bg;
    uint32_t bp;
    chain_grp<RankT, G, U>(act, li >= 0, list, nw_.b, nw_.e, P.pay, rk_c, nw_.w, nw_.s,
                           bg, bp, stage[warp_id()] + grp * G * U);
    if (act && (lane_id() & (G - 1)) == 0) P.res[e * m + j] = ChainRes{bg, bp, 0u};
  }
}

// ... and small nodes (< kLaneMax rows) one lane per chain
template <typename RankT>
__global__ void __launch_bounds__(256) w_chains_lane(const WideArgs a) {
  const uint32_t total = a.off[0][a.B];
  const uint32_t n = static_cast<uint32_t>(a.g.d.n), stride = a.g.L.stride;
  const RankT* rank = static_cast<const RankT*>(a.g.d.rank);
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const uint32_t b = owner(a.off[0], a.B, t), k = t - a.off[0][b];
    const uint32_t m = tree_m(a, b);
    const SlotPtrs P = slot_ptrs(a, b);
    const uint32_t e = P.ecls[k / m];
    const uint32_t slot = e * m + k % m;
    const NodeWork nw_ = P.front[P.e2f[e]];
    const uint32_t c = P.samp[slot];
    const int32_t li = a.g.d.list_of[c];
    const RankT* rk_c = rank + static_cast<size_t>(c) * n;
    double bg;
    uint32_t bp;
    if (li >= 0)
      chain_lane<RankT>(P.lists + static_cast<size_t>(li) * stride, nw_.b, nw_.e,
                        P.pay, rk_c, nw_.w, nw_.s, bg, bp);
    else
      chain_bin_lane<RankT>(P.pay, nw_.b, nw_.e, rk_c, nw_.w, nw_.s, bg, bp);
    P.res[slot] = ChainRes{bg, bp, 0u};
  }
}

// decide + BFS numbering (forest.hpp:299-319), CTA per tree
template <int NT, typename RankT>
__global__ void __launch_bounds__(NT) w_decide(const WideArgs a) {
  constexpr int NW = NT / 32;
  __shared__ uint32_t sh[NW + 2];
  const uint32_t b = blockIdx.x;
  TreeState& st = a.ts[b];
  if (st.done) return;
  const SlotPtrs P = slot_ptrs(a, b);
  const DevData& d = a.g.d;
  const uint32_t n = static_cast<uint32_t>(d.n), m = tree_m(a, b), stride = a.g.L.stride;
  const RankT* rank = static_cast<const RankT*>(d.rank);
  const NodeWork* fr = P.front;
  const uint32_t E = st.E, nodes0 = st.nodes;
  const bool coop_route = d.list_of[0] >= 0;
  uint32_t carry = 0, ccarry = 0, bcarry = 0, wcarry = 0;
  for (uint32_t base = 0; base < E; base += NT) {
    const uint32_t e = base + threadIdx.x;
    uint32_t sp = 0, c = 0, thr_rank = 0;
    double thr = 0.0;
    NodeWork nw{};
    if (e < E) {
      nw = fr[P.e2f[e]];
      double bg = -INFINITY;
      uint32_t bi = 0, bp = 0;
      for (uint32_t i = 0; i < m; ++i) {
        const ChainRes r = P.res[static_cast<size_t>(e) * m + i];
        if (r.gain > bg) {
          bg = r.gain;
          bi = i;
          bp = r.pos;
        }
      }
      if (bg == -INFINITY) {
        P.nval[nw.id] = __ddiv_rn(nw.s, nw.w);
      } else {
        sp = 1;
        c = P.samp[static_cast<size_t>(e) * m + bi];
        const int32_t li = d.list_of[c];
        const double* vals = d.vals + d.vals_off[c];
        double prev, v;
        uint32_t lo, hi;
        if (li >= 0) {
          const uint32_t* lc = P.lists + static_cast<size_t>(li) * stride;
          const uint32_t r1 = P.pay[lc[bp - 1]].row;
          const uint32_t r0 = P.pay[lc[bp]].row;
          prev = d.col[static_cast<size_t>(c) * n + r1];
          v = d.col[static_cast<size_t>(c) * n + r0];
          lo = rank_of(rank + static_cast<size_t>(c) * n, r1);
          hi = rank_of(rank + static_cast<size_t>(c) * n, r0);
        } else {
          prev = vals[0];
          v = vals[1];
          lo = 0;
          hi = 1;
        }
        thr = __dadd_rn(prev, __ddiv_rn(__dsub_rn(v, prev), 2.0));
        if (thr >= v) thr = prev;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (vals[mid] <= thr) lo = mid; else hi = mid;
        }
        thr_rank = lo;
      }
    }
    uint32_t tot;
    const uint32_t ex = block_excl_scan<NT>(sp, sh, &tot);
    const uint32_t cnt = sp ? nw.e - nw.b : 0u;
    uint32_t ctot;
    const uint32_t cex = block_excl_scan<NT>(cnt, sh, &ctot);
    // splits routed by a whole CTA (w_route_coop), compacted into ecls (free after the
    // chain kernels)
    const uint32_t big = sp && coop_route && cnt >= a.coop_min ? 1u : 0u;
    uint32_t btot;
    const uint32_t bex = block_excl_scan<NT>(big, sh, &btot);
    if (big) P.ecls[bcarry + bex] = carry + ex;
    bcarry += btot;
    const uint32_t wsp = sp && !big && cnt >= kLaneMax ? 1u : 0u;  // warp-routed splits
    uint32_t wtot;
    const uint32_t wex = block_excl_scan<NT>(wsp, sh, &wtot);
    if (wsp) P.wsplit[wcarry + wex] = carry + ex;
    wcarry += wtot;
    if (sp) {
      const uint32_t s = carry + ex;
      const uint32_t child = nodes0 + 2 * s;
      if (child + 1 < a.g.L.nodes_cap) {
        P.nf[nw.id] = static_cast<int32_t>(c);
        P.nthr[nw.id] = thr;
        P.nleft[nw.id] = static_cast<int32_t>(child);
        P.nrank[nw.id] = thr_rank;
        for (uint32_t h = 0; h < 2; ++h) {
          P.nf[child + h] = -1;
          P.nthr[child + h] = 0.0;
          P.nleft[child + h] = -1;
          P.nval[child + h] = 0.0;
          P.nrank[child + h] = 0u;
        }
      }
      P.spl[s] = SplitInfo{P.e2f[e], c, thr_rank, cnt, 0u, ccarry + cex, 0u, 0u};
    }
    carry += tot;
    ccarry += ctot;
  }
  if (threadIdx.x == 0) {
    st.S = carry;
    st.Sbig = bcarry;
    st.Swarp = wcarry;
    st.A_next = ccarry;
    st.split_rows += ccarry;
    st.elig_base += E;
    st.nodes = nodes0 + 2 * carry;
    if (carry == 0) {
      st.done = 1;
    } else if (st.nodes > a.g.L.nodes_cap || 2 * carry > a.g.L.fmax) {
      st.done = 1;
      atomicExch(a.g.err, 3);
    } else {
      atomicAdd(a.active, 1u);
    }
  }
}

// route in column-0 order (forest.hpp:323-352): warps take split nodes >= kLaneMax
template <typename RankT, bool kWarp>
__global__ void __launch_bounds__(256) w_route(const WideArgs a) {
  __shared__ double stage[8][128];
  const uint32_t total = a.off[1][a.B];
  const uint32_t n = static_cast<uint32_t>(a.g.d.n), stride = a.g.L.stride;
  const RankT* rank = static_cast<const RankT*>(a.g.d.rank);
  const int32_t list0 = a.g.d.list_of[0];
  const uint32_t k0levels = static_cast<uint32_t>(a.g.d.vals_off[1] - a.g.d.vals_off[0]);
  // warps claim the compacted warp-routed splits dynamically; lanes stride over all
  // splits and take the small ones
  const uint32_t wtotal = a.off[4][a.B];
  const uint32_t id = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t it = id;; it += step) {
    uint32_t b, s;
    if (kWarp) {
      uint32_t t = 0;
      if (lane_id() == 0) t = atomicAdd(a.task_ctr + 2, 1u);
      t = __shfl_sync(kFull, t, 0);
      if (t >= wtotal) break;
      b = owner(a.off[4], a.B, t);
      s = slot_ptrs(a, b).wsplit[t - a.off[4][b]];
    } else {
      if (it >= total) break;
      b = owner(a.off[1], a.B, it);
      s = it - a.off[1][b];
    }
    const SlotPtrs P = slot_ptrs(a, b);
    const SplitInfo si = P.spl[s];
    if (!kWarp && si.cnt >= kLaneMax) continue;
    const NodeWork nw = P.front[si.f];
    const RankT* rk_f = rank + static_cast<size_t>(si.c) * n;
    const uint32_t* l0 = list0 >= 0 ? P.lists + static_cast<size_t>(list0) * stride : nullptr;
    RouteOut o{0, 0, 0, 0.0, 0.0, 0.0, 0.0};
    if (kWarp) {
      if (l0)
        route_warp_p<RankT, kRouteG>(l0, nw.b, nw.e, P.pay, a.g.d.y, rk_f, si.thr_rank,
                               P.bits, o, stage[warp_id()]);
      else
        route_groups_warp<RankT, 4>(P.pay, a.g.d.y, nw.b, nw.e, rank, k0levels,
                                    rk_f, si.thr_rank, P.bits, o, stage[warp_id()]);
      if (lane_id() != 0) continue;
    } else {
      if (l0)
        route_lane<RankT>(l0, nw.b, nw.e, P.pay, a.g.d.y, rk_f, si.thr_rank, P.bits, o);
      else
        route_groups_lane<RankT>(P.pay, a.g.d.y, nw.b, nw.e, rank, k0levels, rk_f,
                                 si.thr_rank, P.bits, o);
    }
    P.spl[s].nl = o.nl;
    const uint32_t child = static_cast<uint32_t>(P.nleft[nw.id]);
    P.front_n[2 * s] = NodeWork{si.base, si.base + o.nl, child, 0u,
                                   static_cast<double>(o.wl), o.sl, o.ql};
    P.front_n[2 * s + 1] = NodeWork{si.base + o.nl, si.base + si.cnt, child + 1, 0u,
                                       static_cast<double>(o.wr), o.sr, o.qr};
  }
}

// route of huge split nodes (column 0 listed): one CTA per node, three producer warps
// gather blocks (list-0 entry -> payload -> y of the row and split-column rank), set the goes-left
// bits and stage the four masked addend streams; warp 0 runs the four sequential sums
// (one 8-lane group each) over the previous block
template <typename RankT>
__global__ void __launch_bounds__(128) w_route_coop(const WideArgs a) {
  __shared__ double s_a[2][4][kCoopBlock];
  __shared__ uint32_t s_cnt[3];
  const uint32_t total = a.off[0][a.B];
  const uint32_t n = static_cast<uint32_t>(a.g.d.n), stride = a.g.L.stride;
  const RankT* rank = static_cast<const RankT*>(a.g.d.rank);
  const int32_t list0 = a.g.d.list_of[0];
  const unsigned lane = lane_id(), wid = warp_id();
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t b = owner(a.off[0], a.B, t), k = t - a.off[0][b];
    const SlotPtrs P = slot_ptrs(a, b);
    const uint32_t s = P.ecls[k];
    const SplitInfo si = P.spl[s];
    const NodeWork nw = P.front[si.f];
    const RankT* rk_f = rank + static_cast<size_t>(si.c) * n;
    const uint32_t* l0 = P.lists + static_cast<size_t>(list0) * stride;
    const uint32_t nblk = (nw.e - nw.b + kCoopBlock - 1) / kCoopBlock;
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    uint32_t c_nl = 0, c_wl = 0, c_wr = 0;  // producer lanes' integer counts
    auto produce = [&](uint32_t blk) {
      const uint32_t base = nw.b + blk * kCoopBlock + (wid - 1) * 32 * kCoopPerLane;
      uint32_t q[kCoopPerLane];
      Payload pv[kCoopPerLane];
      double yy[kCoopPerLane];
#pragma unroll
      for (int j = 0; j < kCoopPerLane; ++j) {
        const uint32_t kk = base + j * 32 + lane;
        q[j] = kk < nw.e ? l0[kk] : 0u;
      }
#pragma unroll
      for (int j = 0; j < kCoopPerLane; ++j)
        if (base + j * 32 + lane < nw.e) {
          pv[j] = P.pay[q[j]];
          yy[j] = __dmul_rn(pv[j].wy, __ldg(a.g.d.y + pv[j].row));
        }
#pragma unroll
      for (int j = 0; j < kCoopPerLane; ++j) {
        const uint32_t kk = base + j * 32 + lane;
        if (kk >= nw.e) continue;
        const uint32_t idx = kk - nw.b - blk * kCoopBlock;
        const bool left = rank_of(rk_f, pv[j].row) <= si.thr_rank;
        if (left) {
          atomicOr(P.bits + (q[j] >> 5), 1u << (q[j] & 31u));
          ++c_nl;
          c_wl += pv[j].mult;
        } else {
          c_wr += pv[j].mult;
        }
        s_a[blk & 1u][0][idx] = left ? pv[j].wy : 0.0;
        s_a[blk & 1u][1][idx] = left ? yy[j] : 0.0;
        s_a[blk & 1u][2][idx] = left ? 0.0 : pv[j].wy;
        s_a[blk & 1u][3][idx] = left ? 0.0 : yy[j];
      }
    };
    if (wid > 0) produce(0);
    __syncthreads();
    double acc = 0.0;  // warp 0: group g = lane / 8 sums stream g
    for (uint32_t blk = 0; blk < nblk; ++blk) {
      if (wid == 0) {
        const uint32_t cntb = min(kCoopBlock, nw.e - nw.b - blk * kCoopBlock);
        const double* sg = s_a[blk & 1u][lane >> 3];
        double r = acc;
        uint32_t i = 0;
        for (; i + 32 <= cntb; i += 32) {
#pragma unroll
          for (int j = 0; j < 32; ++j) r = __dadd_rn(r, sg[i + j]);
        }
        for (; i < cntb; ++i) r = __dadd_rn(r, sg[i]);
        acc = r;
      } else if (blk + 1 < nblk) {
        produce(blk + 1);
      }
      __syncthreads();
    }
    if (wid > 0) {
      c_nl = warp_sum(c_nl);
      c_wl = warp_sum(c_wl);
      c_wr = warp_sum(c_wr);
      if (lane == 0) {
        atomicAdd(&s_cnt[0], c_nl);
        atomicAdd(&s_cnt[1], c_wl);
        atomicAdd(&s_cnt[2], c_wr);
      }
    }
    __syncthreads();
    if (wid == 0) {
      const double sl = __shfl_sync(kFull, acc, 0), ql = __shfl_sync(kFull, acc, 8);
      const double sr = __shfl_sync(kFull, acc, 16), qr = __shfl_sync(kFull, acc, 24);
      if (lane == 0) {
        const uint32_t nl = s_cnt[0];
        P.spl[s].nl = nl;
        const uint32_t child = static_cast<uint32_t>(P.nleft[nw.id]);
        P.front_n[2 * s] = NodeWork{si.base, si.base + nl, child, 0u,
                                    static_cast<double>(s_cnt[1]), sl, ql};
        P.front_n[2 * s + 1] = NodeWork{si.base + nl, si.base + si.cnt, child + 1, 0u,
                                        static_cast<double>(s_cnt[2]), sr, qr};
      }
    }
    __syncthreads();
  }
}

// segment table + per-word prefix of the goes-left bitmap (CTA per tree)
template <int NT>
__global__ void __launch_bounds__(NT) w_segtab(const WideArgs a) {
  constexpr int NW = NT / 32;
  __shared__ uint32_t sh[NW + 2];
  const uint32_t b = blockIdx.x;
  TreeState& st = a.ts[b];
  if (st.done) return;
  const SlotPtrs P = slot_ptrs(a, b);
  const NodeWork* fr = P.front;
  const uint32_t S = st.S, A = st.A;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < S; base += NT) {
    const uint32_t s = base + threadIdx.x;
    const uint32_t nl = s < S ? P.spl[s].nl : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<NT>(nl, sh, &tot);
    if (s < S) {
      const SplitInfo si = P.spl[s];
      const uint32_t bL = carry + ex;
      const uint32_t bb = fr[si.f].b;
      P.segtab[si.f] = SegTab{static_cast<int32_t>(si.base) - static_cast<int32_t>(bL),
                              static_cast<int32_t>(si.base + nl) - static_cast<int32_t>(bb) +
                                  static_cast<int32_t>(bL),
                              2 * s, 0u};
    }
    carry += tot;
  }
  if (threadIdx.x == 0) st.totL = carry;
  const uint32_t aw = (A + 31u) / 32u;
  carry = 0;
  for (uint32_t base = 0; base < aw; base += NT) {
    const uint32_t w = base + threadIdx.x;
    const uint32_t v = w < aw ? __popc(P.bits[w]) : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<NT>(v, sh, &tot);
    if (w < aw) P.pref[w] = carry + ex;
    carry += tot;
  }
}

// payload pass over flattened (tree, position) + per-position segment offsets
__global__ void w_pay(const WideArgs a) {
  const uint32_t total = a.off[2][a.B];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const uint32_t b = owner(a.off[2], a.B, t), k = t - a.off[2][b];
    const SlotPtrs P = slot_ptrs(a, b);
    const uint32_t f = P.seg[k];
    const SegTab tb = P.segtab[f];
    P.off2[k] = make_int2(tb.offL, tb.offR);
    if (tb.offL == INT_MIN) continue;
    const bool l = get_bit(P.bits, k);
    const int32_t lp = static_cast<int32_t>(bits_before(P.bits, P.pref, k));
    const uint32_t dst =
        static_cast<uint32_t>(l ? tb.offL + lp : tb.offR + static_cast<int32_t>(k) - lp);
    P.pay_n[dst] = P.pay[k];
    P.seg_n[dst] = tb.child + (l ? 0u : 1u);
  }
}

// List pass, single read: one CTA per tree with the tree's goes-left bitmap + prefix
// staged in shared memory and one warp per sorted list.  A warp walks its list in
// position order, 384 positions per step as 12 sub-rows of 32 consecutive positions
// (lane i holds position k0 + 32j + i of sub-row j), so the count of left-going entries
// before each entry is the warp's running carry plus ballot counts -- no count pass --
// and each sub-row's left (right) entries land on consecutive destinations: every
// store instruction writes at most two contiguous runs.  The next step's entries are
// loaded before this step is scattered; the step's segment offsets (off2, mostly L2 hits:
// every list reads the same ones) at its start, and the bitmap word and its prefix come
// interleaved from shared memory in one 8-byte load (kept lean: 64 registers, no spills,
// branch-free with a predicated store).
#ifndef AIWC_LW_SUB
#define AIWC_LW_SUB 12
#endif
constexpr int kLwSub = AIWC_LW_SUB;  // sub-rows of 32 positions per list-pass warp step
constexpr uint32_t kLwStep = 32u * kLwSub;
constexpr int kLwWarps = 28;  // warps per list-pass CTA (<= 73 registers per thread)
template <int NW>
__global__ void __launch_bounds__(NW * 32) w_lwarp(const WideArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  const uint32_t b = blockIdx.x;
  const TreeState& st = a.ts[b];
  if (st.done) return;
  const SlotPtrs P = slot_ptrs(a, b);
  const uint32_t A = st.A, aw = (A + 31u) / 32u;
  const uint32_t nl = a.g.d.nlisted, stride = a.g.L.stride;
  // bitmap word and its prefix interleaved: one 8-byte shared load per entry
  uint2* sbp = reinterpret_cast<uint2*>(sm);
  {  // stage bitmap + prefix (word counts rounded up to 4: both arrays are padded)
    const uint32_t aw4 = (aw + 3u) / 4u;
    const uint4* gb = reinterpret_cast<const uint4*>(P.bits);
    const uint4* gp = reinterpret_cast<const uint4*>(P.pref);
    for (uint32_t w = threadIdx.x; w < aw4; w += blockDim.x) {
      const uint4 x = gb[w], y = gp[w];
      uint4* d = reinterpret_cast<uint4*>(sbp + 4 * w);
      d[0] = make_uint4(x.x, y.x, x.y, y.y);
      d[1] = make_uint4(x.z, y.z, x.w, y.w);
    }
  }
  __syncthreads();
  const unsigned lane = lane_id(), lt = lanemask_lt();
  for (uint32_t li = warp_id(); li < nl; li += blockDim.x >> 5) {
    const uint32_t* src = P.lists + static_cast<size_t>(li) * stride;
    uint32_t* dstl = P.lists_n + static_cast<size_t>(li) * stride;
    uint32_t carry = 0;  // left-going entries of this list before the sub-row
    // only the list entries are prefetched a step ahead (8 registers); the step's segment
    // offsets (mostly L2 hits: every list reads the same off2) are loaded at its start
    uint32_t qn[kLwSub];
#pragma unroll
    for (int j = 0; j < kLwSub; ++j) {
      const uint32_t k = 32u * j + lane;
      qn[j] = k < A ? src[k] : 0u;
    }
    for (uint32_t k0 = 0; k0 < A; k0 += kLwStep) {
      uint32_t q[kLwSub];
      int2 t[kLwSub];
#pragma unroll
      for (int j = 0; j < kLwSub; ++j) {
        q[j] = qn[j];
        const uint32_t k = k0 + 32u * j + lane;
        t[j] = k < A ? P.off2[k] : make_int2(INT_MIN, 0);
      }
#pragma unroll
      for (int j = 0; j < kLwSub; ++j) {
        const uint32_t k = k0 + kLwStep + 32u * j + lane;
        qn[j] = k < A ? src[k] : 0u;
      }
      // branch-free per entry: every lane computes its destination, the store is
      // predicated on `keep` (entries of leaf segments are dropped)
#pragma unroll
      for (int j = 0; j < kLwSub; ++j) {
        const bool keep = t[j].x != INT_MIN;
        const uint32_t qq = keep ? q[j] : 0u;
        const uint2 wp = sbp[qq >> 5];
        const uint32_t w = wp.x, pf = wp.y;
        const uint32_t sh = qq & 31u;
        const bool l = keep && ((w >> sh) & 1u);
        const unsigned bl = __ballot_sync(kFull, l);
        const int32_t pl = static_cast<int32_t>(carry + __popc(bl & lt));
        const int32_t lq = static_cast<int32_t>(pf + __popc(w & ((1u << sh) - 1u)));
        const uint32_t kk = k0 + 32u * j + lane;
        // left: offL + (lefts before); right: offR + (position - lefts before), as selects
        const uint32_t off = static_cast<uint32_t>(l ? t[j].x : t[j].y);
        const uint32_t nq = off + (l ? static_cast<uint32_t>(lq) : qq - static_cast<uint32_t>(lq));
        const uint32_t dst = off + (l ? static_cast<uint32_t>(pl) : kk - static_cast<uint32_t>(pl));
        if (keep) dstl[dst] = nq;
        carry += __popc(bl);
      }
    }
  }
}

// list pass, phase 1: kept-left counts per (tree, chunk)
__global__ void w_lcount(const WideArgs a) {
  const uint32_t total = a.off[3][a.B];
  const uint32_t nl = a.g.d.nlisted, stride = a.g.L.stride;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = gw; it < total; it += nw) {
    const uint32_t b = owner(a.off[3], a.B, it), c = it - a.off[3][b];
    const SlotPtrs P = slot_ptrs(a, b);
    const uint32_t A = a.ts[b].A, A16 = (A + 15u) & ~15u;
    const uint32_t ce = min(nl * A16, (c + 1) * kChunk);
    int2 u;
    const bool uni = chunk_uniform(c * kChunk, ce, A16, A, P.seg, P.off2, u);
    uint32_t cnt = 0;
#pragma unroll 2
    for (uint32_t s = c * kChunk; s < ce; s += 128) {
      ListQuad v;
      load_quad(v, s + lane_id() * 4, A16, A, ce, stride, P.lists, P.off2,
                uni ? &u : nullptr);
      cnt += __popc(side_quad(v, P.bits, P.pref));
    }
    cnt = warp_sum(cnt);
    if (lane_id() == 0) P.chunk[c] = cnt;
  }
}

// list pass, phase 3: scatter with the scanned chunk prefixes
__global__ void w_lscatter(const WideArgs a) {
  const uint32_t total = a.off[3][a.B];
  const uint32_t nl = a.g.d.nlisted, stride = a.g.L.stride;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = gw; it < total; it += nw) {
    const uint32_t b = owner(a.off[3], a.B, it), c = it - a.off[3][b];
    const SlotPtrs P = slot_ptrs(a, b);
    const TreeState& st = a.ts[b];
    const uint32_t A = st.A, A16 = (A + 15u) & ~15u, totL = st.totL;
    const uint32_t ce = min(nl * A16, (c + 1) * kChunk);
    int2 u;
    const bool uni = chunk_uniform(c * kChunk, ce, A16, A, P.seg, P.off2, u);
    uint32_t run = P.chunk[c];
#pragma unroll 2
    for (uint32_t s = c * kChunk; s < ce; s += 128) {
      ListQuad v;
      load_quad(v, s + lane_id() * 4, A16, A, ce, stride, P.lists, P.off2,
                uni ? &u : nullptr);
      const uint32_t lf = side_quad(v, P.bits, P.pref);
      const uint32_t mine = __popc(lf);
      const uint32_t inc = warp_incl_scan(mine);
      int32_t pl = static_cast<int32_t>(run + inc - mine - v.li * totL);
      uint32_t* dstl = P.lists_n + static_cast<size_t>(v.li) * stride;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!((v.keep >> j) & 1u)) continue;
        const bool l = (lf >> j) & 1u;
        const int32_t off = static_cast<int32_t>(v.f[j]);
        const uint32_t dst =
            static_cast<uint32_t>(l ? off + pl : off + static_cast<int32_t>(v.k0 + j) - pl);
        pl += l ? 1 : 0;
        dstl[dst] = v.q[j];
      }
      run += __shfl_sync(kFull, inc, 31);
    }
  }
}

// advance the per-tree level state (after the level's last per-tree read of A)
__global__ void w_advance(const WideArgs a) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  TreeState& s = a.ts[b];
  if (s.done) return;
  s.F = 2 * s.S;
  s.A = s.A_next;
}

// ---- emit + OOB ----------------------------------------------------------------------
__global__ void w_emit(const WideArgs a) {
  __shared__ unsigned long long s_off;
  const uint32_t b = blockIdx.x, tl = a.t0 + b;
  const SlotPtrs P = slot_ptrs(a, b);
  const TreeState& st = a.ts[b];
  const uint32_t count = st.nodes;
  if (threadIdx.x == 0) {
    const unsigned long long off = atomicAdd(a.g.pool_used, static_cast<unsigned long long>(count));
    s_off = off;
    a.g.tree_off[tl] = off;
    a.g.tree_cnt[tl] = count;
    atomicAdd(a.g.split_rows, st.split_rows);
    if (off + count > a.g.pool_cap) atomicExch(a.g.err, 1);
  }
  __syncthreads();
  const unsigned long long off = s_off;
  if (off + count > a.g.pool_cap) return;
  for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
    a.g.pool_feature[off + i] = P.nf[i];
    a.g.pool_thr[off + i] = P.nthr[i];
    a.g.pool_left[off + i] = P.nleft[i];
    a.g.pool_value[off + i] = P.nval[i];
    a.g.pool_rank[off + i] = P.nrank[i];
  }
}

template <typename RankT>
__global__ void w_oob(const WideArgs a) {
  const uint32_t b = blockIdx.y, tl = a.t0 + b;
  const SlotPtrs P = slot_ptrs(a, b);
  const uint32_t n = static_cast<uint32_t>(a.g.d.n);
  const RankT* rank = static_cast<const RankT*>(a.g.d.rank);
  uint32_t* ol = a.g.oobleaf + static_cast<size_t>(tl) * n;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (P.mult[r]) {
      ol[r] = kInBag;
      continue;
    }
    int32_t i = 0;
    int32_t fi = P.nf[0];
    while (fi >= 0) {
      const bool left = rank_of(rank + static_cast<size_t>(fi) * n, r) <= P.nrank[i];
      i = P.nleft[i] + (left ? 0 : 1);
      fi = P.nf[i];
    }
    ol[r] = static_cast<uint32_t>(i);
  }
}

// ---- host driver for one batch of trees [t0, t0+B) (local indices) ----------------
template <typename RankT>
cudaError_t run_wide_t(WideArgs a, cudaStream_t st, int sms, uint32_t* h_active,
                       uint64_t* launches) {
  const uint32_t n = static_cast<uint32_t>(a.g.d.n);
  const dim3 rowsgrid((n + 1023) / 1024, a.B);
  const unsigned wgrid = static_cast<unsigned>(sms) * 8;  // persistent grid-stride kernels
  // per-tree list pass with the bitmap + prefix in shared memory when they fit
  size_t lw_smem = ((a.g.L.stride + 31) / 32 + 3) / 4 * 4 * 8;
  {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (lw_smem + 1024 > static_cast<size_t>(optin) || std::getenv("AIWC_LW_GLOBAL") ||
        cudaFuncSetAttribute(w_lwarp<kLwWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(lw_smem)) != cudaSuccess)
      lw_smem = 0;
    cudaGetLastError();
  }
  const int lw_warps = static_cast<int>(std::min<uint32_t>(kLwWarps, std::max<uint32_t>(1u, a.g.d.nlisted)));
#define WCK(x)                              \
  do {                                      \
    x;                                      \
    ++*launches;                            \
    cudaError_t e_ = cudaGetLastError();    \
    if (e_ != cudaSuccess) return e_;       \
  } while (0)
  WCK((w_zero<<<rowsgrid, 256, 0, st>>>(a)));
  WCK((w_boot<<<rowsgrid, 256, 0, st>>>(a)));
  WCK((w_bits<1024><<<a.B, 1024, 0, st>>>(a)));
  WCK((w_payload<<<rowsgrid, 256, 0, st>>>(a)));
  if (a.g.d.nlisted) {
    WCK((w_l0count<<<wgrid, 256, 0, st>>>(a)));
    WCK((w_chunkscan<1024><<<a.B, 1024, 0, st>>>(a, 0)));
    WCK((w_l0scatter<<<wgrid, 256, 0, st>>>(a)));
  }
  WCK((w_root<<<a.B, 32, 0, st>>>(a)));
  // graph-launched levels (small batches, below): the host reads the split count every
  // sync_every levels (a level is tens of microseconds of GPU work)
  uint32_t sync_every = 4u;
  if (const char* e = std::getenv("AIWC_SYNC_EVERY")) sync_every = std::max(1, std::atoi(e));
  // per-tree bookkeeping kernels (front, decide, segtab) with 128-thread CTAs when a tree
  // has at most a few thousand rows (AIWC_SMALL_CTA=0/1 forces 512 / 128)
  bool small_ct = n < 65536;
  if (const char* e = std::getenv("AIWC_SMALL_CTA")) small_ct = std::atoi(e) != 0;
  // one level's kernels for buffer parity a.cur: part 1 front .. decide, part 2 route ..
  // list pass
  auto level_part1 = [&](WideArgs& a) -> cudaError_t {
    if (small_ct)
      WCK((w_front<128><<<a.B, 128, 0, st>>>(a)));
    else
      WCK((w_front<512><<<a.B, 512, 0, st>>>(a)));
    WCK((w_prefix<1024><<<1, 1024, 0, st>>>(a, 0)));
    // kernels whose size class cannot occur on this table (a node has at most n rows)
    // are not launched: on a 2,220-row table a level is launch-bound
    if (n >= a.big_min) {
      if (a.pair_big == 16)
        WCK((w_chains_warp<RankT, 16><<<wgrid, 256, 0, st>>>(a)));
      else if (a.pair_big == 8)
        WCK((w_chains_warp<RankT, 8><<<wgrid, 256, 0, st>>>(a)));
      else
        WCK((w_chains_warp<RankT, 32><<<wgrid, 256, 0, st>>>(a)));
    }
    if (n >= a.coop_min)
      WCK((w_chains_coop<RankT><<<static_cast<unsigned>(sms) * 8, 128, 0, st>>>(a)));
    switch (grp_width(a.g.mtry)) {
      case 32: WCK((w_chains_grp<RankT, 32, kGrpU><<<wgrid, 256, 0, st>>>(a))); break;
      case 16: WCK((w_chains_grp<RankT, 16, kGrpU><<<wgrid, 256, 0, st>>>(a))); break;
      case 8: WCK((w_chains_grp<RankT, 8, kGrpU><<<wgrid, 256, 0, st>>>(a))); break;
      case 4: WCK((w_chains_grp<RankT, 4, kGrpU><<<wgrid, 256, 0, st>>>(a))); break;
      case 2: WCK((w_chains_grp<RankT, 2, kGrpU><<<wgrid, 256, 0, st>>>(a))); break;
      default: WCK((w_chains_grp<RankT, 1, kGrpU><<<wgrid, 256, 0, st>>>(a))); break;
    }
    WCK((w_chains_lane<RankT><<<wgrid, 256, 0, st>>>(a)));
    {  // w_decide counts this level's splitters
      const cudaError_t em = cudaMemsetAsync(a.active, 0, 4, st);
      if (em != cudaSuccess) return em;
    }
    if (small_ct)
      WCK((w_decide<128, RankT><<<a.B, 128, 0, st>>>(a)));
    else
      WCK((w_decide<512, RankT><<<a.B, 512, 0, st>>>(a)));
    return cudaSuccess;
  };
  auto level_part2 = [&](WideArgs& a) -> cudaError_t {  // route .. list pass
    WCK((w_prefix<1024><<<1, 1024, 0, st>>>(a, 1)));
    if (n >= a.coop_min) WCK((w_route_coop<RankT><<<sms * 8, 128, 0, st>>>(a)));
    WCK((w_route<RankT, true><<<wgrid, 256, 0, st>>>(a)));
    WCK((w_route<RankT, false><<<wgrid, 256, 0, st>>>(a)));
    if (small_ct)
      WCK((w_segtab<128><<<a.B, 128, 0, st>>>(a)));
    else
      WCK((w_segtab<512><<<a.B, 512, 0, st>>>(a)));
    WCK((w_pay<<<wgrid * 4, 256, 0, st>>>(a)));
    if (a.g.d.nlisted) {
      if (lw_smem) {
        WCK((w_lwarp<kLwWarps><<<a.B, lw_warps * 32, lw_smem, st>>>(a)));
      } else {
        WCK((w_lcount<<<wgrid, 256, 0, st>>>(a)));
        WCK((w_chunkscan<512><<<a.B, 512, 0, st>>>(a, 1)));
        WCK((w_lscatter<<<wgrid, 256, 0, st>>>(a)));
      }
    }
    WCK((w_advance<<<(a.B + 255) / 256, 256, 0, st>>>(a)));
    return cudaSuccess;
  };
  // small batches on small tables (a paper-sized 500-tree fit): each level's ~12 kernels
  // replayed as one CUDA graph per buffer parity -- the levels are launch-bound (C1 fit
  // 6.3 -> 5.8 ms); a 34K-tree grid batch measured slower with graphs (277 vs 198 ms).
  // AIWC_LEVEL_GRAPHS=0/1 forces it off/on
  bool graphs = n < 65536 && a.B <= 4096;
  if (const char* e = std::getenv("AIWC_LEVEL_GRAPHS")) graphs = std::atoi(e) != 0;
  cudaGraphExec_t gx[2] = {nullptr, nullptr};
  uint64_t per_level = 0;
  struct GxGuard {
    cudaGraphExec_t* g;
    ~GxGuard() {
      for (int i = 0; i < 2; ++i)
        if (g[i]) cudaGraphExecDestroy(g[i]);
    }
  } gxg{gx};
  if (graphs) {
    for (uint32_t par = 0; par < 2; ++par) {
      a.cur = par;
      const uint64_t l0 = *launches;
      cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return e;
      cudaError_t eb = level_part1(a);
      if (eb == cudaSuccess) eb = level_part2(a);
      cudaGraph_t g = nullptr;
      e = cudaStreamEndCapture(st, &g);
      if (eb != cudaSuccess) return eb;
      if (e != cudaSuccess) return e;
      e = cudaGraphInstantiate(&gx[par], g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return e;
      per_level = *launches - l0;
      *launches = l0;
    }
  }
  auto any_active = [&](bool& more) -> cudaError_t {  // w_decide's count of splitters
    cudaMemcpyAsync(h_active, a.active, 4, cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    more = *h_active != 0;
    return e;
  };
  for (uint32_t level = 0;; ++level) {
    a.cur = level & 1u;
    bool more = true;
    if (graphs) {
      // whole levels as graphs; the host checks every sync_every levels (levels run after
      // every tree is done find no work: each kernel skips done trees)
      cudaError_t e = cudaGraphLaunch(gx[a.cur], st);
      if (e != cudaSuccess) return e;
      *launches += per_level;
      if ((level + 1) % sync_every == 0) {
        e = any_active(more);
        if (e != cudaSuccess) return e;
      }
    } else {
      // large batches: a level without work still costs its grids, so the host checks
      // every level, before the route
      cudaError_t e = level_part1(a);
      if (e != cudaSuccess) return e;
      e = any_active(more);
      if (e != cudaSuccess) return e;
      if (more) {
        e = level_part2(a);
        if (e != cudaSuccess) return e;
      }
    }
    if (!more) break;
  }
  WCK((w_emit<<<a.B, 256, 0, st>>>(a)));
  if (a.g.oobleaf) WCK((w_oob<RankT><<<rowsgrid, 256, 0, st>>>(a)));
#undef WCK
  return cudaSuccess;
}

cudaError_t run_wide(int rank_bytes, const WideArgs& a, cudaStream_t st, int sms,
                     uint32_t* h_active, uint64_t* launches) {
  return rank_bytes == 2 ? run_wide_t<uint16_t>(a, st, sms, h_active, launches)
                         : run_wide_t<uint32_t>(a, st, sms, h_active, launches);
}

}  // namespace aiwc_b200
