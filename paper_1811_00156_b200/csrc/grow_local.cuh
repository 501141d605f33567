// Local (small-node) kernels of the wide grower -- included by grow_wide.cuh.
//
// Nodes below `local_max` rows keep NO sorted lists: the list pass stops writing their
// entries, which is most of its traffic (deep levels hold most of the row-levels of a
// C4 tree).  Instead one CTA per node stages the node's payload (row-ordered) in shared
// memory, gathers each row's record (u16 ranks of the listed columns + a bitmask of the
// two-level ones, DevData::rec) once, and per sampled listed column rebuilds the
// reference's (value, row) bucket order (forest.hpp:154-158, 197-209, 355-371) with a
// stable sort of the node's rows by value rank: ranks order values exactly and the rows
// enter in row order, so the sorted sequence is the reference's bucket.  The split chains
// (forest.hpp:268-297) then run over shared memory with the same sequential FP64 order,
// and the route (forest.hpp:323-352) sorts by column 0 to accumulate the child sums in
// the reference's column-0 order.
#pragma once
// (included inside namespace aiwc_b200 by grow_wide.cuh)

constexpr int kLocMB = 8;                 // sampled columns staged per batch
constexpr uint32_t kLocalSmall = kLocalSmallRows;  // nodes up to this size: counting sort,
                                                   // 64-thread CTAs (their own task list)
constexpr uint32_t kLocalMaxRows = 2048;  // largest local node (shared-memory bound)

// listed column slot (>= 0) or -(1 + bit) of a two-level column, for the record lookups
__device__ __forceinline__ int32_t rec_slot(const DevData& d, uint32_t c) {
  const int32_t li = d.list_of[c];
  return li >= 0 ? li : -(1 + d.bin_of[c]);
}
__device__ __forceinline__ uint32_t rec_rank(const DevData& d, uint32_t row, int32_t slot) {
  const uint8_t* r = d.rec + static_cast<size_t>(row) * d.rec_stride;
  if (slot >= 0) return __ldg(reinterpret_cast<const uint16_t*>(r) + slot);
  const uint32_t bit = static_cast<uint32_t>(-slot - 1);
  return (__ldg(r + d.rec_bits + (bit >> 3)) >> (bit & 7u)) & 1u;
}

// shared-memory layout of the local kernels for nodes of up to SMAX rows; ROUTE: the
// route kernel (wyy staged, column-0 ranks + goes-left flags, one permutation)
template <int NT, int SMAX, bool ROUTE>
struct LocalLayout {
  static constexpr int NW = NT / 32;
  static constexpr int NC = ROUTE ? 2 : kLocMB;                  // u16 key rows
  static constexpr int NP = ROUTE ? 1 : kLocMB;                  // permutations
  static constexpr size_t wy = 0;                                 // double[SMAX]
  static constexpr size_t wyy = wy + 8 * SMAX;                    // double[SMAX] (route)
  static constexpr size_t mu = wyy + (ROUTE ? 8 * SMAX : 0);      // u32[SMAX]
  static constexpr size_t row = mu + 4 * SMAX;                    // u32[SMAX]
  static constexpr size_t stage = row + 4 * SMAX;                 // double[NW][64]
  static constexpr size_t cnt = stage + 8 * 64 * NW;              // u32[NW][256]
  static constexpr size_t rk = cnt + (SMAX > int(kLocalSmall) ? 4 * 256 * NW : 0);  // u16[NC][SMAX]
  static constexpr size_t perm = rk + 2 * NC * SMAX;              // u16[NP][SMAX]
  static constexpr size_t tmp = perm + 2 * NP * SMAX;             // u16[SMAX]
  static constexpr size_t bytes = (tmp + 2 * SMAX + 15) & ~size_t{15};
};

// Stable sort of local indices 0..R-1 by key[i] (u16): out[k] = index of the k-th
// smallest (ties in index order).  R <= 64: rank by counting; else LSD radix over
// 8-bit digits (one pass when every key < 256), per-warp digit counters, warp-match
// ranking -- stable because warps own consecutive index chunks and lanes rank in order.
template <int NT, int SMAX>
__device__ void local_sort(const uint16_t* key, uint32_t R, bool two_pass, uint16_t* out,
                           uint16_t* tmp, uint32_t* cnt) {
  constexpr int NW = NT / 32;
  const unsigned tid = threadIdx.x, lane = lane_id(), w = warp_id();
  if (R <= kLocalSmall || SMAX <= int(kLocalSmall)) {
    for (uint32_t i = tid; i < R; i += NT) {
      const uint32_t ki = key[i];
      uint32_t pos = 0;
      for (uint32_t j = 0; j < R; ++j) {
        const uint32_t kj = key[j];
        pos += (kj < ki || (kj == ki && j < i)) ? 1u : 0u;
      }
      out[pos] = static_cast<uint16_t>(i);
    }
    __syncthreads();
    return;
  }
  const uint32_t ch = ((R + NW - 1) / NW + 31) & ~31u;  // indices per warp
  const uint32_t lo = min(R, w * ch), hi = min(R, lo + ch);
  const unsigned lt = lanemask_lt();
  for (int pass = 0; pass < (two_pass ? 2 : 1); ++pass) {
    const uint16_t* in = pass == 0 ? nullptr : tmp;
    uint16_t* dst = (pass == 0 && two_pass) ? tmp : out;
    const int sh = pass == 0 ? 0 : 8;
    uint32_t* c = cnt + w * 256;
    for (int d = lane; d < 256; d += 32) c[d] = 0u;
    __syncwarp();
    for (uint32_t base = lo; base < hi; base += 32) {
      const uint32_t i = base + lane;
      const bool v = i < hi;
      const uint32_t x = v ? (in ? in[i] : i) : 0u;
      const uint32_t dg = v ? (key[x] >> sh) & 255u : 256u + lane;
      const unsigned grp = __match_any_sync(kFull, dg);
      if (v && lane == static_cast<unsigned>(__ffs(grp) - 1)) c[dg] += __popc(grp);
      __syncwarp();
    }
    __syncthreads();
    // digit-major exclusive offsets over (digit, warp)
    constexpr int DPT = (256 + NT - 1) / NT;
    uint32_t loc = 0;
    for (int k = 0; k < DPT; ++k) {
      const int d = tid * DPT + k;
      if (d < 256)
        for (int ww = 0; ww < NW; ++ww) loc += cnt[ww * 256 + d];
    }
    __shared__ uint32_t s_scan[NW + 2];
    uint32_t tot;
    uint32_t run = block_excl_scan<NT>(loc, s_scan, &tot);
    for (int k = 0; k < DPT; ++k) {
      const int d = tid * DPT + k;
      if (d < 256)
        for (int ww = 0; ww < NW; ++ww) {
          const uint32_t v = cnt[ww * 256 + d];
          cnt[ww * 256 + d] = run;
          run += v;
        }
    }
    __syncthreads();
    for (uint32_t base = lo; base < hi; base += 32) {
      const uint32_t i = base + lane;
      const bool v = i < hi;
      const uint32_t x = v ? (in ? in[i] : i) : 0u;
      const uint32_t dg = v ? (key[x] >> sh) & 255u : 256u + lane;
      const unsigned grp = __match_any_sync(kFull, dg);
      uint32_t pos = 0;
      if (v) pos = c[dg] + __popc(grp & lt);
      __syncwarp();
      if (v && lane == static_cast<unsigned>(__ffs(grp) - 1)) c[dg] += __popc(grp);
      __syncwarp();
      if (v) dst[pos] = static_cast<uint16_t>(x);
    }
    __syncthreads();
  }
}

// One sampled column's chain over the node staged in shared memory, by one warp: a
// listed column walks `perm` (the (value,row) order), a two-level column the row order
// summing its value-0 rows.  Writes the column's ChainRes (local flag in pad: the rows
// either side of the best boundary, for w_decide's threshold).
__device__ __forceinline__ void local_chain(bool listed, const uint16_t* perm, const uint16_t* rk,
                                            const double* wy, const uint32_t* mu,
                                            const uint32_t* row, uint32_t R, double W, double S,
                                            double* st, ChainRes* res) {
  const unsigned lane = lane_id();
  double sl = 0.0;
  if (listed) {
    double bg = -INFINITY;
    uint32_t bp = 0xffffffffu, wl = 0, prev = 0;
    for (uint32_t k0 = 0; k0 < R; k0 += 32) {
      const uint32_t k = k0 + lane, nv = min(32u, R - k0);
      const bool valid = k < R;
      const uint32_t i = valid ? perm[k] : 0u;
      const double v = valid ? wy[i] : 0.0;
      const uint32_t m = valid ? mu[i] : 0u;
      const uint32_t r = valid ? rk[i] : 0u;
      const uint32_t inc = warp_incl_scan(m);
      const uint32_t wlb = wl + inc - m;
      const double mine = tile_prefix(v, nv, sl, st);
      uint32_t pr = __shfl_up_sync(kFull, r, 1);
      if (lane == 0) pr = k0 == 0 ? r : prev;
      if (valid && r != pr) {
        const double gn = gain_at(mine, static_cast<double>(wlb), W, S);
        if (gn > bg) {
          bg = gn;
          bp = k;
        }
      }
      wl += __shfl_sync(kFull, inc, 31);
      prev = __shfl_sync(kFull, r, nv - 1);
    }
    warp_best(bg, bp);
    if (lane == 0)
      *res = bg == -INFINITY ? ChainRes{bg, 0xffffffffu, 0u}
                             : ChainRes{bg, row[perm[bp]], row[perm[bp - 1]] | 0x80000000u};
  } else {
    uint32_t n0 = 0, w0 = 0;
    for (uint32_t k0 = 0; k0 < R; k0 += 32) {
      const uint32_t i = k0 + lane;
      const bool z = i < R && rk[i] == 0u;
      const unsigned bz = __ballot_sync(kFull, z);
      n0 += __popc(bz);
      w0 += z ? mu[i] : 0u;
      tile_masked_sum(i < R ? wy[i] : 0.0, bz, sl, st);
    }
    w0 = warp_sum(w0);
    if (lane == 0)
      *res = (n0 == 0 || n0 == R) ? ChainRes{-INFINITY, 0xffffffffu, 0u}
                                  : ChainRes{gain_at(sl, static_cast<double>(w0), W, S), n0, 0u};
  }
}

// split chains of the local nodes with rmin < rows <= SMAX (forest.hpp:255-297)
template <int NT, int SMAX>
__global__ void __launch_bounds__(NT) w_local(const WideArgs a, uint32_t cls, uint32_t ctr) {
  using Lay = LocalLayout<NT, SMAX, false>;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char lsm[];
  double* s_wy = reinterpret_cast<double*>(lsm + Lay::wy);
  uint32_t* s_mu = reinterpret_cast<uint32_t*>(lsm + Lay::mu);
  uint32_t* s_row = reinterpret_cast<uint32_t*>(lsm + Lay::row);
  double* s_stage = reinterpret_cast<double*>(lsm + Lay::stage);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(lsm + Lay::cnt);
  uint16_t* s_rk = reinterpret_cast<uint16_t*>(lsm + Lay::rk);
  uint16_t* s_perm = reinterpret_cast<uint16_t*>(lsm + Lay::perm);
  uint16_t* s_tmp = reinterpret_cast<uint16_t*>(lsm + Lay::tmp);
  __shared__ uint32_t s_task;
  __shared__ int32_t s_slot[kLocMB];
  __shared__ uint32_t s_two[kLocMB];
  const DevData& d = a.g.d;
  const uint32_t* off = a.off[5 + cls];  // cls 0: <= kLocalSmall rows, 1: larger
  const uint32_t total = off[a.B];
  const unsigned tid = threadIdx.x, w = warp_id();
  for (;;) {
    if (tid == 0) s_task = atomicAdd(a.task_ctr + ctr, 1u);  // one counter per size class
    __syncthreads();
    const uint32_t t = s_task;
    __syncthreads();
    if (t >= total) break;
    const uint32_t b = owner(off, a.B, t), k = t - off[b];
    const SlotPtrs P = slot_ptrs(a, b);
    const TreeState& st = a.ts[b];
    const uint32_t e = P.ecls[st.E0 + st.E1 + st.E2 + (cls ? st.E3 : 0u) + k];
    const NodeWork nw = P.front[P.e2f[e]];
    const uint32_t R = nw.e - nw.b;
    const uint32_t m = tree_m(a, b);
    for (uint32_t i = tid; i < R; i += NT) {
      const Payload pv = P.pay[nw.b + i];
      s_row[i] = pv.row;
      s_mu[i] = pv.mult;
      s_wy[i] = pv.wy;
    }
    for (uint32_t j0 = 0; j0 < m; j0 += kLocMB) {
      const uint32_t nb = min(static_cast<uint32_t>(kLocMB), m - j0);
      if (tid < nb) {
        const uint32_t c = P.samp[static_cast<size_t>(e) * m + j0 + tid];
        s_slot[tid] = rec_slot(d, c);
        s_two[tid] = (d.vals_off[c + 1] - d.vals_off[c]) > 256u ? 1u : 0u;
      }
      __syncthreads();
      for (uint32_t x = tid; x < nb * R; x += NT) {  // record gathers (L1 serves the rest)
        const uint32_t jj = x / R, i = x - jj * R;
        s_rk[jj * SMAX + i] = static_cast<uint16_t>(rec_rank(d, s_row[i], s_slot[jj]));
      }
      __syncthreads();
      for (uint32_t jj = 0; jj < nb; ++jj)
        if (s_slot[jj] >= 0)
          local_sort<NT, SMAX>(s_rk + jj * SMAX, R, s_two[jj] != 0, s_perm + jj * SMAX, s_tmp,
                               s_cnt);
      for (uint32_t jj = w; jj < nb; jj += NW)
        local_chain(s_slot[jj] >= 0, s_perm + jj * SMAX, s_rk + jj * SMAX, s_wy, s_mu, s_row, R,
                    nw.w, nw.s, s_stage + w * 64, P.res + static_cast<size_t>(e) * m + j0 + jj);
      __syncthreads();
    }
  }
}

// route of the local split nodes with rmin < rows <= SMAX: rows in column-0 order
// (a stable sort by the column-0 rank), child (weight, sum, sumsq) as sequential FP64
// sums in that order (forest.hpp:323-352), goes-left bits for the payload pass
template <int NT, int SMAX>
__global__ void __launch_bounds__(NT) w_local_route(const WideArgs a, uint32_t cls, uint32_t ctr) {
  using Lay = LocalLayout<NT, SMAX, true>;
  extern __shared__ __align__(16) unsigned char lsm[];
  double* s_wy = reinterpret_cast<double*>(lsm + Lay::wy);
  double* s_wyy = reinterpret_cast<double*>(lsm + Lay::wyy);
  uint32_t* s_mu = reinterpret_cast<uint32_t*>(lsm + Lay::mu);
  uint32_t* s_row = reinterpret_cast<uint32_t*>(lsm + Lay::row);
  double* s_stage = reinterpret_cast<double*>(lsm + Lay::stage);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(lsm + Lay::cnt);
  uint16_t* s_rk0 = reinterpret_cast<uint16_t*>(lsm + Lay::rk);
  uint16_t* s_left = s_rk0 + SMAX;
  uint16_t* s_perm = reinterpret_cast<uint16_t*>(lsm + Lay::perm);
  uint16_t* s_tmp = reinterpret_cast<uint16_t*>(lsm + Lay::tmp);
  __shared__ uint32_t s_task, s_cnts[3];
  __shared__ double s_sum[4];
  const DevData& d = a.g.d;
  const uint32_t* off = a.off[5 + cls];
  const uint32_t total = off[a.B];
  const unsigned tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const int32_t slot0 = rec_slot(d, 0);
  const bool two0 = (d.vals_off[1] - d.vals_off[0]) > 256u;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(a.task_ctr + ctr, 1u);  // one counter per size class
    __syncthreads();
    const uint32_t t = s_task;
    __syncthreads();
    if (t >= total) break;
    const uint32_t b = owner(off, a.B, t), k = t - off[b];
    const SlotPtrs P = slot_ptrs(a, b);
    const uint32_t s = (cls ? P.lsplit2 : P.lsplit)[k];
    const SplitInfo si = P.spl[s];
    const NodeWork nw = P.front[si.f];
    const uint32_t R = nw.e - nw.b;
    const int32_t slotc = rec_slot(d, si.c);
    if (tid < 3) s_cnts[tid] = 0u;
    uint32_t c_nl = 0, c_wl = 0, c_wr = 0;
    for (uint32_t i = tid; i < R; i += NT) {
      const Payload pv = P.pay[nw.b + i];
      s_row[i] = pv.row;
      s_mu[i] = pv.mult;
      s_wy[i] = pv.wy;
      s_wyy[i] = P.wyy[nw.b + i];
      s_rk0[i] = static_cast<uint16_t>(rec_rank(d, pv.row, slot0));
      const bool l = rec_rank(d, pv.row, slotc) <= si.thr_rank;
      s_left[i] = l ? 1 : 0;
      c_nl += l ? 1u : 0u;
      c_wl += l ? pv.mult : 0u;
      c_wr += l ? 0u : pv.mult;
    }
    c_nl = warp_sum(c_nl);
    c_wl = warp_sum(c_wl);
    c_wr = warp_sum(c_wr);
    __syncthreads();  // s_cnts zeroed
    if (lane == 0) {
      atomicAdd(&s_cnts[0], c_nl);
      atomicAdd(&s_cnts[1], c_wl);
      atomicAdd(&s_cnts[2], c_wr);
    }
    // goes-left bits of positions nw.b .. nw.e-1: a ballot per 32 consecutive positions
    for (uint32_t i0 = w * 32; i0 < R; i0 += NT) {
      const uint32_t i = i0 + lane;
      const unsigned bl = __ballot_sync(kFull, i < R && s_left[i]);
      if (lane == 0 && bl) {
        const uint32_t q = nw.b + i0, sh = q & 31u;
        atomicOr(P.bits + (q >> 5), bl << sh);
        if (sh && (bl >> (32 - sh))) atomicOr(P.bits + (q >> 5) + 1, bl >> (32 - sh));
      }
    }
    local_sort<NT, SMAX>(s_rk0, R, two0, s_perm, s_tmp, s_cnt);
    if (w < 2) {  // warp 0: left (sum, sumsq), warp 1: right, in column-0 order
      double x = 0.0, y = 0.0;
      for (uint32_t k0 = 0; k0 < R; k0 += 32) {
        const uint32_t kk = k0 + lane;
        const uint32_t i = kk < R ? s_perm[kk] : 0u;
        const bool take = kk < R && (s_left[i] != 0) == (w == 0);
        const unsigned msk = __ballot_sync(kFull, take);
        tile_masked_sum2(take ? s_wy[i] : 0.0, take ? s_wyy[i] : 0.0, msk, x, y,
                         s_stage + w * 64);
      }
      if (lane == 0) {
        s_sum[2 * w] = x;
        s_sum[2 * w + 1] = y;
      }
    }
    __syncthreads();
    if (tid == 0) {
      const uint32_t nl = s_cnts[0];
      P.spl[s].nl = nl;
      const uint32_t child = static_cast<uint32_t>(P.nleft[nw.id]);
      P.front_n[2 * s] = NodeWork{si.base, si.base + nl, child, 0u,
                                  static_cast<double>(s_cnts[1]), s_sum[0], s_sum[1]};
      P.front_n[2 * s + 1] = NodeWork{si.base + nl, si.base + si.cnt, child + 1, 0u,
                                      static_cast<double>(s_cnts[2]), s_sum[2], s_sum[3]};
    }
    __syncthreads();
  }
}
