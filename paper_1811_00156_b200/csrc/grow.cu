// Forest grower: one persistent CTA per tree, level-synchronous growth inside the CTA.
//
// Reproduces TreeGrower::grow (forest.hpp:179-376) bit-exactly:
//   * bootstrap: n counter-based splitmix64 draws (forest.hpp:184-195, rng.hpp:45-59);
//   * per tree, the in-bag rows live in a node-grouped, row-ordered "payload" array;
//     every column with >= 3 distinct values keeps a list of payload positions in
//     (value, row) order, partitioned stably by node each level -- the reference's
//     presort/partition invariant (forest.hpp:163-166, 197-209, 355-371) realised
//     as flat CTA-wide scan+scatter passes over compacted arrays.  Columns with <= 2
//     distinct values (the one-hot device columns) need no list: their (value,row)
//     order is "value-0 rows in row order, then value-1 rows", read off the payload;
//   * split scan: one warp (or, for nodes < kLaneMax rows, one lane) per
//     (node, sampled column) chain; the running sum sl is accumulated strictly
//     sequentially in FP64 (warp-shuffle chain, no reassociation) so every gain is
//     bit-identical to forest.hpp:277-296; wl is an exact integer prefix;
//   * first-max argmax over (column slot, position), threshold midpoint rule
//     (forest.hpp:282-283, 287);
//   * children numbered in frontier order (BFS ids, forest.hpp:310-318);
//   * child sums accumulated in column-0 order (forest.hpp:326-344);
//   * mtry draws: exactly mtry per eligible node, counter = n + mtry*(BFS index
//     among eligible nodes) (forest.hpp:255-266).
// Partition destinations come from a shared-memory bitmap of "goes left" flags over
// payload positions plus per-word prefix counts, so no per-element index map is
// gathered from global memory.
// All FP64 arithmetic uses explicit _rn intrinsics (no FMA contraction).
// Row routing compares dense value ranks: x <= thr  <=>  rank(x) <= thr_rank,
// thr_rank = largest distinct-value rank with value <= thr (exact for every
// training row).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>

#include "device_common.cuh"
#include "forest_kernels.cuh"
#include "grow.cuh"

namespace aiwc_b200 {

namespace {

constexpr uint32_t kLaneMax = 48;  // nodes below this size use one lane per chain
constexpr uint32_t kMaxP = 1024;
constexpr int kPhases = 14;
constexpr int kE = 16;  // elements per thread in the flat partition passes
}  // namespace
constexpr uint32_t kListChunk = 4096;  // list-pass chunk (flat elements) per warp task
namespace {
constexpr uint32_t kChunk = kListChunk;

__device__ __forceinline__ uint32_t get_bit(const uint32_t* bits, uint32_t i) {
  return (bits[i >> 5] >> (i & 31u)) & 1u;
}

// set bits strictly before position q (per-word prefix counts)
__device__ __forceinline__ uint32_t bits_before(const uint32_t* bits, const uint32_t* pref,
                                                uint32_t q) {
  return pref[q >> 5] + __popc(bits[q >> 5] & ((1u << (q & 31u)) - 1u));
}

// in-bag rank of row r (per-64-row prefix counts)
__device__ __forceinline__ uint32_t inbag_pos(const uint32_t* bits, const uint32_t* pref64,
                                              uint32_t r) {
  const uint32_t w = r >> 5;
  return pref64[r >> 6] + ((w & 1u) ? __popc(bits[w - 1]) : 0u) +
         __popc(bits[w] & ((1u << (r & 31u)) - 1u));
}

template <typename RankT>
__device__ __forceinline__ uint32_t rank_of(const RankT* rank_c, uint32_t row) {
  return static_cast<uint32_t>(__ldg(rank_c + row));
}

__device__ __forceinline__ double gain_at(double sl, double wl, double W, double S) {
  // sl*sl/wl + (sum-sl)*(sum-sl)/wr   (forest.hpp:284-286)
  const double wr = __dsub_rn(W, wl);
  const double d = __dsub_rn(S, sl);
  return __dadd_rn(__ddiv_rn(__dmul_rn(sl, sl), wl), __ddiv_rn(__dmul_rn(d, d), wr));
}

// ---- sequential FP64 accumulation over one 32-element tile -----------------------
// The values go through this warp's shared-memory stage and every lane runs the same
// fully unrolled add chain, so the chain is bound by DADD latency alone (the loads are
// independent of it).  The order of the adds is the lane order -- exactly the order
// the reference visits these rows -- so results are bit-identical.

// running value before each lane's element (lanes j < nv), `run` advanced past them
__device__ __forceinline__ double tile_prefix(double v, uint32_t nv, double& run, double* st) {
  const unsigned lane = lane_id();
  st[lane] = v;
  __syncwarp();
  double r = run, mine = 0.0;
  if (nv == 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double x = st[j];
      mine = (lane == static_cast<unsigned>(j)) ? r : mine;
      r = __dadd_rn(r, x);
    }
  } else {
#pragma unroll 8
    for (uint32_t j = 0; j < nv; ++j) {
      const double x = st[j];
      mine = (lane == j) ? r : mine;
      r = __dadd_rn(r, x);
    }
  }
  __syncwarp();
  run = r;
  return mine;
}

// add the masked lanes' (a, b) values, in lane order, onto (ra, rb)
__device__ __forceinline__ void tile_masked_sum2(double a, double b, unsigned mask, double& ra,
                                                 double& rb, double* st) {
  const unsigned lane = lane_id();
  if ((mask >> lane) & 1u) {
    const unsigned k = __popc(mask & lanemask_lt());
    st[k] = a;
    st[32 + k] = b;
  }
  __syncwarp();
  const uint32_t cnt = __popc(mask);
  double x = ra, y = rb;
  if (cnt == 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      x = __dadd_rn(x, st[j]);
      y = __dadd_rn(y, st[32 + j]);
    }
  } else {
#pragma unroll 8
    for (uint32_t j = 0; j < cnt; ++j) {
      x = __dadd_rn(x, st[j]);
      y = __dadd_rn(y, st[32 + j]);
    }
  }
  __syncwarp();
  ra = x;
  rb = y;
}

__device__ __forceinline__ void tile_masked_sum(double a, unsigned mask, double& ra, double* st) {
  const unsigned lane = lane_id();
  if ((mask >> lane) & 1u) st[__popc(mask & lanemask_lt())] = a;
  __syncwarp();
  const uint32_t cnt = __popc(mask);
  double x = ra;
  if (cnt == 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x = __dadd_rn(x, st[j]);
  } else {
#pragma unroll 8
    for (uint32_t j = 0; j < cnt; ++j) x = __dadd_rn(x, st[j]);
  }
  __syncwarp();
  ra = x;
}

// ---- list-pass element quads -------------------------------------------------------
// Four consecutive positions of one list (flat index g0 over (list, position)).
struct ListQuad {
  uint32_t q[4];  // list entries (payload positions); after side_quad: next-level entries
  uint32_t f[4];  // after side_quad: the destination offset (offL or offR)
  int2 t[4];      // (offL, offR) of each position's segment (offL == INT_MIN: leaf)
  uint32_t li, k0, keep;
};

// off2: per position of this level, its segment's (offL, offR) -- expanded once per
// level so the list pass has no dependent segment-table lookup
__device__ __forceinline__ void load_quad(ListQuad& v, uint32_t g0, uint32_t A16, uint32_t A,
                                          uint32_t end, uint32_t stride, const uint32_t* lists,
                                          const int2* off2, const int2* uniform = nullptr) {
  v.keep = 0;
  v.li = g0 / A16;
  v.k0 = g0 - v.li * A16;
  if (g0 < end && v.k0 < A) {
    const uint4 x = *reinterpret_cast<const uint4*>(lists + static_cast<size_t>(v.li) * stride + v.k0);
    v.q[0] = x.x; v.q[1] = x.y; v.q[2] = x.z; v.q[3] = x.w;
    if (uniform) {  // the whole chunk lies in one segment: no per-position offsets
      v.t[0] = v.t[1] = v.t[2] = v.t[3] = *uniform;
    } else {
      const int4 y0 = *reinterpret_cast<const int4*>(off2 + v.k0);
      const int4 y1 = *reinterpret_cast<const int4*>(off2 + v.k0 + 2);
      v.t[0] = make_int2(y0.x, y0.y); v.t[1] = make_int2(y0.z, y0.w);
      v.t[2] = make_int2(y1.x, y1.y); v.t[3] = make_int2(y1.z, y1.w);
    }
    const uint32_t left = A - v.k0;
    v.keep = left >= 4 ? 0xfu : ((1u << left) - 1u);
  }
}

// side bits of the quad's kept entries (entries of leaf segments are dropped); also
// rewrites q to the entries' next-level payload positions and f to their offsets
__device__ __forceinline__ uint32_t side_quad(ListQuad& v, const uint32_t* bits,
                                              const uint32_t* pref) {
  uint32_t lf = 0, keep = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (!((v.keep >> j) & 1u)) continue;
    const int2 t = v.t[j];
    if (t.x == INT_MIN) continue;
    keep |= 1u << j;
    const uint32_t qq = v.q[j];
    const uint32_t w = bits[qq >> 5];
    const uint32_t b = (w >> (qq & 31u)) & 1u;
    const int32_t lq = static_cast<int32_t>(pref[qq >> 5] + __popc(w & ((1u << (qq & 31u)) - 1u)));
    lf |= b << j;
    v.q[j] = static_cast<uint32_t>(b ? t.x + lq : t.y + static_cast<int32_t>(qq) - lq);
    v.f[j] = static_cast<uint32_t>(b ? t.x : t.y);
  }
  v.keep = keep;
  return lf;
}

__device__ __forceinline__ void warp_best(double& bg, uint32_t& bp) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double og = __shfl_xor_sync(kFull, bg, o);
    const uint32_t op = __shfl_xor_sync(kFull, bp, o);
    if (og > bg || (og == bg && op < bp)) {
      bg = og;
      bp = op;
    }
  }
}

// ---- split chain over a sorted list, warp-cooperative (large nodes) ---------------
template <typename RankT, int G>
__device__ void chain_warp(const uint32_t* list, uint32_t b, uint32_t e,
                           const Payload* pay, const RankT* __restrict__ rk_c,
                           double W, double S, double& best_gain, uint32_t& best_pos,
                           double* st) {
  const unsigned lane = lane_id();
  double sl = 0.0;
  uint32_t wl = 0, prev_rank = 0;
  bool first = true;
  double bg = -INFINITY;
  uint32_t bp = 0xffffffffu;
  for (uint32_t k0 = b; k0 < e; k0 += 32 * G) {
    uint32_t q[G], rk[G], mu[G];
    double wy[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      q[g] = k < e ? list[k] : 0u;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      if (k < e) {
        const Payload P = pay[q[g]];
        q[g] = P.row;
        mu[g] = P.mult;
        wy[g] = P.wy;
      } else {
        mu[g] = 0;
        wy[g] = 0.0;
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      rk[g] = k < e ? rank_of(rk_c, q[g]) : 0u;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t t0 = k0 + g * 32;
      if (t0 >= e) break;
      const uint32_t nv = min(32u, e - t0);
      const bool valid = lane < nv;
      const uint32_t inc = warp_incl_scan(mu[g]);
      const uint32_t wl_before = wl + inc - mu[g];
      const double mine = tile_prefix(wy[g], nv, sl, st);
      uint32_t pr = __shfl_up_sync(kFull, rk[g], 1);
      if (lane == 0) pr = first ? rk[g] : prev_rank;
      if (valid && rk[g] != pr) {
        const double gn = gain_at(mine, static_cast<double>(wl_before), W, S);
        if (gn > bg) {
          bg = gn;
          bp = t0 + lane;
        }
      }
      wl += __shfl_sync(kFull, inc, 31);
      prev_rank = __shfl_sync(kFull, rk[g], nv - 1);
      first = false;
    }
  }
  warp_best(bg, bp);
  best_gain = bg;
  best_pos = bp;
}

// Pipelined warp chains for the wide grower: tiles of 32*G positions; while tile i is
// scanned, the payload gathers of tile i+1 and the list loads of tile i+2 are in
// flight.  Same arithmetic (and order) as chain_warp / chain_bin_warp.
template <typename RankT, int G>
__device__ void chain_warp_p(bool listed, const uint32_t* list, uint32_t b, uint32_t e,
                             const Payload* pay, const RankT* __restrict__ rk_c, double W,
                             double S, double& best_gain, uint32_t& best_pos, double* st) {
  const unsigned lane = lane_id();
  double sl = 0.0, bg = -INFINITY;
  uint32_t wl = 0, prev_rank = 0, bp = 0xffffffffu, n0 = 0, wl_lane = 0;
  bool first = true;
  uint32_t qn[G], rowc[G], muc[G], rown[G], mun[G];
  double wyc[G], wyn[G];
  auto load_q = [&](uint32_t k0, uint32_t (&q)[G]) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      q[g] = k < e ? (listed ? list[k] : k) : 0u;
    }
  };
  auto load_p = [&](uint32_t k0, const uint32_t (&q)[G], uint32_t (&row)[G], uint32_t (&mu)[G],
                    double (&wy)[G]) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      if (k < e) {
        const Payload P = pay[q[g]];
        row[g] = P.row;
        mu[g] = P.mult;
        wy[g] = P.wy;
      } else {
        row[g] = 0u;
        mu[g] = 0u;
        wy[g] = 0.0;
      }
    }
  };
  // 3-stage pipeline: tile i is scanned while the rank gathers of tile i+1, the payload
  // gathers of tile i+2 and the list loads of tile i+3 are in flight
  auto load_r = [&](uint32_t k0, const uint32_t (&row)[G], uint32_t (&rk)[G]) {
#pragma unroll
    for (int g = 0; g < G; ++g)
      rk[g] = k0 + g * 32 + lane < e ? rank_of(rk_c, row[g]) : 0u;
  };
  uint32_t rk[G], rkn[G];
  load_q(b, qn);
  load_p(b, qn, rowc, muc, wyc);
  load_q(b + 32 * G, qn);
  load_p(b + 32 * G, qn, rown, mun, wyn);
  load_q(b + 64 * G, qn);
  load_r(b, rowc, rk);
  for (uint32_t k0 = b; k0 < e; k0 += 32 * G) {
    load_r(k0 + 32 * G, rown, rkn);
    uint32_t rownn[G], munn[G];
    double wynn[G];
    load_p(k0 + 64 * G, qn, rownn, munn, wynn);
    load_q(k0 + 96 * G, qn);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t t0 = k0 + g * 32;
      if (t0 >= e) break;
      const uint32_t nv = min(32u, e - t0);
      const bool valid = lane < nv;
      if (listed) {
        const uint32_t inc = warp_incl_scan(muc[g]);
        const uint32_t wl_before = wl + inc - muc[g];
        const double mine = tile_prefix(wyc[g], nv, sl, st);
        uint32_t pr = __shfl_up_sync(kFull, rk[g], 1);
        if (lane == 0) pr = first ? rk[g] : prev_rank;
        if (valid && rk[g] != pr) {
          const double gn = gain_at(mine, static_cast<double>(wl_before), W, S);
          if (gn > bg) {
            bg = gn;
            bp = t0 + lane;
          }
        }
        wl += __shfl_sync(kFull, inc, 31);
        prev_rank = __shfl_sync(kFull, rk[g], nv - 1);
        first = false;
      } else {  // two-level column: value-0 rows in row order, +0.0 for the others
        const bool z = valid && rk[g] == 0u;
        n0 += __popc(__ballot_sync(kFull, z));
        wl_lane += z ? muc[g] : 0u;  // integer: reduced once at the end
        st[lane] = z ? wyc[g] : 0.0;
        __syncwarp();
        double r = sl;
#pragma unroll
        for (int j = 0; j < 32; ++j) r = __dadd_rn(r, st[j]);
        sl = r;
        __syncwarp();
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      muc[g] = mun[g];
      wyc[g] = wyn[g];
      rk[g] = rkn[g];
      rown[g] = rownn[g];
      mun[g] = munn[g];
      wyn[g] = wynn[g];
    }
  }
  if (!listed) wl = warp_sum(wl_lane);
  if (listed) {
    warp_best(bg, bp);
    best_gain = bg;
    best_pos = bp;
  } else if (n0 == 0 || n0 == e - b) {
    best_gain = -INFINITY;
    best_pos = 0xffffffffu;
  } else {
    best_gain = gain_at(sl, static_cast<double>(wl), W, S);
    best_pos = b + n0;
  }
}

// ---- split chain over a sorted list, one lane (small nodes) -----------------------
template <typename RankT>
__device__ void chain_lane(const uint32_t* list, uint32_t b, uint32_t e,
                           const Payload* pay, const RankT* __restrict__ rk_c,
                           double W, double S, double& best_gain, uint32_t& best_pos) {
  double sl = 0.0, bg = -INFINITY;
  uint32_t wl = 0, prev = 0, bp = 0xffffffffu;
  for (uint32_t k = b; k < e; k += 4) {
    uint32_t q[4], rk[4], mu[4];
    double wy[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) q[g] = k + g < e ? list[k + g] : 0u;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (k + g < e) {
        const Payload P = pay[q[g]];
        q[g] = P.row;
        mu[g] = P.mult;
        wy[g] = P.wy;
      } else {
        mu[g] = 0;
        wy[g] = 0.0;
      }
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) rk[g] = k + g < e ? rank_of(rk_c, q[g]) : 0u;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint32_t kk = k + g;
      if (kk >= e) break;
      if (kk > b && rk[g] != prev) {
        const double gn = gain_at(sl, static_cast<double>(wl), W, S);
        if (gn > bg) {
          bg = gn;
          bp = kk;
        }
      }
      wl += mu[g];
      sl = __dadd_rn(sl, wy[g]);
      prev = rk[g];
    }
  }
  best_gain = bg;
  best_pos = bp;
}

// ---- split chain of a two-level column: the only boundary sits after the value-0
// rows, and sl there is their sequential sum in row (= payload) order --------------
template <typename RankT, int G>
__device__ void chain_bin_warp(const Payload* pay, uint32_t b, uint32_t e,
                               const RankT* __restrict__ rk_c, double W, double S,
                               double& best_gain, uint32_t& best_pos, double* st) {
  const unsigned lane = lane_id();
  double s0 = 0.0;
  uint32_t w0 = 0, n0 = 0;
  for (uint32_t k0 = b; k0 < e; k0 += 32 * G) {
    uint32_t row[G], mu[G];
    double wy[G];
    bool z[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      if (k < e) {
        const Payload P = pay[k];
        row[g] = P.row;
        mu[g] = P.mult;
        wy[g] = P.wy;
      } else {
        row[g] = 0;
        mu[g] = 0;
        wy[g] = 0.0;
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) z[g] = (k0 + g * 32 + lane < e) && rank_of(rk_c, row[g]) == 0u;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t t0 = k0 + g * 32;
      if (t0 >= e) break;
      const unsigned bz = __ballot_sync(kFull, z[g]);
      n0 += __popc(bz);
      w0 += warp_sum(z[g] ? mu[g] : 0u);
      tile_masked_sum(wy[g], bz, s0, st);
    }
  }
  const uint32_t R = e - b;
  if (n0 == 0 || n0 == R) {
    best_gain = -INFINITY;
    best_pos = 0xffffffffu;
  } else {
    best_gain = gain_at(s0, static_cast<double>(w0), W, S);
    best_pos = b + n0;
  }
}

template <typename RankT>
__device__ void chain_bin_lane(const Payload* pay, uint32_t b, uint32_t e,
                               const RankT* __restrict__ rk_c, double W, double S,
                               double& best_gain, uint32_t& best_pos) {
  double s0 = 0.0;
  uint32_t w0 = 0, n0 = 0;
  for (uint32_t k = b; k < e; k += 4) {
    Payload P[4];
    bool z[4];
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if (k + g < e) P[g] = pay[k + g];
#pragma unroll
    for (int g = 0; g < 4; ++g) z[g] = k + g < e && rank_of(rk_c, P[g].row) == 0u;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (!z[g]) continue;
      ++n0;
      w0 += P[g].mult;
      s0 = __dadd_rn(s0, P[g].wy);
    }
  }
  const uint32_t R = e - b;
  if (n0 == 0 || n0 == R) {
    best_gain = -INFINITY;
    best_pos = 0xffffffffu;
  } else {
    best_gain = gain_at(s0, static_cast<double>(w0), W, S);
    best_pos = b + n0;
  }
}

// ---- split chains of one node, G lanes per (node, column) -------------------------
// A warp holds 32/G lane groups, each running one sampled column of the SAME node (so
// every group walks the same range [b, e) and the warp stays converged).  A round
// covers G*U consecutive positions; lane gl of a group owns positions
// k0 + gl*U + u (u < U), so the visiting order is (gl, u) lexicographic.  The
// sequential FP64 chain of a round runs in every lane of the group over a shared-memory
// stage (each DADD instruction serves 32/G chains instead of one), the integer weight
// prefix is a group scan, and gains are evaluated per lane at value boundaries.
// `listed`: the column's sorted list gives the order (forest.hpp:268-297); otherwise the
// column is two-level and its chain is the row-order sum of the value-0 rows (a masked
// add of +0.0 is exact: the running sum starts at +0.0 and can never become -0.0).
template <typename RankT, int G, int U>
__device__ __forceinline__ void chain_grp(bool active, bool listed, const uint32_t* list,
                                          uint32_t b, uint32_t e, const Payload* pay,
                                          const RankT* __restrict__ rk_c, double W, double S,
                                          double& best_gain, uint32_t& best_pos, double* st) {
  static_assert(U % 4 == 0, "U must be a multiple of 4 (uint4 list loads)");
  constexpr uint32_t R = G * U;  // positions per round
  const unsigned gl = lane_id() & (G - 1);
  double sl = 0.0, bg = -INFINITY;
  uint32_t wl = 0, prev_rank = 0, bp = 0xffffffffu, n0 = 0;
  bool pg[G];
#pragma unroll
  for (int g = 0; g < G; ++g) pg[g] = gl == static_cast<unsigned>(g);
  // software pipeline over rounds: while round i is summed, the payload gathers of round
  // i+1 and the list loads of round i+2 are in flight
  auto load_q = [&](uint32_t kb, uint32_t (&q)[U]) {
    if (active && listed) {
#pragma unroll
      for (int v = 0; v < U; v += 4) {
        if (kb + v < e) {
          const uint4 x = *reinterpret_cast<const uint4*>(list + kb + v);
          q[v] = x.x; q[v + 1] = x.y; q[v + 2] = x.z; q[v + 3] = x.w;
        } else {
          q[v] = q[v + 1] = q[v + 2] = q[v + 3] = 0u;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) q[u] = kb + u;
    }
  };
  auto load_p = [&](uint32_t kb, const uint32_t (&q)[U], uint32_t (&row)[U], uint32_t (&mu)[U],
                    double (&wy)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = kb + u;
      if (active && k >= b && k < e) {
        const Payload P = pay[q[u]];
        row[u] = P.row;
        mu[u] = P.mult;
        wy[u] = P.wy;
      } else {
        row[u] = 0u;
        mu[u] = 0u;
        wy[u] = 0.0;
      }
    }
  };
  // 3-stage pipeline: round i is summed while the rank gathers of round i+1, the
  // payload gathers of round i+2 and the list loads of round i+3 are in flight
  auto load_r = [&](uint32_t kb, const uint32_t (&row)[U], uint32_t (&rk)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = kb + u;
      rk[u] = (active && k >= b && k < e) ? rank_of(rk_c, row[u]) : 0u;
    }
  };
  uint32_t k0 = b & ~3u;
  uint32_t qn[U], rowc[U], muc[U], rown[U], mun[U], rk[U], rkn[U];
  double wyc[U], wyn[U];
  load_q(k0 + gl * U, qn);
  load_p(k0 + gl * U, qn, rowc, muc, wyc);
  load_q(k0 + R + gl * U, qn);
  load_p(k0 + R + gl * U, qn, rown, mun, wyn);
  load_q(k0 + 2 * R + gl * U, qn);
  load_r(k0 + gl * U, rowc, rk);
  for (; k0 < e; k0 += R) {
    const uint32_t kb = k0 + gl * U;
    uint32_t mu[U];
    double a[U];
    load_r(kb + R, rown, rkn);
    uint32_t rownn[U], munn[U];
    double wynn[U];
    load_p(kb + 2 * R, qn, rownn, munn, wynn);
    load_q(kb + 3 * R, qn);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      mu[u] = muc[u];
      a[u] = wyc[u];
      if (!listed) {  // two-level column: only value-0 rows enter the chain
        const uint32_t k = kb + u;
        const bool z = active && k >= b && k < e && rk[u] == 0u;
        n0 += z ? 1u : 0u;
        if (!z) {
          mu[u] = 0u;
          a[u] = 0.0;
        }
      }
    }
    // integer weight prefix (exact): lane-local, then across the group
    uint32_t loc = 0, wb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      wb[u] = loc;
      loc += mu[u];
    }
    uint32_t inc = loc;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, inc, o, G);
      if (gl >= static_cast<unsigned>(o)) inc += t;
    }
    const uint32_t wbase = wl + inc - loc;
    wl += __shfl_sync(kFull, inc, G - 1, G);
    // sequential FP64 chain of the round
#pragma unroll
    for (int u = 0; u < U; ++u) st[gl * U + u] = a[u];
    __syncwarp();
    double mine[U];
    double r = sl;
#pragma unroll
    for (int j = 0; j < static_cast<int>(R); ++j) {
      if (pg[j / U]) mine[j % U] = r;
      r = __dadd_rn(r, st[j]);
    }
    sl = r;
    __syncwarp();
    // (shuffles stay outside the `listed` branch: groups of one warp may differ)
    uint32_t pr = __shfl_up_sync(kFull, rk[U - 1], 1, G);
    if (gl == 0) pr = prev_rank;
    prev_rank = __shfl_sync(kFull, rk[U - 1], G - 1, G);
    if (listed) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = kb + u;
        const uint32_t pru = u == 0 ? pr : rk[u - 1];
        if (active && k > b && k < e && rk[u] != pru) {
          const double gn = gain_at(mine[u], static_cast<double>(wbase + wb[u]), W, S);
          if (gn > bg) {
            bg = gn;
            bp = k;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      muc[u] = mun[u];
      wyc[u] = wyn[u];
      rk[u] = rkn[u];
      rown[u] = rownn[u];
      mun[u] = munn[u];
      wyn[u] = wynn[u];
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    const double og = __shfl_xor_sync(kFull, bg, o, G);
    const uint32_t op = __shfl_xor_sync(kFull, bp, o, G);
    if (og > bg || (og == bg && op < bp)) {
      bg = og;
      bp = op;
    }
    n0 += __shfl_xor_sync(kFull, n0, o, G);
  }
  if (listed) {
    best_gain = bg;
    best_pos = bp;
  } else {
    if (n0 == 0 || n0 == e - b) {
      best_gain = -INFINITY;
      best_pos = 0xffffffffu;
    } else {
      best_gain = gain_at(sl, static_cast<double>(wl), W, S);
      best_pos = b + n0;
    }
  }
}

struct RouteOut {
  uint32_t nl;
  uint32_t wl, wr;
  double sl, ql, sr, qr;
};

// ---- route + child sums in column-0 order (list of column 0), warp-cooperative -----
template <typename RankT, int G>
__device__ void route_warp(const uint32_t* list0, uint32_t b, uint32_t e,
                           const Payload* pay, const double* __restrict__ y,
                           const RankT* __restrict__ rk_f, uint32_t thr_rank, uint32_t* bits,
                           RouteOut& o, double* st) {
  const unsigned lane = lane_id();
  for (uint32_t k0 = b; k0 < e; k0 += 32 * G) {
    uint32_t q[G], row[G], mu[G];
    double wy[G], yy[G];
    bool lft[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      q[g] = k < e ? list0[k] : 0u;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      if (k < e) {
        const Payload P = pay[q[g]];
        row[g] = P.row;
        mu[g] = P.mult;
        wy[g] = P.wy;
        yy[g] = __dmul_rn(P.wy, __ldg(y + P.row));  // = the row's wy * y (forest.hpp:344)
      } else {
        row[g] = 0;
        mu[g] = 0;
        wy[g] = 0.0;
        yy[g] = 0.0;
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
      lft[g] = (k0 + g * 32 + lane < e) && rank_of(rk_f, row[g]) <= thr_rank;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t t0 = k0 + g * 32;
      if (t0 >= e) break;
      const uint32_t nv = min(32u, e - t0);
      const bool valid = lane < nv;
      const bool left = lft[g];
      if (left) atomicOr(bits + (q[g] >> 5), 1u << (q[g] & 31u));
      const unsigned bl = __ballot_sync(kFull, left);
      const unsigned bv = __ballot_sync(kFull, valid);
      o.nl += __popc(bl);
      o.wl += warp_sum(left ? mu[g] : 0u);
      o.wr += warp_sum((valid && !left) ? mu[g] : 0u);
      tile_masked_sum2(wy[g], yy[g], bl, o.sl, o.ql, st);
      tile_masked_sum2(wy[g], yy[g], bv & ~bl, o.sr, o.qr, st);
    }
  }
}

// Pipelined variant for the wide grower: tiles of 32*G positions; while tile i is
// summed, the payload gathers of tile i+1 and the list loads of tile i+2 are in flight.
// The four sequential sums (left/right x sum/sumsq) run in four 8-lane groups over a
// staged tile in which elements of the other side are +0.0 (an exact no-op, see
// chain_grp), so every tile costs 32 dependent DADDs per group and no masked loops.
template <typename RankT, int G>
__device__ void route_warp_p(const uint32_t* list0, uint32_t b, uint32_t e,
                             const Payload* pay, const double* __restrict__ y,
                             const RankT* __restrict__ rk_f, uint32_t thr_rank, uint32_t* bits,
                             RouteOut& o, double* st /* 4*32 doubles */) {
  const unsigned lane = lane_id(), grp = lane >> 3;
  double acc = 0.0;  // this lane's group chain: 0 sl, 1 ql, 2 sr, 3 qr
  uint32_t wl_lane = 0, wr_lane = 0;
  uint32_t qn[G], qc[G], rowc[G], muc[G], rown[G], mun[G];
  double wyc[G], yyc[G], wyn[G], yyn[G];
  auto load_q = [&](uint32_t k0, uint32_t (&q)[G]) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      q[g] = k < e ? list0[k] : 0u;
    }
  };
  auto load_p = [&](uint32_t k0, const uint32_t (&q)[G], uint32_t (&row)[G], uint32_t (&mu)[G],
                    double (&wy)[G], double (&yy)[G]) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      if (k < e) {
        const Payload P = pay[q[g]];
        row[g] = P.row;
        mu[g] = P.mult;
        wy[g] = P.wy;
        yy[g] = __dmul_rn(P.wy, __ldg(y + P.row));  // = the row's wy * y (forest.hpp:344)
      } else {
        row[g] = 0u;
        mu[g] = 0u;
        wy[g] = 0.0;
        yy[g] = 0.0;
      }
    }
  };
  // 3-stage pipeline: tile i is summed while the rank gathers of tile i+1, the payload
  // gathers of tile i+2 and the list loads of tile i+3 are in flight
  // (raw ranks are kept and compared at use, so the gathers never stall the issue)
  auto load_s = [&](uint32_t k0, const uint32_t (&row)[G], uint32_t (&rk)[G]) {
#pragma unroll
    for (int g = 0; g < G; ++g)
      rk[g] = (k0 + g * 32 + lane < e) ? rank_of(rk_f, row[g]) : 0xffffffffu;
  };
  uint32_t qnn[G];
  uint32_t lft[G], lftn[G];
  load_q(b, qc);
  load_p(b, qc, rowc, muc, wyc, yyc);
  load_q(b + 32 * G, qn);
  load_p(b + 32 * G, qn, rown, mun, wyn, yyn);
  load_q(b + 64 * G, qnn);
  load_s(b, rowc, lft);
  for (uint32_t k0 = b; k0 < e; k0 += 32 * G) {
    load_s(k0 + 32 * G, rown, lftn);
    uint32_t rownn[G], munn[G], qnnn[G];
    double wynn[G], yynn[G];
    load_p(k0 + 64 * G, qnn, rownn, munn, wynn, yynn);
    load_q(k0 + 96 * G, qnnn);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t t0 = k0 + g * 32;
      const bool valid = t0 + lane < e;
      const bool left = lft[g] <= thr_rank;
      if (left) atomicOr(bits + (qc[g] >> 5), 1u << (qc[g] & 31u));
      o.nl += __popc(__ballot_sync(kFull, left));
      wl_lane += left ? muc[g] : 0u;  // integer weights: reduced once at the end
      wr_lane += (valid && !left) ? muc[g] : 0u;
      st[lane] = left ? wyc[g] : 0.0;
      st[32 + lane] = left ? yyc[g] : 0.0;
      st[64 + lane] = (valid && !left) ? wyc[g] : 0.0;
      st[96 + lane] = (valid && !left) ? yyc[g] : 0.0;
      __syncwarp();
      const double* sg = st + grp * 32;
      double r = acc;
#pragma unroll
      for (int j = 0; j < 32; ++j) r = __dadd_rn(r, sg[j]);
      acc = r;
      __syncwarp();
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      qc[g] = qn[g];
      qn[g] = qnn[g];
      qnn[g] = qnnn[g];
      muc[g] = mun[g];
      wyc[g] = wyn[g];
      yyc[g] = yyn[g];
      lft[g] = lftn[g];
      rown[g] = rownn[g];
      mun[g] = munn[g];
      wyn[g] = wynn[g];
      yyn[g] = yynn[g];
    }
  }
  o.wl += warp_sum(wl_lane);
  o.wr += warp_sum(wr_lane);
  o.sl = __shfl_sync(kFull, acc, 0);
  o.ql = __shfl_sync(kFull, acc, 8);
  o.sr = __shfl_sync(kFull, acc, 16);
  o.qr = __shfl_sync(kFull, acc, 24);
}

template <typename RankT>
__device__ void route_lane(const uint32_t* list0, uint32_t b, uint32_t e,
                           const Payload* pay, const double* __restrict__ y,
                           const RankT* __restrict__ rk_f, uint32_t thr_rank, uint32_t* bits,
                           RouteOut& o) {
  for (uint32_t k = b; k < e; k += 4) {
    uint32_t q[4], row[4], mu[4];
    double wy[4], yy[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) q[g] = k + g < e ? list0[k + g] : 0u;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (k + g < e) {
        const Payload P = pay[q[g]];
        row[g] = P.row;
        mu[g] = P.mult;
        wy[g] = P.wy;
        yy[g] = __dmul_rn(P.wy, __ldg(y + P.row));  // = the row's wy * y (forest.hpp:344)
      }
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (k + g >= e) break;
      const bool left = rank_of(rk_f, row[g]) <= thr_rank;
      if (left) {
        atomicOr(bits + (q[g] >> 5), 1u << (q[g] & 31u));
        ++o.nl;
        o.wl += mu[g];
        o.sl = __dadd_rn(o.sl, wy[g]);
        o.ql = __dadd_rn(o.ql, yy[g]);
      } else {
        o.wr += mu[g];
        o.sr = __dadd_rn(o.sr, wy[g]);
        o.qr = __dadd_rn(o.qr, yy[g]);
      }
    }
  }
}

// ---- route when column 0 has <= 2 distinct values: its order is the payload rows
// with rank 0, then those with rank 1 (one pass per level of column 0) -------------
template <typename RankT, int G>
__device__ void route_groups_warp(const Payload* pay,
                                  const double* __restrict__ y, uint32_t b, uint32_t e,
                                  const RankT* __restrict__ rk0, uint32_t k0levels,
                                  const RankT* __restrict__ rk_f, uint32_t thr_rank,
                                  uint32_t* bits, RouteOut& o, double* st) {
  const unsigned lane = lane_id();
  for (uint32_t grp = 0; grp < k0levels; ++grp) {
    for (uint32_t k0 = b; k0 < e; k0 += 32) {
      const uint32_t k = k0 + lane;
      Payload P{0, 0, 0.0};
      double yy = 0.0;
      bool sel = false, left = false;
      if (k < e) {
        P = pay[k];
        yy = __dmul_rn(P.wy, __ldg(y + P.row));
        sel = k0levels == 1 || rank_of(rk0, P.row) == grp;
        left = sel && rank_of(rk_f, P.row) <= thr_rank;
      }
      if (left) atomicOr(bits + (k >> 5), 1u << (k & 31u));
      const unsigned bl = __ballot_sync(kFull, left);
      const unsigned bs = __ballot_sync(kFull, sel);
      o.nl += __popc(bl);
      o.wl += warp_sum(left ? P.mult : 0u);
      o.wr += warp_sum((sel && !left) ? P.mult : 0u);
      tile_masked_sum2(P.wy, yy, bl, o.sl, o.ql, st);
      tile_masked_sum2(P.wy, yy, bs & ~bl, o.sr, o.qr, st);
    }
  }
}

template <typename RankT>
__device__ void route_groups_lane(const Payload* pay,
                                  const double* __restrict__ y, uint32_t b, uint32_t e,
                                  const RankT* __restrict__ rk0, uint32_t k0levels,
                                  const RankT* __restrict__ rk_f, uint32_t thr_rank,
                                  uint32_t* bits, RouteOut& o) {
  for (uint32_t grp = 0; grp < k0levels; ++grp) {
    for (uint32_t k = b; k < e; ++k) {
      const Payload P = pay[k];
      if (k0levels != 1 && rank_of(rk0, P.row) != grp) continue;
      const double yy = __dmul_rn(P.wy, __ldg(y + P.row));
      if (rank_of(rk_f, P.row) <= thr_rank) {
        atomicOr(bits + (k >> 5), 1u << (k & 31u));
        ++o.nl;
        o.wl += P.mult;
        o.sl = __dadd_rn(o.sl, P.wy);
        o.ql = __dadd_rn(o.ql, yy);
      } else {
        o.wr += P.mult;
        o.sr = __dadd_rn(o.sr, P.wy);
        o.qr = __dadd_rn(o.qr, yy);
      }
    }
  }
}

// sequential FP64 sums over the payload in row order (root stats, forest.hpp:221-226)
template <int G>
__device__ void root_sums_warp(const Payload* pay, const double* __restrict__ y,
                               uint32_t A, double& s_out, double& q_out, double* st) {
  const unsigned lane = lane_id();
  double s = 0.0, q = 0.0;
  for (uint32_t k0 = 0; k0 < A; k0 += 32 * G) {
    double x[G], c[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t k = k0 + g * 32 + lane;
      const Payload P = k < A ? pay[k] : Payload{0u, 0u, 0.0};
      x[g] = P.wy;
      c[g] = k < A ? __dmul_rn(P.wy, __ldg(y + P.row)) : 0.0;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t t0 = k0 + g * 32;
      if (t0 >= A) break;
      const uint32_t nv = min(32u, A - t0);
      tile_masked_sum2(x[g], c[g], nv == 32 ? kFull : ((1u << nv) - 1u), s, q, st);
    }
  }
  s_out = s;
  q_out = q;
}

}  // namespace

template <int NT, typename RankT>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) grow_kernel(const GrowArgs a) {
  constexpr int NW = NT / 32;
  constexpr int G = 4;
  extern __shared__ uint32_t dyn_smem[];
  __shared__ uint32_t sh_scan[NW + 2];
  __shared__ uint64_t sh_scan64[NW + 2];
  __shared__ double s_stage[NW][64];  // per-warp tile stage for the FP64 chains
  __shared__ uint32_t s_tree, s_A, s_F, s_E, s_S, s_nodes, s_totL, s_err;
  __shared__ unsigned long long s_pool;

  const DevData& d = a.d;
  const uint32_t n = static_cast<uint32_t>(d.n);
  const uint32_t p = d.p;
  const uint32_t tid = threadIdx.x;
  const unsigned lane = lane_id();
  const unsigned wid = warp_id();
  const SlotLayout& L = a.L;
  const uint32_t stride = L.stride;
  const uint32_t nl_cols = d.nlisted;
  const uint32_t ostride = d.order_stride;

  char* slot = a.scratch + static_cast<size_t>(blockIdx.x) * L.bytes;
  uint32_t* mult_g = reinterpret_cast<uint32_t*>(slot + L.off_mult);
  Payload* pay[2] = {reinterpret_cast<Payload*>(slot + L.off_pay0),
                     reinterpret_cast<Payload*>(slot + L.off_pay1)};
  uint32_t* lists[2] = {reinterpret_cast<uint32_t*>(slot + L.off_list0),
                        reinterpret_cast<uint32_t*>(slot + L.off_list1)};
  uint32_t* seg[2] = {reinterpret_cast<uint32_t*>(slot + L.off_seg0),
                      reinterpret_cast<uint32_t*>(slot + L.off_seg1)};
  NodeWork* front[2] = {reinterpret_cast<NodeWork*>(slot + L.off_front0),
                        reinterpret_cast<NodeWork*>(slot + L.off_front1)};
  SegTab* segtab = reinterpret_cast<SegTab*>(slot + L.off_segtab);
  uint32_t* e2f = reinterpret_cast<uint32_t*>(slot + L.off_e2f);
  uint16_t* samp = reinterpret_cast<uint16_t*>(slot + L.off_samp);
  ChainRes* res = reinterpret_cast<ChainRes*>(slot + L.off_res);
  SplitInfo* spl = reinterpret_cast<SplitInfo*>(slot + L.off_split);
  int32_t* nf = reinterpret_cast<int32_t*>(slot + L.off_nf);
  double* nthr = reinterpret_cast<double*>(slot + L.off_nthr);
  int32_t* nleft = reinterpret_cast<int32_t*>(slot + L.off_nleft);
  double* nval = reinterpret_cast<double*>(slot + L.off_nval);
  uint32_t* nrank = reinterpret_cast<uint32_t*>(slot + L.off_nrank);
  uint32_t* chunk_cnt = reinterpret_cast<uint32_t*>(slot + L.off_chunk);
  int2* off2 = reinterpret_cast<int2*>(slot + L.off_off2);
  const uint32_t nwords = (n + 31u) / 32u;
  const uint32_t nblk64 = (n + 63u) / 64u;
  const size_t bw = grow_bits_words(n, stride);
  uint32_t* bits = a.bits_in_smem ? dyn_smem : reinterpret_cast<uint32_t*>(slot + L.off_gbits);
  uint32_t* pref = a.bits_in_smem ? dyn_smem + bw : reinterpret_cast<uint32_t*>(slot + L.off_gpref);
  const RankT* rank = static_cast<const RankT*>(d.rank);
  const int32_t list0 = d.list_of[0];
  const uint32_t k0levels =
      static_cast<uint32_t>(d.vals_off[1] - d.vals_off[0]);  // distinct values of column 0

  // optional per-phase cycle accounting (thread 0, clock64), enabled by a.prof
  long long ph_acc[kPhases];
  long long ph_last = clock64();
  for (int i = 0; i < kPhases; ++i) ph_acc[i] = 0;
#define PHASE(k)                        \
  do {                                  \
    if (a.prof && tid == 0) {           \
      const long long now_ = clock64(); \
      ph_acc[(k)] += now_ - ph_last;    \
      ph_last = now_;                   \
    }                                   \
  } while (0)

  for (;;) {
    __syncthreads();
    PHASE(13);
    if (tid == 0) {
      s_tree = atomicAdd(a.queue, 1u);
      s_err = 0;
    }
    __syncthreads();
    const uint32_t tl = s_tree;
    if (tl >= a.tree_end - a.tree_begin) break;
    // this tree's parameters and its index in its forest (several forests: tree_cell)
    const uint32_t cell = a.tree_cell ? a.tree_cell[tl] : 0u;
    const uint32_t m = a.tree_cell ? a.cell_mtry[cell] : a.mtry;
    const uint32_t mns = a.tree_cell ? a.cell_mns[cell] : a.mns;
    const uint64_t t = a.tree_cell ? uint64_t{a.tree_t[tl]} : uint64_t{a.tree_begin} + tl;
    const uint64_t seed = a.tree_cell ? a.cell_seed[cell] : a.seed;
    const uint64_t key = dmix64(seed ^ a.tag_tree ^ dmix64(t));

    // ---- bootstrap (forest.hpp:184-195) ----
    for (uint32_t i = tid; i < n; i += NT) mult_g[i] = 0u;
    __syncthreads();
    for (uint32_t j = tid; j < n; j += NT) {
      const uint32_t r = static_cast<uint32_t>(draw_bounded(key, uint64_t{j} + 1u, n));
      if (a.inbag) a.inbag[static_cast<size_t>(tl) * n + j] = r;
      atomicAdd(mult_g + r, 1u);
    }
    __syncthreads();
    PHASE(0);
    // in-bag bitmap by row + 64-row prefix counts
    for (uint32_t w = wid; w < nwords; w += NW) {
      const uint32_t r = w * 32u + lane;
      const unsigned bl = __ballot_sync(kFull, r < n && mult_g[r] > 0u);
      if (lane == 0) bits[w] = bl;
    }
    __syncthreads();
    {
      uint32_t carry = 0;
      for (uint32_t base = 0; base < nblk64; base += NT) {
        const uint32_t i = base + tid;
        uint32_t v = 0;
        if (i < nblk64)
          v = __popc(bits[2 * i]) + (2 * i + 1 < nwords ? __popc(bits[2 * i + 1]) : 0u);
        uint32_t tot;
        const uint32_t ex = block_excl_scan<NT>(v, sh_scan, &tot);
        if (i < nblk64) pref[i] = carry + ex;
        carry += tot;
      }
      if (tid == 0) s_A = carry;
    }
    __syncthreads();
    PHASE(1);
    const uint32_t A0 = s_A;
    if (A0 > stride) {
      if (tid == 0) atomicExch(a.err, 2);
      continue;
    }
    // payload in row order (forest.hpp:194-195: weighted_y = mult*y)
    for (uint32_t r = tid; r < n; r += NT) {
      if (!get_bit(bits, r)) continue;
      const uint32_t pos = inbag_pos(bits, pref, r);
      const uint32_t mu = mult_g[r];
      const double yr = __ldg(d.y + r);
      const double wy = __dmul_rn(static_cast<double>(mu), yr);
      pay[0][pos] = Payload{r, mu, wy};
      seg[0][pos] = 0u;
    }
    __syncthreads();
    PHASE(2);
    // per listed column: stable in-bag filter of the presort, flattened over
    // (list, position); every list holds exactly A0 in-bag rows
    {
      const uint64_t total = uint64_t{nl_cols} * ostride;
      constexpr uint32_t kRow = NT * 4;
      uint64_t carry = 0;
      for (uint64_t base = 0; base < total; base += uint64_t{kRow} * 4) {
        uint32_t r[16], in = 0, li[4], k0[4];
        uint64_t cnt = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint64_t g0 = base + uint64_t{v} * kRow + uint64_t{tid} * 4;
          li[v] = 0;
          k0[v] = 0;
          uint32_t c = 0;
          if (g0 < total) {
            li[v] = static_cast<uint32_t>(g0 / ostride);
            k0[v] = static_cast<uint32_t>(g0 - uint64_t{li[v]} * ostride);
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(d.order + g0));
            r[4 * v] = x.x;
            r[4 * v + 1] = x.y;
            r[4 * v + 2] = x.z;
            r[4 * v + 3] = x.w;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (k0[v] + j < n && get_bit(bits, r[4 * v + j])) {
                in |= 1u << (4 * v + j);
                ++c;
              }
          }
          cnt |= uint64_t{c} << (16 * v);
        }
        uint64_t tot;
        const uint64_t ex = block_excl_scan64<NT>(cnt, sh_scan64, &tot);
        uint64_t rowbase = carry;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint32_t o = static_cast<uint32_t>(rowbase + ((ex >> (16 * v)) & 0xffffu) -
                                             uint64_t{li[v]} * A0);
          uint32_t* out = lists[0] + static_cast<size_t>(li[v]) * stride;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if ((in >> (4 * v + j)) & 1u) out[o++] = inbag_pos(bits, pref, r[4 * v + j]);
          rowbase += (tot >> (16 * v)) & 0xffffu;
        }
        carry = rowbase;
      }
    }
    __syncthreads();
    if (wid == 0) {
      double s, q;
      root_sums_warp<G>(pay[0], a.d.y, A0, s, q, s_stage[wid]);
      if (lane == 0) {
        front[0][0] = NodeWork{0u, A0, 0u, 0u, static_cast<double>(n), s, q};
        nf[0] = -1;
        nthr[0] = 0.0;
        nleft[0] = -1;
        nval[0] = 0.0;
        nrank[0] = 0u;
        s_F = 1;
        s_nodes = 1;
      }
    }
    __syncthreads();
    PHASE(3);

    // ---- level loop (forest.hpp:233-374) ----
    uint32_t cur = 0, A = A0;
    uint64_t elig_base = 0;
    unsigned long long split_rows_acc = 0;  // meaningful in thread 0 only
    for (;;) {
      const uint32_t F = s_F;
      const NodeWork* fr = front[cur];
      // leaf tests + eligible compaction (forest.hpp:244-253)
      {
        uint32_t carry = 0;
        for (uint32_t base = 0; base < F; base += NT) {
          const uint32_t f = base + tid;
          uint32_t el = 0;
          if (f < F) {
            const NodeWork nw = fr[f];
            const double sse = __dsub_rn(nw.q, __ddiv_rn(__dmul_rn(nw.s, nw.s), nw.w));
            const bool too_small = nw.w < 2.0 * static_cast<double>(mns);
            const bool pure = sse <= __dmul_rn(1e-12, nw.q > 1.0 ? nw.q : 1.0);
            if (too_small || pure)
              nval[nw.id] = __ddiv_rn(nw.s, nw.w);
            else
              el = 1;
            segtab[f].offL = INT_MIN;
          }
          uint32_t tot;
          const uint32_t ex = block_excl_scan<NT>(el, sh_scan, &tot);
          if (el) e2f[carry + ex] = f;
          carry += tot;
        }
        if (tid == 0) s_E = carry;
      }
      __syncthreads();
      PHASE(5);
      const uint32_t E = s_E;
      // mtry sampling: partial Fisher-Yates over a fresh pool, then ascending
      // (forest.hpp:258-266); counters continue the tree's stream after the n
      // bootstrap draws, m per eligible node in BFS order
      for (uint32_t e = tid; e < E; e += NT) {
        uint16_t pool[kMaxP];
        for (uint32_t c = 0; c < p; ++c) pool[c] = static_cast<uint16_t>(c);
        const uint64_t ctr = uint64_t{n} + (elig_base + e) * m;
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
        for (uint32_t i = 0; i < m; ++i) samp[static_cast<size_t>(e) * m + i] = pool[i];
      }
      __syncthreads();
      PHASE(6);
      // split chains (forest.hpp:268-297)
      const uint32_t ntask = E * m;
      for (uint32_t k = wid; k < ntask; k += NW) {
        const NodeWork nw = fr[e2f[k / m]];
        if (nw.e - nw.b < kLaneMax) continue;
        const uint32_t c = samp[k];
        const int32_t li = d.list_of[c];
        const RankT* rk_c = rank + static_cast<size_t>(c) * n;
        double bg;
        uint32_t bp;
        if (li >= 0)
          chain_warp<RankT, G>(lists[cur] + static_cast<size_t>(li) * stride, nw.b, nw.e,
                               pay[cur], rk_c, nw.w, nw.s, bg, bp, s_stage[wid]);
        else
          chain_bin_warp<RankT, G>(pay[cur], nw.b, nw.e, rk_c, nw.w, nw.s, bg, bp,
                                   s_stage[wid]);
        if (lane == 0) res[k] = ChainRes{bg, bp, 0u};
      }
      for (uint32_t k = tid; k < ntask; k += NT) {
        const NodeWork nw = fr[e2f[k / m]];
        if (nw.e - nw.b >= kLaneMax) continue;
        const uint32_t c = samp[k];
        const int32_t li = d.list_of[c];
        const RankT* rk_c = rank + static_cast<size_t>(c) * n;
        double bg;
        uint32_t bp;
        if (li >= 0)
          chain_lane<RankT>(lists[cur] + static_cast<size_t>(li) * stride, nw.b, nw.e,
                            pay[cur], rk_c, nw.w, nw.s, bg, bp);
        else
          chain_bin_lane<RankT>(pay[cur], nw.b, nw.e, rk_c, nw.w, nw.s, bg, bp);
        res[k] = ChainRes{bg, bp, 0u};
      }
      __syncthreads();
      PHASE(7);
      // decide + number children in frontier order (forest.hpp:299-319)
      {
        const uint32_t nodes0 = s_nodes;
        uint32_t carry = 0, ccarry = 0;
        for (uint32_t base = 0; base < E; base += NT) {
          const uint32_t e = base + tid;
          uint32_t sp = 0, c = 0, thr_rank = 0;
          double thr = 0.0;
          NodeWork nw{};
          if (e < E) {
            nw = fr[e2f[e]];
            double bg = -INFINITY;
            uint32_t bi = 0, bp = 0;
            for (uint32_t i = 0; i < m; ++i) {
              const ChainRes r = res[static_cast<size_t>(e) * m + i];
              if (r.gain > bg) {
                bg = r.gain;
                bi = i;
                bp = r.pos;
              }
            }
            if (bg == -INFINITY) {
              nval[nw.id] = __ddiv_rn(nw.s, nw.w);  // all sampled columns constant
            } else {
              sp = 1;
              c = samp[static_cast<size_t>(e) * m + bi];
              const int32_t li = d.list_of[c];
              const double* vals = d.vals + d.vals_off[c];
              double prev, v;
              uint32_t lo, hi;
              if (li >= 0) {
                const uint32_t* lc = lists[cur] + static_cast<size_t>(li) * stride;
                const uint32_t r1 = pay[cur][lc[bp - 1]].row;
                const uint32_t r0 = pay[cur][lc[bp]].row;
                prev = d.col[static_cast<size_t>(c) * n + r1];
                v = d.col[static_cast<size_t>(c) * n + r0];
                lo = rank_of(rank + static_cast<size_t>(c) * n, r1);
                hi = rank_of(rank + static_cast<size_t>(c) * n, r0);
              } else {  // two-level column: the boundary is between its two values
                prev = vals[0];
                v = vals[1];
                lo = 0;
                hi = 1;
              }
              thr = __dadd_rn(prev, __ddiv_rn(__dsub_rn(v, prev), 2.0));
              if (thr >= v) thr = prev;
              // largest distinct-value rank whose value <= thr (vals[lo] <= thr < vals[hi])
              while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (vals[mid] <= thr) lo = mid; else hi = mid;
              }
              thr_rank = lo;
            }
          }
          uint32_t tot;
          const uint32_t ex = block_excl_scan<NT>(sp, sh_scan, &tot);
          const uint32_t cnt = sp ? nw.e - nw.b : 0u;
          uint32_t ctot;
          const uint32_t cex = block_excl_scan<NT>(cnt, sh_scan, &ctot);
          if (sp) {
            const uint32_t s = carry + ex;
            const uint32_t child = nodes0 + 2 * s;
            nf[nw.id] = static_cast<int32_t>(c);
            nthr[nw.id] = thr;
            nleft[nw.id] = static_cast<int32_t>(child);
            nrank[nw.id] = thr_rank;
            for (uint32_t h = 0; h < 2; ++h) {
              nf[child + h] = -1;
              nthr[child + h] = 0.0;
              nleft[child + h] = -1;
              nval[child + h] = 0.0;
              nrank[child + h] = 0u;
            }
            spl[s] = SplitInfo{e2f[e], c, thr_rank, cnt, 0u, ccarry + cex, 0u, 0u};
          }
          carry += tot;
          ccarry += ctot;
        }
        if (tid == 0) {
          s_S = carry;
          s_nodes = nodes0 + 2 * carry;
          s_A = ccarry;
          split_rows_acc += ccarry;
        }
      }
      // the goes-left bitmap over payload positions starts empty each level
      for (uint32_t w = tid; w < (A + 31u) / 32u; w += NT) bits[w] = 0u;
      __syncthreads();
      PHASE(8);
      const uint32_t S = s_S;
      elig_base += E;
      if (S == 0) break;
      if (s_nodes > L.nodes_cap || 2 * S > L.fmax) {
        if (tid == 0) atomicExch(a.err, 3);
        s_err = 1;
        break;
      }
      const uint32_t nxt = cur ^ 1u;
      // route rows of every split node through column-0 order (forest.hpp:323-352)
      {
        const uint32_t* l0 = list0 >= 0 ? lists[cur] + static_cast<size_t>(list0) * stride
                                        : nullptr;
        const RankT* rk0 = rank;  // column 0
        for (int pass = 0; pass < 2; ++pass) {
          // pass 0: warps take large nodes; pass 1: lanes take small ones
          const uint32_t step = pass == 0 ? NW : NT;
          for (uint32_t s = pass == 0 ? wid : tid; s < S; s += step) {
            const SplitInfo si = spl[s];
            if ((pass == 0) != (si.cnt >= kLaneMax)) continue;
            const NodeWork nw = fr[si.f];
            const RankT* rk_f = rank + static_cast<size_t>(si.c) * n;
            RouteOut o{0, 0, 0, 0.0, 0.0, 0.0, 0.0};
            if (pass == 0) {
              if (l0)
                route_warp<RankT, G>(l0, nw.b, nw.e, pay[cur], a.d.y, rk_f, si.thr_rank,
                                     bits, o, s_stage[wid]);
              else
                route_groups_warp<RankT, G>(pay[cur], a.d.y, nw.b, nw.e, rk0, k0levels,
                                            rk_f, si.thr_rank, bits, o, s_stage[wid]);
              if (lane != 0) continue;
            } else {
              if (l0)
                route_lane<RankT>(l0, nw.b, nw.e, pay[cur], a.d.y, rk_f, si.thr_rank, bits,
                                  o);
              else
                route_groups_lane<RankT>(pay[cur], a.d.y, nw.b, nw.e, rk0, k0levels, rk_f,
                                         si.thr_rank, bits, o);
            }
            spl[s].nl = o.nl;
            const uint32_t child = static_cast<uint32_t>(nleft[nw.id]);
            front[nxt][2 * s] = NodeWork{si.base, si.base + o.nl, child, 0u,
                                         static_cast<double>(o.wl), o.sl, o.ql};
            front[nxt][2 * s + 1] = NodeWork{si.base + o.nl, si.base + si.cnt, child + 1, 0u,
                                             static_cast<double>(o.wr), o.sr, o.qr};
          }
        }
      }
      __syncthreads();
      PHASE(9);
      // segment table (stable partition offsets into compacted children) and
      // per-word prefix counts of the goes-left bitmap
      {
        uint32_t carry = 0;
        for (uint32_t base = 0; base < S; base += NT) {
          const uint32_t s = base + tid;
          const uint32_t nl = s < S ? spl[s].nl : 0u;
          uint32_t tot;
          const uint32_t ex = block_excl_scan<NT>(nl, sh_scan, &tot);
          if (s < S) {
            const SplitInfo si = spl[s];
            const uint32_t bL = carry + ex;  // lefts before this segment
            const uint32_t b = fr[si.f].b;
            segtab[si.f] = SegTab{static_cast<int32_t>(si.base) - static_cast<int32_t>(bL),
                                  static_cast<int32_t>(si.base + nl) -
                                      static_cast<int32_t>(b) + static_cast<int32_t>(bL),
                                  2 * s, 0u};
          }
          carry += tot;
        }
        if (tid == 0) s_totL = carry;
        const uint32_t aw = (A + 31u) / 32u;
        carry = 0;
        for (uint32_t base = 0; base < aw; base += NT) {
          const uint32_t w = base + tid;
          const uint32_t v = w < aw ? __popc(bits[w]) : 0u;
          uint32_t tot;
          const uint32_t ex = block_excl_scan<NT>(v, sh_scan, &tot);
          if (w < aw) pref[w] = carry + ex;
          carry += tot;
        }
      }
      __syncthreads();
      PHASE(10);
      // payload pass: element k goes to offL + lefts-before-k, or offR + k - that
      // (it also expands the segment offsets per position for the list pass)
      for (uint32_t k = tid; k < A; k += NT) {
        const uint32_t f = seg[cur][k];
        const SegTab tb = segtab[f];
        off2[k] = make_int2(tb.offL, tb.offR);
        if (tb.offL == INT_MIN) continue;
        const bool l = get_bit(bits, k);
        const int32_t lp = static_cast<int32_t>(bits_before(bits, pref, k));
        const uint32_t dst = static_cast<uint32_t>(l ? tb.offL + lp
                                                     : tb.offR + static_cast<int32_t>(k) - lp);
        pay[nxt][dst] = pay[cur][k];
        seg[nxt][dst] = tb.child + (l ? 0u : 1u);
      }
      __syncthreads();
      PHASE(11);
      // list pass: the same partition applied to every listed column, flattened
      // over (list, position) with a per-list left-count offset li*totL; the new
      // entry (payload position in the next level) comes from the same bitmap
      // Tile = 4 rows x NT threads x 4 consecutive elements: every uint4 load and
      // every row of stores is coalesced across the warp; one packed 64-bit block
      // scan yields the four rows' left-count prefixes.
      // Per element: one 8-byte segment-offset load and one shared bitmap word give
      // both the side and the element's next-level payload position; both are kept in
      // registers across the scan (32-bit index math: nlisted * A < 2^32).
      // Two phases, no block barrier per tile: (1) every warp counts the kept-left
      // entries of its chunks (kChunk flat elements), (2) one block scan over the chunk
      // counts, (3) every warp re-reads its chunks and scatters with its own running
      // prefix (warp-level scans only), so warps stream independently with several
      // loads in flight.
      {
        const uint32_t A16 = (A + 15u) & ~15u;
        const uint32_t total = nl_cols * A16;
        const uint32_t totL = s_totL;
        const uint32_t nchunk = (total + kChunk - 1) / kChunk;
        for (uint32_t c = wid; c < nchunk; c += NW) {
          const uint32_t ce = min(total, (c + 1) * kChunk);
          uint32_t cnt = 0;
#pragma unroll 2
          for (uint32_t s = c * kChunk; s < ce; s += 128) {
            ListQuad v;
            load_quad(v, s + lane * 4, A16, A, ce, stride, lists[cur], off2);
            cnt += __popc(side_quad(v, bits, pref));
          }
          cnt = warp_sum(cnt);
          if (lane == 0) chunk_cnt[c] = cnt;
        }
        __syncthreads();
        {
          uint32_t carry = 0;
          for (uint32_t base = 0; base < nchunk; base += NT) {
            const uint32_t c = base + tid;
            const uint32_t v = c < nchunk ? chunk_cnt[c] : 0u;
            uint32_t tot;
            const uint32_t ex = block_excl_scan<NT>(v, sh_scan, &tot);
            if (c < nchunk) chunk_cnt[c] = carry + ex;
            carry += tot;
          }
        }
        __syncthreads();
        for (uint32_t c = wid; c < nchunk; c += NW) {
          const uint32_t ce = min(total, (c + 1) * kChunk);
          uint32_t run = chunk_cnt[c];
#pragma unroll 2
          for (uint32_t s = c * kChunk; s < ce; s += 128) {
            ListQuad v;
            load_quad(v, s + lane * 4, A16, A, ce, stride, lists[cur], off2);
            const uint32_t lf = side_quad(v, bits, pref);
            const uint32_t mine = __popc(lf);
            const uint32_t inc = warp_incl_scan(mine);
            int32_t pl = static_cast<int32_t>(run + inc - mine - v.li * totL);
            uint32_t* dstl = lists[nxt] + static_cast<size_t>(v.li) * stride;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (!((v.keep >> j) & 1u)) continue;
              const bool l = (lf >> j) & 1u;
              const int32_t off = static_cast<int32_t>(v.f[j]);
              const uint32_t dst = static_cast<uint32_t>(
                  l ? off + pl : off + static_cast<int32_t>(v.k0 + j) - pl);
              pl += l ? 1 : 0;
              dstl[dst] = v.q[j];
            }
            run += __shfl_sync(kFull, inc, 31);
          }
        }
      }
      __syncthreads();
      PHASE(12);
      if (tid == 0) s_F = 2 * S;
      A = s_A;
      cur = nxt;
      __syncthreads();
    }
    __syncthreads();
    if (s_err) continue;

    // ---- emit the tree: BFS node SoA into the forest pool ----
    const uint32_t count = s_nodes;
    if (tid == 0) {
      const unsigned long long off = atomicAdd(a.pool_used, static_cast<unsigned long long>(count));
      s_pool = off;
      a.tree_off[tl] = off;
      a.tree_cnt[tl] = count;
      atomicAdd(a.split_rows, split_rows_acc);
      if (off + count > a.pool_cap) atomicExch(a.err, 1);
    }
    __syncthreads();
    const unsigned long long off = s_pool;
    if (off + count <= a.pool_cap) {
      for (uint32_t i = tid; i < count; i += NT) {
        a.pool_feature[off + i] = nf[i];
        a.pool_thr[off + i] = nthr[i];
        a.pool_left[off + i] = nleft[i];
        a.pool_value[off + i] = nval[i];
        a.pool_rank[off + i] = nrank[i];
      }
    }
    // ---- out-of-bag leaves (walk per OOB row, forest.hpp:418-435) ----
    if (a.oobleaf) {
      uint32_t* ol = a.oobleaf + static_cast<size_t>(tl) * n;
      for (uint32_t r = tid; r < n; r += NT) {
        if (mult_g[r]) {
          ol[r] = kInBag;
          continue;
        }
        int32_t i = 0;
        int32_t fi = nf[0];
        while (fi >= 0) {
          const bool left = rank_of(rank + static_cast<size_t>(fi) * n, r) <= nrank[i];
          i = nleft[i] + (left ? 0 : 1);
          fi = nf[i];
        }
        ol[r] = static_cast<uint32_t>(i);
      }
    }
  }
  if (a.prof && tid == 0)
    for (int i = 0; i < kPhases; ++i)
      atomicAdd(a.prof + i, static_cast<unsigned long long>(ph_acc[i]));
#undef PHASE
}

namespace {
template <int NT, typename RankT>
cudaError_t launch_t(const GrowArgs& a, int slots, size_t smem, cudaStream_t st,
                     int* blocks_per_sm) {
  auto k = grow_kernel<NT, RankT>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (blocks_per_sm) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k, NT, smem);
  k<<<slots, NT, smem, st>>>(a);
  return cudaGetLastError();
}
}  // namespace

// slots == 0 with blocks_per_sm != nullptr: occupancy query only
cudaError_t launch_grow(int nt, int rank_bytes, const GrowArgs& a, int slots, size_t smem,
                        cudaStream_t st, int* blocks_per_sm) {
  if (nt == 512)
    return rank_bytes == 2 ? launch_t<512, uint16_t>(a, slots, smem, st, blocks_per_sm)
                           : launch_t<512, uint32_t>(a, slots, smem, st, blocks_per_sm);
  return rank_bytes == 2 ? launch_t<256, uint16_t>(a, slots, smem, st, blocks_per_sm)
                         : launch_t<256, uint32_t>(a, slots, smem, st, blocks_per_sm);
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

SlotLayout make_layout(uint64_t n, uint32_t p, uint32_t nlisted, uint32_t mtry, uint32_t mns,
                       bool gbits) {
  (void)p;
  SlotLayout L{};
  // in-bag distinct rows: 0.632 n on average; bound it generously (checked at run time)
  const double exp_a = 0.6322 * static_cast<double>(n) + 8.0 * std::sqrt(static_cast<double>(n)) + 64.0;
  uint64_t stride = static_cast<uint64_t>(exp_a);
  if (stride > n) stride = n;
  stride = (stride + 15) & ~uint64_t{15};
  L.stride = static_cast<uint32_t>(stride);
  // a splittable node weighs >= 2*mns, so a level has <= n/(2 mns) eligible nodes
  // and <= n/mns frontier nodes
  const uint64_t emax = std::min<uint64_t>(stride, n / (2 * uint64_t{mns}) + 2);
  const uint64_t fmax = std::min<uint64_t>(stride + 2, 2 * emax + 2);
  L.emax = static_cast<uint32_t>(emax);
  L.fmax = static_cast<uint32_t>(fmax);
  L.nodes_cap = static_cast<uint32_t>(2 * stride + 2);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L.off_mult = take(n * 4);
  L.off_pay0 = take(stride * sizeof(Payload));
  L.off_pay1 = take(stride * sizeof(Payload));
  L.off_list0 = take(size_t{nlisted} * stride * 4 + 64);
  L.off_list1 = take(size_t{nlisted} * stride * 4 + 64);
  L.off_seg0 = take(stride * 4 + 64);
  L.off_seg1 = take(stride * 4 + 64);
  L.off_front0 = take(fmax * sizeof(NodeWork));
  L.off_front1 = take(fmax * sizeof(NodeWork));
  L.off_segtab = take(fmax * sizeof(SegTab));
  L.off_e2f = take(emax * 4);
  L.off_ecls = take(emax * 4);
  L.off_wsplit = take(emax * 4);
  L.off_samp = take(emax * mtry * 2);
  L.off_res = take(emax * mtry * sizeof(ChainRes));
  L.off_split = take(emax * sizeof(SplitInfo));
  L.off_nf = take(size_t{L.nodes_cap} * 4);
  L.off_nthr = take(size_t{L.nodes_cap} * 8);
  L.off_nleft = take(size_t{L.nodes_cap} * 4);
  L.off_nval = take(size_t{L.nodes_cap} * 8);
  L.off_nrank = take(size_t{L.nodes_cap} * 4);
  // chunk counters: list pass (nlisted x stride) and the wide grower's list init
  // (nlisted x padded n)
  L.off_chunk = take((size_t{nlisted} * std::max<uint64_t>(stride, (n + 15) & ~uint64_t{15}) /
                          kListChunk + 4) * 4);
  L.off_off2 = take(stride * 8 + 64);
  if (gbits) {
    L.off_gbits = take(grow_bits_words(n, L.stride) * 4);
    L.off_gpref = take(grow_pref_words(n, L.stride) * 4);
  }
  L.bytes = o;
  return L;
}

}  // namespace aiwc_b200

// the batched (wide) grower shares this file's device helpers
#include "grow_wide.cuh"
