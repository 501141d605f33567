/* TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Never linked into the product;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * A plain-C restatement of the reference forest path,
 * written from the algorithm, not from the reference's data structures:
 *   - the reference keeps p presorted row lists per tree and stably partitions
 *     them every level (forest.hpp:197-209, 355-371); this oracle instead sorts
 *     each node's rows by (value, row) on demand, which yields the same visiting
 *     order because a stable partition of a (value,row)-sorted list stays sorted;
 *   - splitmix64 / FNV-1a / derive_seed / bounded(): rng.hpp:13-59;
 *   - bootstrap: forest.hpp:182-195;  root sums in row order: forest.hpp:217-228;
 *   - leaf tests: forest.hpp:244-253;  mtry partial Fisher-Yates: forest.hpp:255-266;
 *   - split scan (midpoint, strict '>' first max): forest.hpp:268-297;
 *   - child numbering in frontier order (BFS ids): forest.hpp:299-319;
 *   - child sums in column-0 order: forest.hpp:323-344;
 *   - OOB in tree order: forest.hpp:393-454;  predict: forest.hpp:42-50, 77-81.
 * All floating point is IEEE binary64, round-to-nearest, no contraction
 * (built with -ffp-contract=off), matching the reference's x86-64 build.
 *
 * Pinned against the reference itself: tests/test_oracle.py compares this
 * oracle tree-for-tree with oracle/_ref/libaiwc_ref.so and with the committed
 * goldens in tests/golden/ (made by tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9e3779b97f4a7c15ull

uint64_t oracle_mix64(uint64_t x) {
  x += GOLDEN;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

uint64_t oracle_fnv1a64(const char* s, uint64_t len) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < len; ++i) {
    h ^= (unsigned char)s[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t oracle_derive_seed(uint64_t seed, const char* tag, uint64_t index) {
  return oracle_mix64(seed ^ oracle_fnv1a64(tag, strlen(tag)) ^ oracle_mix64(index));
}

/* draw k (1-based) of the stream keyed by `key` is mix64(key + k*GOLDEN) */
static uint64_t draw_bounded(uint64_t* state, uint64_t n) {
  *state += GOLDEN;
  const uint64_t x = oracle_mix64(*state);
  return (uint64_t)(((unsigned __int128)x * n) >> 64);
}

typedef struct {
  double v;
  uint32_t r;
} Pair;

static int pair_cmp(const void* a, const void* b) {
  const Pair* x = (const Pair*)a;
  const Pair* y = (const Pair*)b;
  if (x->v < y->v) return -1;
  if (x->v > y->v) return 1;
  return (x->r > y->r) - (x->r < y->r);
}

/* node's rows (row order) -> (value of column c, row) ascending */
static void sorted_by(const double* colc, const uint32_t* rows, uint64_t cnt, Pair* out) {
  for (uint64_t k = 0; k < cnt; ++k) {
    out[k].v = colc[rows[k]];
    out[k].r = rows[k];
  }
  qsort(out, cnt, sizeof(Pair), pair_cmp);
}

typedef struct {
  int32_t id;
  uint64_t b, e; /* range in the level's row buffer (rows ascending) */
  double w, s, q;
} Work;

/* Grows tree `tree_index` of a forest keyed by `seed`.  Node arrays must hold
 * 2n entries; inbag_out (nullable) receives the n bootstrap draws.
 * Returns node count, or -1 on allocation failure. */
int64_t oracle_grow_tree(const double* col, const double* y, uint64_t n, uint32_t p,
                         uint32_t mtry, uint32_t mns, uint64_t seed, uint64_t tree_index,
                         int32_t* feature, double* threshold, int32_t* left,
                         int32_t* right, double* value, uint32_t* inbag_out) {
  uint64_t st = oracle_derive_seed(seed, "tree", tree_index);
  uint32_t* mult = calloc(n, sizeof(uint32_t));
  double* wy = malloc(n * sizeof(double));
  uint32_t* rows = malloc(n * sizeof(uint32_t));
  uint32_t* rows2 = malloc(n * sizeof(uint32_t));
  Work* front = malloc((n + 1) * sizeof(Work));
  Work* next = malloc((n + 1) * sizeof(Work));
  Pair* pairs = malloc(n * sizeof(Pair));
  uint32_t* pool = malloc(p * sizeof(uint32_t));
  char* goes_left = malloc(n);
  if (!mult || !wy || !rows || !rows2 || !front || !next || !pairs || !pool || !goes_left)
    return -1;

  for (uint64_t j = 0; j < n; ++j) {
    const uint32_t r = (uint32_t)draw_bounded(&st, n);
    if (inbag_out) inbag_out[j] = r;
    mult[r]++;
  }
  uint64_t active = 0;
  double s = 0, q = 0;
  for (uint64_t i = 0; i < n; ++i) {
    wy[i] = (double)mult[i] * y[i];
    if (!mult[i]) continue;
    rows[active++] = (uint32_t)i;
    s += wy[i];
    q += wy[i] * y[i];
  }

  int64_t count = 1;
  feature[0] = -1; threshold[0] = 0; left[0] = -1; right[0] = -1; value[0] = 0;
  uint64_t nf = 1;
  front[0].id = 0; front[0].b = 0; front[0].e = active;
  front[0].w = (double)n; front[0].s = s; front[0].q = q;
  const uint32_t m = mtry < p ? mtry : p;

  while (nf) {
    uint64_t nn = 0, fill = 0;
    for (uint64_t f = 0; f < nf; ++f) {
      const Work nw = front[f];
      const double sse = nw.q - nw.s * nw.s / nw.w;
      const double qmax = nw.q > 1.0 ? nw.q : 1.0;
      if (nw.w < 2.0 * (double)mns || sse <= 1e-12 * qmax) {
        value[nw.id] = nw.s / nw.w;
        continue;
      }
      for (uint32_t c = 0; c < p; ++c) pool[c] = c;
      for (uint32_t i = 0; i < m; ++i) {
        const uint32_t j = i + (uint32_t)draw_bounded(&st, p - i);
        const uint32_t t = pool[i]; pool[i] = pool[j]; pool[j] = t;
      }
      for (uint32_t i = 1; i < m; ++i) /* insertion sort of the sample */
        for (uint32_t k = i; k > 0 && pool[k - 1] > pool[k]; --k) {
          const uint32_t t = pool[k]; pool[k] = pool[k - 1]; pool[k - 1] = t;
        }
      const uint64_t cnt = nw.e - nw.b;
      double best = -INFINITY, best_thr = 0;
      int32_t best_col = -1;
      for (uint32_t ci = 0; ci < m; ++ci) {
        const uint32_t c = pool[ci];
        sorted_by(col + (uint64_t)c * n, rows + nw.b, cnt, pairs);
        double wl = 0, sl = 0, prev = pairs[0].v;
        for (uint64_t k = 0; k < cnt; ++k) {
          const double v = pairs[k].v;
          if (v != prev) {
            double thr = prev + (v - prev) / 2.0;
            if (thr >= v) thr = prev;
            const double wr = nw.w - wl;
            const double g = sl * sl / wl + (nw.s - sl) * (nw.s - sl) / wr;
            if (g > best) { best = g; best_col = (int32_t)c; best_thr = thr; }
            prev = v;
          }
          wl += (double)mult[pairs[k].r];
          sl += wy[pairs[k].r];
        }
      }
      if (best_col < 0) {
        value[nw.id] = nw.s / nw.w;
        continue;
      }
      feature[nw.id] = best_col;
      threshold[nw.id] = best_thr;
      left[nw.id] = (int32_t)count;
      right[nw.id] = (int32_t)count + 1;
      for (int k = 0; k < 2; ++k) {
        feature[count + k] = -1; threshold[count + k] = 0;
        left[count + k] = -1; right[count + k] = -1; value[count + k] = 0;
      }
      /* child sums visit the parent's rows in column-0 order */
      Work L = {(int32_t)count, 0, 0, 0, 0, 0}, R = {(int32_t)count + 1, 0, 0, 0, 0, 0};
      count += 2;
      const double* fcol = col + (uint64_t)best_col * n;
      sorted_by(col, rows + nw.b, cnt, pairs);
      uint64_t nl = 0;
      for (uint64_t k = 0; k < cnt; ++k) {
        const uint32_t r = pairs[k].r;
        Work* ch = fcol[r] <= best_thr ? &L : &R;
        ch->w += (double)mult[r];
        ch->s += wy[r];
        ch->q += wy[r] * y[r];
      }
      /* children's rows for the next level, row order kept */
      for (uint64_t k = nw.b; k < nw.e; ++k) {
        goes_left[rows[k]] = fcol[rows[k]] <= best_thr;
        nl += goes_left[rows[k]];
      }
      L.b = fill; L.e = fill + nl;
      R.b = L.e; R.e = fill + cnt;
      uint64_t li = L.b, ri = R.b;
      for (uint64_t k = nw.b; k < nw.e; ++k) {
        const uint32_t r = rows[k];
        if (goes_left[r]) rows2[li++] = r; else rows2[ri++] = r;
      }
      fill += cnt;
      next[nn++] = L;
      next[nn++] = R;
    }
    Work* tw = front; front = next; next = tw;
    uint32_t* tr = rows; rows = rows2; rows2 = tr;
    nf = nn;
  }
  free(mult); free(wy); free(rows); free(rows2); free(front); free(next);
  free(pairs); free(pool); free(goes_left);
  return count;
}

static double walk(const int32_t* feature, const double* threshold, const int32_t* left,
                   const int32_t* right, const double* value, const double* x,
                   uint64_t stride) {
  int32_t i = 0;
  while (feature[i] >= 0)
    i = x[(uint64_t)feature[i] * stride] <= threshold[i] ? left[i] : right[i];
  return value[i];
}

/* OOB statistics; trees are concatenated SoA with offsets[t]..offsets[t+1].
 * out6 = {degenerate, mse, var, error_pct, r2, rows_evaluated}; per-row
 * sum/count (nullable).  Returns 0, or 3 when no row is out of bag. */
int oracle_oob(const double* col, const double* y, uint64_t n, uint32_t p, uint32_t T,
               const uint64_t* offsets, const int32_t* feature, const double* threshold,
               const int32_t* left, const int32_t* right, const double* value,
               const uint32_t* inbag, double* out6, double* row_sum,
               uint32_t* row_count) {
  (void)p;
  double mean = 0;
  for (uint64_t i = 0; i < n; ++i) mean += y[i];
  mean /= (double)n;
  double var = 0;
  int constant = 1;
  for (uint64_t i = 0; i < n; ++i) {
    var += (y[i] - mean) * (y[i] - mean);
    if (y[i] != y[0]) constant = 0;
  }
  var /= (double)n;
  memset(out6, 0, 6 * sizeof(double));
  out6[2] = var;
  if (constant) { out6[0] = 1; return 0; }
  double* sum = calloc(n, sizeof(double));
  uint32_t* cnt = calloc(n, sizeof(uint32_t));
  char* bag = malloc(n);
  for (uint32_t t = 0; t < T; ++t) {
    memset(bag, 0, n);
    for (uint64_t j = 0; j < n; ++j) bag[inbag[(uint64_t)t * n + j]] = 1;
    const uint64_t o = offsets[t];
    for (uint64_t i = 0; i < n; ++i) {
      if (bag[i]) continue;
      sum[i] += walk(feature + o, threshold + o, left + o, right + o, value + o, col + i, n);
      cnt[i]++;
    }
  }
  double mse = 0;
  uint64_t ev = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (!cnt[i]) continue;
    const double pred = sum[i] / (double)cnt[i];
    mse += (pred - y[i]) * (pred - y[i]);
    ev++;
  }
  if (row_sum) memcpy(row_sum, sum, n * sizeof(double));
  if (row_count) memcpy(row_count, cnt, n * sizeof(uint32_t));
  free(sum); free(cnt); free(bag);
  if (!ev) return 3;
  mse /= (double)ev;
  out6[1] = mse;
  out6[3] = 100.0 * mse / var;
  out6[4] = 1.0 - mse / var;
  out6[5] = (double)ev;
  return 0;
}

/* mean over trees (tree order) of the leaf reached; rows are row-major q x p */
void oracle_predict(const double* rows, uint64_t q, uint32_t p, uint32_t T,
                    const uint64_t* offsets, const int32_t* feature,
                    const double* threshold, const int32_t* left, const int32_t* right,
                    const double* value, double* out) {
  for (uint64_t i = 0; i < q; ++i) {
    double s = 0;
    for (uint32_t t = 0; t < T; ++t) {
      const uint64_t o = offsets[t];
      s += walk(feature + o, threshold + o, left + o, right + o, value + o,
                rows + i * p, 1);
    }
    out[i] = s / (double)T;
  }
}
