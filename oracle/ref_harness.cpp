// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference headers (/root/reference/proj/include/aiwc),
// compiled by oracle/Makefile into oracle/_ref/libaiwc_ref.so.  It is the parity
// checker (tests/, __graft_entry__.smoke()) and the CPU arm of bench.py
// (`--impl reference`, cpu_baseline.kind = "reference").  Nothing in this file
// re-implements the forest: every entry point calls the reference's own code:
//   synthesize            synth.hpp:126      make_dataset       dataset.hpp:280
//   PreparedDataset       forest.hpp:458     fit                forest.hpp:480
//   TreeGrower::grow      forest.hpp:179     compute_oob        forest.hpp:393
//   Forest::predict_response forest.hpp:77   evaluate           experiments.hpp:383
//   Forest::to_json       forest.hpp:527     derive_seed/Rng    rng.hpp:32/41
// The raw-array entry (ref_fit_raw) builds a detail::FitContext from a 2-row
// dummy Dataset and then overwrites its public fields, so arbitrary (col, y)
// tables (step datasets, edge cases) run through the reference grower too.
#include <aiwc/experiments.hpp>
#include <aiwc/forest.hpp>
#include <aiwc/synth.hpp>

#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

using namespace aiwc;

#ifdef AIWC_REF_QUARANTINE
// Golden-generation build only (oracle/_ref/libaiwc_ref_q.so, linked -Bsymbolic so these
// bind for the reference code inside this library alone): freed blocks are held in a
// FIFO quarantine (like AddressSanitizer's) before they go back to malloc, so the
// reference's dangling read of node.left/right after tree.nodes reallocates
// (forest.hpp:245, 312-318 -- REFERENCE_DEFECT.md) always sees the values it just wrote,
// i.e. the reference's intended semantics, whatever the heap state.
#include <malloc.h>
#include <cstdlib>
#include <mutex>
#include <new>
namespace {
struct Quarantine {  // a malloc'd ring of pending frees (no allocation through delete)
  std::mutex mu;
  void** ring = nullptr;
  std::size_t cap = 0, head = 0, len = 0, bytes = 0;
  static constexpr std::size_t kBudget = std::size_t{1} << 29;  // 512 MB
  void put(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(mu);
    if (len == cap) {  // grow the ring (malloc / free only)
      const std::size_t nc = cap ? 2 * cap : 1024;
      void** nr = static_cast<void**>(std::malloc(nc * sizeof(void*)));
      for (std::size_t i = 0; i < len; ++i) nr[i] = ring[(head + i) % cap];
      std::free(ring);
      ring = nr;
      cap = nc;
      head = 0;
    }
    ring[(head + len) % cap] = p;
    ++len;
    bytes += malloc_usable_size(p);
    while (bytes > kBudget && len) {
      void* o = ring[head];
      head = (head + 1) % cap;
      --len;
      bytes -= malloc_usable_size(o);
      std::free(o);
    }
  }
};
Quarantine& quarantine() {
  static Quarantine* z = new Quarantine;
  return *z;
}
}  // namespace
void* operator new(std::size_t n) {
  if (void* p = std::malloc(n ? n : 1)) return p;
  throw std::bad_alloc();
}
void* operator new[](std::size_t n) { return ::operator new(n); }
void operator delete(void* p) noexcept { quarantine().put(p); }
void operator delete[](void* p) noexcept { quarantine().put(p); }
void operator delete(void* p, std::size_t) noexcept { quarantine().put(p); }
void operator delete[](void* p, std::size_t) noexcept { quarantine().put(p); }
#endif

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 2;
  } catch (const SchemaError& e) {
    g_err = e.what();
    return 5;
  } catch (const IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const ExecutionError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct RefForest {
  Forest forest;
};

struct RefData {
  Dataset data;
};

// FitContext over raw arrays: the reference constructor needs a Dataset, so
// build it from a throwaway 2-row dataset and replace every public field with
// the same recipe the constructor uses (forest.hpp:140-160).
detail::FitContext raw_context(const double* col, const double* y, std::size_t n,
                               std::size_t p) {
  Dataset d;
  DataRow r;
  r.kernel = "k";
  r.device = "d";
  r.measured_time_s = 1.0;
  d.rows = {r, r};
  d.devices = {"d"};
  detail::FitContext ctx(d, ResponseTransform::Raw);
  ctx.n = n;
  ctx.p = p;
  ctx.col.assign(p, std::vector<double>(n));
  for (std::size_t c = 0; c < p; ++c)
    for (std::size_t i = 0; i < n; ++i) ctx.col[c][i] = col[c * n + i];
  ctx.y.assign(y, y + n);
  ctx.order.assign(p, {});
  for (std::size_t c = 0; c < p; ++c) {
    auto& ord = ctx.order[c];
    ord.resize(n);
    for (std::size_t i = 0; i < n; ++i) ord[i] = static_cast<std::uint32_t>(i);
    const auto& v = ctx.col[c];
    std::sort(ord.begin(), ord.end(), [&](std::uint32_t a, std::uint32_t b) {
      if (v[a] != v[b]) return v[a] < v[b];
      return a < b;
    });
  }
  return ctx;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix64(uint64_t x) { return mix64(x); }
uint64_t ref_fnv1a64(const char* s, uint64_t len) {
  return fnv1a64(std::string_view(s, len));
}
uint64_t ref_derive_seed(uint64_t seed, const char* tag, uint64_t index) {
  return derive_seed(seed, tag, index);
}
// first `count` bounded(n) draws of Rng(key)
void ref_rng_bounded(uint64_t key, uint64_t n, uint64_t count, uint64_t* out) {
  Rng r(key);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.bounded(n);
}

// ---- datasets ----
int ref_synth(uint64_t kernel_count, uint64_t device_count, double noise,
              uint64_t seed, void** out) {
  return guarded([&] {
    SynthConfig cfg;
    cfg.kernel_count = kernel_count;
    cfg.device_count = device_count;
    cfg.noise = noise;
    cfg.seed = seed;
    SynthResult s = synthesize(cfg);
    auto* d = new RefData{make_dataset(s.features, s.runtimes)};
    *out = d;
  });
}
void ref_data_free(void* h) { delete static_cast<RefData*>(h); }
uint64_t ref_data_rows(void* h) { return static_cast<RefData*>(h)->data.rows.size(); }
uint64_t ref_data_cols(void* h) { return static_cast<RefData*>(h)->data.predictor_count(); }
// column-major predictors (p*n), log10 responses, measured seconds, kernel index
void ref_data_export(void* h, double* col, double* y, double* seconds,
                     uint32_t* kernel_idx) {
  const Dataset& d = static_cast<RefData*>(h)->data;
  const std::size_t n = d.rows.size(), p = d.predictor_count();
  if (col)
    for (std::size_t c = 0; c < p; ++c)
      for (std::size_t i = 0; i < n; ++i) col[c * n + i] = d.predictor_value(i, c);
  if (y) {
    const auto r = d.responses(ResponseTransform::Log10);
    std::memcpy(y, r.data(), n * sizeof(double));
  }
  if (seconds)
    for (std::size_t i = 0; i < n; ++i) seconds[i] = d.rows[i].measured_time_s;
  if (kernel_idx) {
    const auto ks = d.kernels();
    for (std::size_t i = 0; i < n; ++i)
      kernel_idx[i] = static_cast<uint32_t>(
          std::lower_bound(ks.begin(), ks.end(), d.rows[i].kernel) - ks.begin());
  }
}
uint64_t ref_data_fingerprint(void* h) {
  const Dataset& d = static_cast<RefData*>(h)->data;
  return schema_fingerprint(d.predictor_names(), ResponseTransform::Log10);
}
// '\n'-joined predictor names into buf (returns needed length)
uint64_t ref_data_names(void* h, char* buf, uint64_t cap) {
  const Dataset& d = static_cast<RefData*>(h)->data;
  std::string s;
  for (const auto& nm : d.predictor_names()) s += nm + "\n";
  if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  return s.size();
}

// ---- prepared dataset + fit through the public API ----
void* ref_prepare(void* h) {
  return new PreparedDataset(static_cast<RefData*>(h)->data, ResponseTransform::Log10);
}
void ref_prepared_free(void* p) { delete static_cast<PreparedDataset*>(p); }

int ref_fit_prepared(void* prep, uint32_t num_trees, uint32_t mtry, uint32_t mns,
                     uint64_t seed, unsigned jobs, void** out) {
  return guarded([&] {
    auto* f = new RefForest{fit(*static_cast<PreparedDataset*>(prep),
                                ForestParams{num_trees, mtry, mns, seed}, jobs)};
    *out = f;
  });
}

// grow trees [t0, t1) only (no OOB) -- the bounded CPU sample for big configs
int ref_grow_range(void* prep, uint32_t num_trees, uint32_t mtry, uint32_t mns,
                   uint64_t seed, uint32_t t0, uint32_t t1, unsigned jobs,
                   uint64_t* total_nodes) {
  return guarded([&] {
    const auto& ctx = static_cast<PreparedDataset*>(prep)->context();
    ForestParams params{num_trees, mtry, mns, seed};
    std::vector<std::uint64_t> nodes(t1 - t0, 0);
    parallel_for_with_state(
        t1 - t0, jobs, [&] { return detail::TreeGrower(ctx, params); },
        [&](detail::TreeGrower& g, std::size_t i) {
          std::vector<std::uint32_t> draws;
          nodes[i] = g.grow(t0 + i, draws).nodes.size();
        });
    uint64_t s = 0;
    for (auto v : nodes) s += v;
    if (total_nodes) *total_nodes = s;
  });
}

// The reference's fit body (forest.hpp:492-508) over the tree range [t0, t1) of a
// num_trees forest: TreeGrower::grow for each tree via parallel_for_with_state with
// `jobs` threads, then compute_oob over those trees -- the bounded CPU sample of a big
// fit that includes OOB (bench.py's reference arm: distinct trees per step).
int ref_fit_range(void* prep, uint32_t num_trees, uint32_t mtry, uint32_t mns, uint64_t seed,
                  uint32_t t0, uint32_t t1, unsigned jobs, double* out6) {
  return guarded([&] {
    const auto& ctx = static_cast<PreparedDataset*>(prep)->context();
    ForestParams params{num_trees, mtry, mns, seed};
    Forest f;
    f.params = params;
    f.trees.resize(t1 - t0);
    f.inbag.resize(t1 - t0);
    parallel_for_with_state(
        t1 - t0, jobs, [&] { return detail::TreeGrower(ctx, params); },
        [&](detail::TreeGrower& g, std::size_t i) {
          f.trees[i] = g.grow(t0 + i, f.inbag[i]);
        });
    const OobStats o = compute_oob(f, ctx);
    if (out6) {
      out6[0] = o.degenerate ? 1.0 : 0.0;
      out6[1] = o.mse;
      out6[2] = o.response_variance;
      out6[3] = o.error_pct;
      out6[4] = o.r_squared;
      out6[5] = static_cast<double>(o.rows_evaluated);
    }
  });
}

// Grow tree t alone (single thread, the intended semantics -- REFERENCE_DEFECT.md) and
// walk its out-of-bag rows exactly as compute_oob does (forest.hpp:418-433): oob[i] =
// the leaf value tree t gives row i, NaN for in-bag rows.  Node arrays go to the caller
// when `cap` holds them (returns the node count in *nodes either way).  Used to pin the
// 1000-tree C4 forest, one process per tree range (tests/golden/make_c4_forest.py).
int ref_grow_tree_oob(void* prep, uint32_t num_trees, uint32_t mtry, uint32_t mns,
                      uint64_t seed, uint32_t t, double* oob, uint64_t cap, uint64_t* nodes,
                      int32_t* feature, double* threshold, int32_t* left, int32_t* right,
                      double* value, uint32_t* inbag_out) {
  return guarded([&] {
    const auto& ctx = static_cast<PreparedDataset*>(prep)->context();
    detail::TreeGrower g(ctx, ForestParams{num_trees, mtry, mns, seed});
    std::vector<std::uint32_t> draws;
    const Tree tree = g.grow(t, draws);
    const std::size_t n = ctx.n;
    std::vector<char> inbag(n, 0);
    for (std::uint32_t r : draws) inbag[r] = 1;
    for (std::size_t i = 0; i < n; ++i) {
      if (inbag[i]) {
        oob[i] = std::numeric_limits<double>::quiet_NaN();
        continue;
      }
      std::int32_t node = 0;
      while (tree.nodes[static_cast<std::size_t>(node)].feature >= 0) {
        const TreeNode& nd = tree.nodes[static_cast<std::size_t>(node)];
        node = ctx.col[static_cast<std::size_t>(nd.feature)][i] <= nd.threshold ? nd.left
                                                                                 : nd.right;
      }
      oob[i] = tree.nodes[static_cast<std::size_t>(node)].value;
    }
    *nodes = tree.nodes.size();
    if (cap >= tree.nodes.size())
      for (std::size_t i = 0; i < tree.nodes.size(); ++i) {
        feature[i] = tree.nodes[i].feature;
        threshold[i] = tree.nodes[i].threshold;
        left[i] = tree.nodes[i].left;
        right[i] = tree.nodes[i].right;
        value[i] = tree.nodes[i].value;
      }
    if (inbag_out) std::memcpy(inbag_out, draws.data(), draws.size() * sizeof(std::uint32_t));
  });
}

// reference fit over a raw column-major table (TreeGrower + compute_oob, exactly
// the body of fit(), forest.hpp:492-508)
int ref_fit_raw(const double* col, const double* y, uint64_t n, uint32_t p,
                uint32_t num_trees, uint32_t mtry, uint32_t mns, uint64_t seed,
                unsigned jobs, void** out) {
  return guarded([&] {
    if (n < 2) throw ExecutionError("dataset must have at least 2 rows");
    if (num_trees < 1) throw ExecutionError("num_trees must be >= 1");
    if (mns < 1) throw ExecutionError("min_node_size must be >= 1");
    if (mtry < 1 || mtry > p) throw ExecutionError("mtry out of range");
    const detail::FitContext ctx = raw_context(col, y, n, p);
    ForestParams params{num_trees, mtry, mns, seed};
    auto* f = new RefForest;
    f->forest.params = params;
    f->forest.trees.resize(num_trees);
    f->forest.inbag.resize(num_trees);
    parallel_for_with_state(
        num_trees, jobs, [&] { return detail::TreeGrower(ctx, params); },
        [&](detail::TreeGrower& g, std::size_t t) {
          f->forest.trees[t] = g.grow(t, f->forest.inbag[t]);
        });
    f->forest.oob = compute_oob(f->forest, ctx);
    *out = f;
  });
}

void ref_forest_free(void* f) { delete static_cast<RefForest*>(f); }
uint32_t ref_forest_trees(void* f) {
  return static_cast<uint32_t>(static_cast<RefForest*>(f)->forest.trees.size());
}
uint64_t ref_forest_nodes(void* f, uint32_t t) {
  return static_cast<RefForest*>(f)->forest.trees[t].nodes.size();
}
void ref_forest_tree(void* f, uint32_t t, int32_t* feature, double* threshold,
                     int32_t* left, int32_t* right, double* value) {
  const auto& nodes = static_cast<RefForest*>(f)->forest.trees[t].nodes;
  for (std::size_t i = 0; i < nodes.size(); ++i) {
    feature[i] = nodes[i].feature;
    threshold[i] = nodes[i].threshold;
    left[i] = nodes[i].left;
    right[i] = nodes[i].right;
    value[i] = nodes[i].value;
  }
}
void ref_forest_inbag(void* f, uint32_t t, uint32_t* out) {
  const auto& v = static_cast<RefForest*>(f)->forest.inbag[t];
  std::memcpy(out, v.data(), v.size() * sizeof(uint32_t));
}
// degenerate, mse, var, error_pct, r2, rows
void ref_forest_oob(void* f, double* out6) {
  const OobStats& o = static_cast<RefForest*>(f)->forest.oob;
  out6[0] = o.degenerate ? 1.0 : 0.0;
  out6[1] = o.mse;
  out6[2] = o.response_variance;
  out6[3] = o.error_pct;
  out6[4] = o.r_squared;
  out6[5] = static_cast<double>(o.rows_evaluated);
}
// canonical model bytes as Forest::save writes them: size + FNV-1a64
uint64_t ref_forest_json_fnv(void* f, uint64_t* size) {
  const std::string s = static_cast<RefForest*>(f)->forest.to_json().dump() + "\n";
  if (size) *size = s.size();
  return fnv1a64(s);
}
uint64_t ref_forest_json(void* f, char* buf, uint64_t cap) {
  const std::string s = static_cast<RefForest*>(f)->forest.to_json().dump() + "\n";
  if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  return s.size();
}

// Forest::predict_response over q row-major rows, parallel_for over 4096-row chunks
void ref_predict(void* f, const double* rows, uint64_t q, uint32_t p, unsigned jobs,
                 double* out) {
  const Forest& forest = static_cast<RefForest*>(f)->forest;
  const std::size_t chunks = (q + 4095) / 4096;
  parallel_for(chunks, jobs, [&](std::size_t c) {
    const std::size_t b = c * 4096, e = std::min<std::size_t>(q, b + 4096);
    for (std::size_t i = b; i < e; ++i)
      out[i] = forest.predict_response(std::span<const double>(rows + i * p, p));
  });
}

// hold-one-kernel-out evaluate (experiments.hpp:383): predicted seconds per row
// and the rank report's pair counts
int ref_evaluate(void* h, uint32_t num_trees, uint32_t mtry, uint32_t mns,
                 uint64_t seed, unsigned jobs, double* predicted, uint64_t* pairs,
                 uint64_t* pairs_correct) {
  return guarded([&] {
    const Dataset& d = static_cast<RefData*>(h)->data;
    const EvaluateResult r =
        evaluate(d, ForestParams{num_trees, mtry, mns, 0}, seed,
                 ResponseTransform::Log10, jobs);
    std::memcpy(predicted, r.predicted_time_s.data(),
                r.predicted_time_s.size() * sizeof(double));
    *pairs = r.rank.pairs;
    *pairs_correct = r.rank.pairs_correct;
  });
}

// heatmap_scan (experiments.hpp:79-123): the SA chains from the 4 corners + random
// starts, every objective a reference fit (tuner.hpp:247-253).  Cells (num_trees, mtry,
// mean error_pct) go to out (3 doubles each); *nevals = total objective evaluations.
int ref_heatmap(void* prep, int64_t nt_lo, int64_t nt_hi, int64_t mt_lo, int64_t mt_hi,
                int64_t mns, uint64_t max_evals, uint64_t random_starts, uint64_t forest_seed,
                uint64_t sa_seed, unsigned jobs, double* out, uint64_t cap, uint64_t* ncells,
                uint64_t* nevals) {
  return guarded([&] {
    HeatmapConfig cfg;
    cfg.space.num_trees = {nt_lo, nt_hi};
    cfg.space.mtry = {mt_lo, mt_hi};
    cfg.fixed_min_node_size = mns;
    cfg.schedule.max_evaluations = max_evals;
    cfg.random_starts = random_starts;
    cfg.forest_seed = forest_seed;
    cfg.sa_seed = sa_seed;
    cfg.jobs = jobs;
    const HeatmapResult r = heatmap_scan(*static_cast<PreparedDataset*>(prep), cfg);
    *ncells = r.cells.size();
    uint64_t ev = 0;
    for (const auto& c : r.chains) ev += c.entries.size();
    *nevals = ev;
    for (std::size_t i = 0; i < r.cells.size() && 3 * i + 2 < cap; ++i) {
      out[3 * i] = static_cast<double>(r.cells[i].num_trees);
      out[3 * i + 1] = static_cast<double>(r.cells[i].mtry);
      out[3 * i + 2] = r.cells[i].error_pct;
    }
  });
}

}  // extern "C"
