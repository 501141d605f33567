// Drop-in replacement for the reference's proj/include/aiwc/forest.hpp, backed by the
// B200 kernels of libaiwc_cuda.so through the C-ABI in aiwc_cuda.h.
//
// Same namespace, types, fields and signatures as the reference:
//   ForestParams forest.hpp:22 | TreeNode :31 | Tree :39 | OobStats :57 | Forest :66
//   detail::FitContext :134 | compute_oob :393 | PreparedDataset :458
//   fit(PreparedDataset, ForestParams, jobs) :480 | fit(Dataset, ...) :511 | oob_error :518
//   Forest::to_json / from_json / save / load :527-604 (canonical JSON, byte-identical)
// so tuner.hpp, experiments.hpp and tools/main.cpp compile unchanged: put this
// directory BEFORE the reference's include directory.  The rest
// of the reference's headers (dataset.hpp, csv.hpp, error.hpp, parallel.hpp, rng.hpp)
// are used as they are.
//
// Differences a caller can observe:
//   * `jobs` is accepted and ignored (the forest grows on the GPU; results never
//     depended on it in the reference's intended semantics, forest.hpp:477-479).
//     Concurrent fits on one PreparedDataset (the heatmap / loko / tune threads) are
//     merged by the library into one multi-forest launch per batch, and successive
//     calls are spread round-robin over the visible GPUs (AIWC_DEVICES limits them);
//   * Tree::predict walks its one tree on the host (the reference's loop, exact);
//   * FitContext::order is left empty (the presort lives on the device);
//   * predictions run on the GPU: the Forest lazily uploads its trees and caches the
//     device copy (call invalidate_device_cache() after mutating `trees` by hand);
//   * there is no CPU fallback: without a usable sm_100 device every fit / predict
//     throws ExecutionError carrying the library's message.
#pragma once

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <string>
#include <vector>

#include <json.hpp>

#include "aiwc/csv.hpp"
#include "aiwc/dataset.hpp"
#include "aiwc/error.hpp"
#include "aiwc/parallel.hpp"
#include "aiwc/rng.hpp"
#include "aiwc_cuda.h"

namespace aiwc {

namespace b200 {
// C-ABI status -> the reference's exception taxonomy (error.hpp:8-54)
inline void check(int rc) {
  if (rc == AIWC_OK) return;
  const std::string msg = aiwc_last_error();
  switch (rc) {
    case AIWC_EPARSE: throw ParseError(msg);
    case AIWC_EIO: throw IoError(msg);
    case AIWC_ESCHEMA: throw SchemaError(msg);
    default: throw ExecutionError(msg);
  }
}
// devices used by the drop-in (AIWC_DEVICES=k: the first k; default all visible)
inline int device_count() {
  static const int n = [] {
    int c = 0;
    if (aiwc_device_count(&c) != AIWC_OK || c < 1) c = 1;
    if (const char* e = std::getenv("AIWC_DEVICES")) c = std::max(1, std::min(c, std::atoi(e)));
    return c;
  }();
  return n;
}
inline int device() { return 0; }
// round-robin device of the next fit
inline int next_device() {
  static std::atomic<unsigned> rr{0};
  return static_cast<int>(rr.fetch_add(1) % static_cast<unsigned>(device_count()));
}
}  // namespace b200

struct ForestParams {
  std::uint32_t num_trees = 500;
  std::uint32_t mtry = 1;
  std::uint32_t min_node_size = 1;
  std::uint64_t seed = 1;

  bool operator==(const ForestParams&) const = default;
};

struct TreeNode {
  std::int32_t feature = -1;  // -1 marks a leaf
  double threshold = 0;
  std::int32_t left = -1;
  std::int32_t right = -1;
  double value = 0;  // leaf mean
};

struct OobStats {
  bool degenerate = false;
  double mse = 0;
  double response_variance = 0;
  double error_pct = 0;
  double r_squared = 0;
  std::uint64_t rows_evaluated = 0;
};

namespace b200 {
// concatenated SoA of a tree list (the C-ABI's forest layout)
struct Soa {
  std::vector<std::uint64_t> off{0};
  std::vector<std::int32_t> f, l, r;
  std::vector<double> thr, val;
};
template <typename TreeList>
Soa to_soa(const TreeList& trees) {
  Soa s;
  for (const auto& t : trees) {
    for (const TreeNode& nd : t.nodes) {
      s.f.push_back(nd.feature);
      s.thr.push_back(nd.threshold);
      s.l.push_back(nd.left);
      s.r.push_back(nd.right);
      s.val.push_back(nd.value);
    }
    s.off.push_back(s.f.size());
  }
  return s;
}
struct ForestHandle {
  aiwc_forest* h = nullptr;
  explicit ForestHandle(aiwc_forest* x) : h(x) {}
  ~ForestHandle() { aiwc_forest_free(h); }
};
}  // namespace b200

struct Tree {
  std::vector<TreeNode> nodes;

  // One tree, one row (forest.hpp:42-50): a handful of node visits, walked here -- a
  // device round trip per call would cost more than the walk.  Batched callers use
  // Forest::predict_response / predict_responses (GPU).
  double predict(std::span<const double> row) const {
    std::int32_t node = 0;
    while (nodes[static_cast<std::size_t>(node)].feature >= 0) {
      const TreeNode& nd = nodes[static_cast<std::size_t>(node)];
      node = row[static_cast<std::size_t>(nd.feature)] <= nd.threshold ? nd.left : nd.right;
    }
    return nodes[static_cast<std::size_t>(node)].value;
  }
};

class Forest {
 public:
  ForestParams params;
  ResponseTransform response = ResponseTransform::Log10;
  std::vector<std::string> columns;  // predictor schema, fixed order
  std::uint64_t fingerprint = 0;
  std::vector<Tree> trees;
  std::vector<std::vector<std::uint32_t>> inbag;  // per tree, the n draws
  OobStats oob;

  // mean over trees (tree order) of the leaf value reached, in response space
  double predict_response(std::span<const double> row) const {
    double out = 0;
    b200::check(aiwc_predict(device_forest(), row.data(), 1,
                             static_cast<std::uint32_t>(row.size()), &out));
    return out;
  }

  // batched extension: q row-major rows of columns.size() predictors
  std::vector<double> predict_responses(std::span<const double> rows) const {
    const std::size_t p = columns.empty() ? 1 : columns.size();
    std::vector<double> out(rows.size() / p);
    b200::check(aiwc_predict(device_forest(), rows.data(), out.size(),
                             static_cast<std::uint32_t>(p), out.data()));
    return out;
  }

  double predict_time(std::span<const double> row) const {
    return from_response(response, predict_response(row));
  }

  void check_schema(const std::vector<std::string>& predictor_names,
                    ResponseTransform t) const {
    if (schema_fingerprint(predictor_names, t) != fingerprint)
      throw SchemaError("model schema fingerprint " + fingerprint_hex(fingerprint) +
                        " does not match input schema " +
                        fingerprint_hex(schema_fingerprint(predictor_names, t)));
  }

  std::vector<double> make_row(const FeatureVector& features, const std::string& device) const {
    std::vector<double> row(columns.size(), 0.0);
    const auto f = features.to_array();
    std::copy(f.begin(), f.end(), row.begin());
    const auto it = std::find(columns.begin() + static_cast<long>(kFeatureCount), columns.end(),
                              "device=" + device);
    if (it == columns.end()) throw SchemaError("device '" + device + "' is not part of the model");
    row[static_cast<std::size_t>(it - columns.begin())] = 1.0;
    return row;
  }

  std::vector<std::string> devices() const {
    std::vector<std::string> out;
    for (std::size_t i = kFeatureCount; i < columns.size(); ++i)
      out.push_back(columns[i].substr(7));  // strip "device="
    return out;
  }

  nlohmann::ordered_json to_json() const;
  static Forest from_json(const nlohmann::json& j);
  // model files (forest.hpp:596-604): the canonical bytes of to_json().dump() + "\n",
  // written / read directly (b200::json_write / json_read) without a JSON DOM
  void save(const std::string& path) const;
  static Forest load(const std::string& path);

  void invalidate_device_cache() const {
    std::lock_guard<std::mutex> lock(cache_->mu);
    cache_->dev.reset();
  }

 private:
  struct Cache {
    std::mutex mu;
    std::shared_ptr<b200::ForestHandle> dev;
    std::size_t trees = 0, nodes = 0;
  };
  std::shared_ptr<Cache> cache_ = std::make_shared<Cache>();

  aiwc_forest* device_forest() const {
    std::size_t nodes = 0;
    for (const Tree& t : trees) nodes += t.nodes.size();
    std::lock_guard<std::mutex> lock(cache_->mu);
    if (!cache_->dev || cache_->trees != trees.size() || cache_->nodes != nodes) {
      if (trees.empty()) throw ExecutionError("forest has no trees");
      const b200::Soa s = b200::to_soa(trees);
      aiwc_forest* h = nullptr;
      b200::check(aiwc_forest_import(static_cast<std::uint32_t>(trees.size()), s.off.data(),
                                     s.f.data(), s.thr.data(), s.l.data(), s.r.data(),
                                     s.val.data(), nullptr, 0, b200::device(), &h));
      cache_->dev = std::make_shared<b200::ForestHandle>(h);
      cache_->trees = trees.size();
      cache_->nodes = nodes;
    }
    return cache_->dev->h;
  }
};

namespace detail {

// Column store + responses (forest.hpp:134-161) plus the device-resident presort.
struct FitContext {
  std::size_t n = 0, p = 0;
  std::vector<std::vector<double>> col;           // p columns of n values
  std::vector<double> y;                          // response
  std::vector<std::vector<std::uint32_t>> order;  // left empty: the presort is on the GPU
  std::shared_ptr<aiwc_ctx> dev;                  // device 0's copy (created eagerly)

  FitContext(const Dataset& data, ResponseTransform t) {
    n = data.rows.size();
    p = data.predictor_count();
    col.assign(p, std::vector<double>(n));
    for (std::size_t c = 0; c < p; ++c)
      for (std::size_t i = 0; i < n; ++i) col[c][i] = data.predictor_value(i, c);
    y = data.responses(t);
    devs_ = std::make_shared<Devs>();
    devs_->ctx.resize(static_cast<std::size_t>(b200::device_count()));
    if (n >= 2) dev = on_device(0);
  }

  // the dataset's device copy on device d (uploaded and presorted on first use)
  std::shared_ptr<aiwc_ctx> on_device(int d) const {
    std::lock_guard<std::mutex> lock(devs_->mu);
    auto& c = devs_->ctx[static_cast<std::size_t>(d)];
    if (!c) {
      std::vector<double> flat(p * n);
      for (std::size_t k = 0; k < p; ++k) std::copy(col[k].begin(), col[k].end(), flat.begin() + k * n);
      aiwc_ctx* h = nullptr;
      b200::check(aiwc_ctx_create(flat.data(), y.data(), n, static_cast<std::uint32_t>(p), d, &h));
      c = std::shared_ptr<aiwc_ctx>(h, [](aiwc_ctx* x) { aiwc_ctx_free(x); });
    }
    return c;
  }

 private:
  struct Devs {
    std::mutex mu;
    std::vector<std::shared_ptr<aiwc_ctx>> ctx;
  };
  std::shared_ptr<Devs> devs_;
};

}  // namespace detail

// OOB statistics of a forest against the dataset it was trained on (forest.hpp:393):
// the forest's trees + in-bag lists go to the device, rows are walked there and the
// per-row sums are reduced in tree order, then finalised in row order.
inline OobStats compute_oob(const Forest& forest, const detail::FitContext& ctx) {
  if (!ctx.dev) throw ExecutionError("dataset must have at least 2 rows");
  const b200::Soa s = b200::to_soa(forest.trees);
  std::vector<std::uint32_t> inb;
  inb.reserve(forest.inbag.size() * ctx.n);
  for (const auto& v : forest.inbag) {
    if (v.size() != ctx.n) throw ExecutionError("in-bag list length differs from the dataset");
    inb.insert(inb.end(), v.begin(), v.end());
  }
  aiwc_forest* h = nullptr;
  b200::check(aiwc_forest_import(static_cast<std::uint32_t>(forest.trees.size()), s.off.data(),
                                 s.f.data(), s.thr.data(), s.l.data(), s.r.data(), s.val.data(),
                                 inb.data(), ctx.n, b200::device(), &h));
  b200::ForestHandle guard(h);
  aiwc_oob_stats st{};
  b200::check(aiwc_oob(ctx.dev.get(), h, &st, nullptr, nullptr));
  return OobStats{st.degenerate != 0, st.mse, st.response_variance, st.error_pct, st.r_squared,
                  st.rows_evaluated};
}

class PreparedDataset {
 public:
  PreparedDataset(const Dataset& data, ResponseTransform response)
      : ctx_(data, response), response_(response), columns_(data.predictor_names()) {}

  const detail::FitContext& context() const { return ctx_; }
  ResponseTransform response() const { return response_; }
  const std::vector<std::string>& columns() const { return columns_; }
  std::size_t rows() const { return ctx_.n; }
  std::size_t predictor_count() const { return ctx_.p; }

 private:
  detail::FitContext ctx_;
  ResponseTransform response_;
  std::vector<std::string> columns_;
};

// Fits a random-forest regressor on the GPU (forest.hpp:480).  Deterministic in
// params.seed; identical to the reference's intended (single-threaded) result.
inline Forest fit(const PreparedDataset& prepared, const ForestParams& params,
                  unsigned jobs = 1) {
  (void)jobs;
  if (prepared.rows() < 2) throw ExecutionError("dataset must have at least 2 rows");
  if (params.num_trees < 1) throw ExecutionError("num_trees must be >= 1");
  if (params.min_node_size < 1) throw ExecutionError("min_node_size must be >= 1");
  if (params.mtry < 1 || params.mtry > prepared.predictor_count())
    throw ExecutionError("mtry must be in [1, " + std::to_string(prepared.predictor_count()) +
                         "], got " + std::to_string(params.mtry));
  aiwc_forest* h = nullptr;
  const std::shared_ptr<aiwc_ctx> ctx = prepared.context().on_device(b200::next_device());
  b200::check(aiwc_fit(ctx.get(), params.num_trees, params.mtry, params.min_node_size,
                       params.seed, 0, params.num_trees, 1, &h));
  b200::ForestHandle guard(h);
  Forest forest;
  forest.params = params;
  forest.response = prepared.response();
  forest.columns = prepared.columns();
  forest.fingerprint = schema_fingerprint(forest.columns, forest.response);
  std::uint64_t total = 0;
  std::uint32_t T = 0, tb = 0;
  b200::check(aiwc_forest_info(h, &T, &total, &tb));
  std::vector<std::uint64_t> off(T + 1);
  std::vector<std::int32_t> f(total), l(total), r(total);
  std::vector<double> thr(total), val(total);
  b200::check(aiwc_forest_export(h, off.data(), f.data(), thr.data(), l.data(), r.data(),
                                 val.data()));
  forest.trees.resize(T);
  for (std::uint32_t t = 0; t < T; ++t) {
    auto& nodes = forest.trees[t].nodes;
    nodes.resize(off[t + 1] - off[t]);
    for (std::size_t i = 0; i < nodes.size(); ++i) {
      const std::size_t k = off[t] + i;
      nodes[i] = TreeNode{f[k], thr[k], l[k], r[k], val[k]};
    }
  }
  const std::size_t n = prepared.rows();
  std::vector<std::uint32_t> inb(static_cast<std::size_t>(T) * n);
  b200::check(aiwc_forest_export_inbag(h, inb.data()));
  forest.inbag.resize(T);
  for (std::uint32_t t = 0; t < T; ++t)
    forest.inbag[t].assign(inb.begin() + static_cast<long>(t * n),
                           inb.begin() + static_cast<long>((t + 1) * n));
  aiwc_oob_stats st{};
  b200::check(aiwc_forest_oob_stats(h, &st));
  forest.oob = OobStats{st.degenerate != 0, st.mse, st.response_variance, st.error_pct,
                        st.r_squared, st.rows_evaluated};
  return forest;
}

inline Forest fit(const Dataset& data, const ForestParams& params,
                  ResponseTransform response = ResponseTransform::Log10, unsigned jobs = 1) {
  return fit(PreparedDataset(data, response), params, jobs);
}

inline OobStats oob_error(const Forest& forest, const Dataset& data) {
  const detail::FitContext ctx(data, forest.response);
  forest.check_schema(data.predictor_names(), forest.response);
  return compute_oob(forest, ctx);
}

// ---- model file: canonical JSON (the reference's field order, so identical forests
// serialise to identical bytes) ----

inline nlohmann::ordered_json Forest::to_json() const {
  nlohmann::ordered_json j;
  j["format"] = "aiwc-forest";
  j["version"] = 1;
  j["response"] = response_name(response);
  j["columns"] = columns;
  j["schema_fingerprint"] = fingerprint_hex(fingerprint);
  nlohmann::ordered_json jp;
  jp["num_trees"] = params.num_trees;
  jp["mtry"] = params.mtry;
  jp["min_node_size"] = params.min_node_size;
  jp["seed"] = params.seed;
  j["params"] = std::move(jp);
  nlohmann::ordered_json jo;
  jo["degenerate"] = oob.degenerate;
  jo["mse"] = oob.mse;
  jo["response_variance"] = oob.response_variance;
  jo["error_pct"] = oob.error_pct;
  jo["r_squared"] = oob.r_squared;
  jo["rows_evaluated"] = oob.rows_evaluated;
  j["oob"] = std::move(jo);
  auto jt = nlohmann::ordered_json::array();
  for (const Tree& t : trees) {
    auto jn = nlohmann::ordered_json::array();
    for (const TreeNode& nd : t.nodes)
      jn.push_back(nlohmann::ordered_json::array(
          {nd.feature, nd.threshold, nd.left, nd.right, nd.value}));
    jt.push_back(std::move(jn));
  }
  j["trees"] = std::move(jt);
  j["inbag"] = inbag;
  return j;
}

inline Forest Forest::from_json(const nlohmann::json& j) {
  if (j.value("format", "") != "aiwc-forest" || j.value("version", 0) != 1)
    throw ParseError("model file: unknown format or version");
  Forest f;
  f.response = parse_response(j.at("response").get<std::string>());
  f.columns = j.at("columns").get<std::vector<std::string>>();
  f.fingerprint = schema_fingerprint(f.columns, f.response);
  if (j.at("schema_fingerprint").get<std::string>() != fingerprint_hex(f.fingerprint))
    throw ParseError("model file: schema fingerprint does not match columns");
  const auto& jp = j.at("params");
  f.params = ForestParams{jp.at("num_trees").get<std::uint32_t>(), jp.at("mtry").get<std::uint32_t>(),
                          jp.at("min_node_size").get<std::uint32_t>(),
                          jp.at("seed").get<std::uint64_t>()};
  const auto& jo = j.at("oob");
  f.oob = OobStats{jo.at("degenerate").get<bool>(), jo.at("mse").get<double>(),
                   jo.at("response_variance").get<double>(), jo.at("error_pct").get<double>(),
                   jo.at("r_squared").get<double>(), jo.at("rows_evaluated").get<std::uint64_t>()};
  for (const auto& jt : j.at("trees")) {
    Tree t;
    for (const auto& jn : jt)
      t.nodes.push_back(TreeNode{jn[0].get<std::int32_t>(), jn[1].get<double>(),
                                 jn[2].get<std::int32_t>(), jn[3].get<std::int32_t>(),
                                 jn[4].get<double>()});
    f.trees.push_back(std::move(t));
  }
  f.inbag = j.at("inbag").get<std::vector<std::vector<std::uint32_t>>>();
  if (f.trees.size() != f.params.num_trees || f.inbag.size() != f.trees.size())
    throw ParseError("model file: tree/inbag counts disagree with params");
  return f;
}

namespace b200 {

// The model file's bytes without building the JSON DOM: the same key order and compact
// separators as to_json().dump(), numbers through nlohmann's own shortest round-trip
// double printer (detail::to_chars, what dump() calls) and decimal integers, so the
// output is byte-identical (the C1 model's FNV-1a is pinned in tests/test_dropin.py).
inline void put_double(std::string& o, double x) {
  if (!std::isfinite(x)) {
    o += "null";
    return;
  }
  char buf[64];
  char* e = ::nlohmann::detail::to_chars(buf, buf + sizeof(buf), x);
  o.append(buf, static_cast<std::size_t>(e - buf));
}
template <typename I>
inline void put_int(std::string& o, I v) {
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  o.append(buf, static_cast<std::size_t>(r.ptr - buf));
}
inline void put_str(std::string& o, const std::string& s) { o += nlohmann::json(s).dump(); }

inline std::string json_write(const Forest& f) {
  std::size_t nodes = 0, draws = 0;
  for (const Tree& t : f.trees) nodes += t.nodes.size();
  for (const auto& v : f.inbag) draws += v.size();
  std::string o;
  o.reserve(nodes * 48 + draws * 8 + 4096);
  o += "{\"format\":\"aiwc-forest\",\"version\":1,\"response\":";
  put_str(o, response_name(f.response));
  o += ",\"columns\":[";
  for (std::size_t i = 0; i < f.columns.size(); ++i) {
    if (i) o += ',';
    put_str(o, f.columns[i]);
  }
  o += "],\"schema_fingerprint\":";
  put_str(o, fingerprint_hex(f.fingerprint));
  o += ",\"params\":{\"num_trees\":";
  put_int(o, f.params.num_trees);
  o += ",\"mtry\":";
  put_int(o, f.params.mtry);
  o += ",\"min_node_size\":";
  put_int(o, f.params.min_node_size);
  o += ",\"seed\":";
  put_int(o, f.params.seed);
  o += "},\"oob\":{\"degenerate\":";
  o += f.oob.degenerate ? "true" : "false";
  o += ",\"mse\":";
  put_double(o, f.oob.mse);
  o += ",\"response_variance\":";
  put_double(o, f.oob.response_variance);
  o += ",\"error_pct\":";
  put_double(o, f.oob.error_pct);
  o += ",\"r_squared\":";
  put_double(o, f.oob.r_squared);
  o += ",\"rows_evaluated\":";
  put_int(o, f.oob.rows_evaluated);
  o += "},\"trees\":[";
  for (std::size_t t = 0; t < f.trees.size(); ++t) {
    if (t) o += ',';
    o += '[';
    const auto& ns = f.trees[t].nodes;
    for (std::size_t i = 0; i < ns.size(); ++i) {
      if (i) o += ',';
      o += '[';
      put_int(o, ns[i].feature);
      o += ',';
      put_double(o, ns[i].threshold);
      o += ',';
      put_int(o, ns[i].left);
      o += ',';
      put_int(o, ns[i].right);
      o += ',';
      put_double(o, ns[i].value);
      o += ']';
    }
    o += ']';
  }
  o += "],\"inbag\":[";
  for (std::size_t t = 0; t < f.inbag.size(); ++t) {
    if (t) o += ',';
    o += '[';
    const auto& v = f.inbag[t];
    for (std::size_t i = 0; i < v.size(); ++i) {
      if (i) o += ',';
      put_int(o, v[i]);
    }
    o += ']';
  }
  o += "]}\n";
  return o;
}

// Reader of exactly that layout (the canonical file): false on any deviation, and the
// caller falls back to the general JSON parser.  Numbers are parsed with from_chars
// (correctly rounded, as the JSON parser's strtod).
struct JsonCursor {
  const char* p;
  const char* e;
  bool lit(const char* s) {
    const std::size_t n = std::strlen(s);
    if (static_cast<std::size_t>(e - p) < n || std::memcmp(p, s, n) != 0) return false;
    p += n;
    return true;
  }
  bool ch(char c) {
    if (p < e && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  template <typename I>
  bool integer(I& v) {
    const auto r = std::from_chars(p, e, v);
    if (r.ec != std::errc()) return false;
    p = r.ptr;
    return true;
  }
  bool number(double& v) {
    if (lit("null")) {
      v = std::numeric_limits<double>::quiet_NaN();
      return true;
    }
    const auto r = std::from_chars(p, e, v);
    if (r.ec != std::errc()) return false;
    p = r.ptr;
    return true;
  }
  bool string(std::string& s) {  // plain strings only (no escapes in canonical names)
    if (!ch('"')) return false;
    const char* q = p;
    while (q < e && *q != '"') {
      if (*q == '\\') return false;
      ++q;
    }
    if (q >= e) return false;
    s.assign(p, q);
    p = q + 1;
    return true;
  }
};

inline bool json_read(const std::string& text, Forest& f) {
  JsonCursor c{text.data(), text.data() + text.size()};
  std::string resp, fp;
  if (!c.lit("{\"format\":\"aiwc-forest\",\"version\":1,\"response\":") || !c.string(resp))
    return false;
  try {
    f.response = parse_response(resp);
  } catch (...) {
    return false;
  }
  if (!c.lit(",\"columns\":[")) return false;
  f.columns.clear();
  if (!c.ch(']')) {
    for (;;) {
      std::string col;
      if (!c.string(col)) return false;
      f.columns.push_back(std::move(col));
      if (c.ch(']')) break;
      if (!c.ch(',')) return false;
    }
  }
  if (!c.lit(",\"schema_fingerprint\":") || !c.string(fp)) return false;
  f.fingerprint = schema_fingerprint(f.columns, f.response);
  if (fp != fingerprint_hex(f.fingerprint)) throw ParseError("model file: schema fingerprint does not match columns");
  if (!c.lit(",\"params\":{\"num_trees\":") || !c.integer(f.params.num_trees) ||
      !c.lit(",\"mtry\":") || !c.integer(f.params.mtry) || !c.lit(",\"min_node_size\":") ||
      !c.integer(f.params.min_node_size) || !c.lit(",\"seed\":") || !c.integer(f.params.seed) ||
      !c.lit("},\"oob\":{\"degenerate\":"))
    return false;
  if (c.lit("true")) f.oob.degenerate = true;
  else if (c.lit("false")) f.oob.degenerate = false;
  else return false;
  if (!c.lit(",\"mse\":") || !c.number(f.oob.mse) || !c.lit(",\"response_variance\":") ||
      !c.number(f.oob.response_variance) || !c.lit(",\"error_pct\":") ||
      !c.number(f.oob.error_pct) || !c.lit(",\"r_squared\":") || !c.number(f.oob.r_squared) ||
      !c.lit(",\"rows_evaluated\":") || !c.integer(f.oob.rows_evaluated) ||
      !c.lit("},\"trees\":["))
    return false;
  f.trees.clear();
  if (!c.ch(']')) {
    for (;;) {
      Tree t;
      if (!c.ch('[')) return false;
      if (!c.ch(']')) {
        for (;;) {
          TreeNode nd;
          if (!c.ch('[') || !c.integer(nd.feature) || !c.ch(',') || !c.number(nd.threshold) ||
              !c.ch(',') || !c.integer(nd.left) || !c.ch(',') || !c.integer(nd.right) ||
              !c.ch(',') || !c.number(nd.value) || !c.ch(']'))
            return false;
          t.nodes.push_back(nd);
          if (c.ch(']')) break;
          if (!c.ch(',')) return false;
        }
      }
      f.trees.push_back(std::move(t));
      if (c.ch(']')) break;
      if (!c.ch(',')) return false;
    }
  }
  if (!c.lit(",\"inbag\":[")) return false;
  f.inbag.clear();
  if (!c.ch(']')) {
    for (;;) {
      std::vector<std::uint32_t> v;
      if (!c.ch('[')) return false;
      if (!c.ch(']')) {
        for (;;) {
          std::uint32_t x;
          if (!c.integer(x)) return false;
          v.push_back(x);
          if (c.ch(']')) break;
          if (!c.ch(',')) return false;
        }
      }
      f.inbag.push_back(std::move(v));
      if (c.ch(']')) break;
      if (!c.ch(',')) return false;
    }
  }
  if (!c.ch('}')) return false;
  while (c.p < c.e && (*c.p == '\n' || *c.p == ' ' || *c.p == '\r' || *c.p == '\t')) ++c.p;
  if (c.p != c.e) return false;
  if (f.trees.size() != f.params.num_trees || f.inbag.size() != f.trees.size())
    throw ParseError("model file: tree/inbag counts disagree with params");
  return true;
}

}  // namespace b200

inline void Forest::save(const std::string& path) const { write_text_file(path, b200::json_write(*this)); }

inline Forest Forest::load(const std::string& path) {
  const std::string text = read_text_file(path);
  {
    Forest f;
    if (b200::json_read(text, f)) return f;  // the canonical layout, parsed directly
  }
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw ParseError("model file: " + std::string(e.what()));
  }
  return from_json(j);
}

}  // namespace aiwc
