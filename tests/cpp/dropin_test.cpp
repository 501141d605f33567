// Drop-in check: the reference's UNMODIFIED experiments.hpp / tuner.hpp / synth.hpp
// compiled against include/aiwc/forest.hpp (this repo) instead of the reference's
// forest.hpp, linked to libaiwc_cuda.so.  Built by oracle/Makefile (target `dropin`,
// needs /root/reference) into oracle/_ref/dropin_test; tests/test_dropin.py runs it on
// the GPU box and compares its JSON line with the reference goldens.
#include <aiwc/experiments.hpp>
#include <aiwc/synth.hpp>
#include <aiwc/tuner.hpp>

#include <chrono>
#include <cstdio>
#include <string>

using namespace aiwc;

// heatmap mode: the reference's heatmap_scan (experiments.hpp:79-123) with 12 SA chains on
// 12 threads, every objective a drop-in fit (concurrent fits on one PreparedDataset: the
// library batches them); configuration = tests/golden/make_heatmap_golden.py
static int heatmap() {
  const SynthResult s = synthesize(SynthConfig{});
  const Dataset d = make_dataset(s.features, s.runtimes);
  const PreparedDataset prep(d, ResponseTransform::Log10);
  HeatmapConfig cfg;
  cfg.space.num_trees = {10, 300};
  cfg.space.mtry = {1, 34};
  cfg.fixed_min_node_size = 9;
  cfg.schedule.max_evaluations = 30;
  cfg.random_starts = 8;
  cfg.forest_seed = derive_seed(1, "forest");
  cfg.sa_seed = 1;
  cfg.jobs = 12;
  (void)fit(prep, ForestParams{10, 6, 9, cfg.forest_seed});  // warm: contexts, pools
  const auto t0 = std::chrono::steady_clock::now();
  const HeatmapResult r = heatmap_scan(prep, cfg);
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::size_t ev = 0;
  for (const auto& c : r.chains) ev += c.entries.size();
  std::printf("{\"seconds\": %.6f, \"evaluations\": %zu, \"cells\": [", sec, ev);
  for (std::size_t i = 0; i < r.cells.size(); ++i)
    std::printf("%s[%lld, %lld, %.17g]", i ? ", " : "", static_cast<long long>(r.cells[i].num_trees),
                static_cast<long long>(r.cells[i].mtry), r.cells[i].error_pct);
  std::printf("]}\n");
  return 0;
}

// json mode: the model file path (forest.hpp:527-604) -- the reference's DOM route
// (to_json().dump() / json::parse + from_json) against the drop-in's direct
// writer / reader (b200::json_write / Forest::load), same bytes, timed
static int json_mode() {
  using clk = std::chrono::steady_clock;
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const SynthResult s = synthesize(SynthConfig{});
  const Dataset d = make_dataset(s.features, s.runtimes);
  const Forest f = fit(d, ForestParams{500, 6, 5, derive_seed(1, "forest")});
  auto t0 = clk::now();
  const std::string dom = f.to_json().dump() + "\n";
  auto t1 = clk::now();
  const std::string fast = b200::json_write(f);
  auto t2 = clk::now();
  const std::string path = "/tmp/aiwc_dropin_model.json";
  write_text_file(path, fast);
  auto t3 = clk::now();
  const Forest g = Forest::from_json(nlohmann::json::parse(read_text_file(path)));
  auto t4 = clk::now();
  const Forest h = Forest::load(path);
  auto t5 = clk::now();
  const bool same = dom == fast && g.to_json().dump() + "\n" == fast && b200::json_write(h) == fast;
  const std::string body = fast.substr(0, fast.size() - 1);  // the JSON text (no newline)
  std::printf("{\"bytes\": %zu, \"fnv\": %llu, \"identical\": %s, \"dom_write_ms\": %.3f, "
              "\"fast_write_ms\": %.3f, \"dom_read_ms\": %.3f, \"fast_read_ms\": %.3f}\n",
              body.size(), static_cast<unsigned long long>(fnv1a64(body)), same ? "true" : "false",
              ms(t0, t1), ms(t1, t2), ms(t3, t4), ms(t4, t5));
  return same ? 0 : 4;
}

// jsonfile mode (no GPU): a model file written by the reference -> Forest::load (direct
// reader) -> b200::json_write must give the file's bytes back; DOM route timed alongside
static int jsonfile_mode(const std::string& path) {
  using clk = std::chrono::steady_clock;
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const std::string text = read_text_file(path);
  auto t0 = clk::now();
  const Forest g = Forest::from_json(nlohmann::json::parse(text));
  auto t1 = clk::now();
  const Forest h = Forest::load(path);
  auto t2 = clk::now();
  const std::string dom = g.to_json().dump() + "\n";
  auto t3 = clk::now();
  const std::string fast = b200::json_write(h);
  auto t4 = clk::now();
  const bool same = dom == text && fast == text;
  std::printf("{\"bytes\": %zu, \"fnv\": %llu, \"identical\": %s, \"dom_read_ms\": %.3f, "
              "\"fast_read_ms\": %.3f, \"dom_write_ms\": %.3f, \"fast_write_ms\": %.3f}\n",
              text.size(), static_cast<unsigned long long>(fnv1a64(text)), same ? "true" : "false",
              ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
  return same ? 0 : 4;
}

int main(int argc, char** argv) {
  if (argc > 2 && std::string(argv[1]) == "jsonfile") {
    try {
      return jsonfile_mode(argv[2]);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "dropin_test jsonfile: %s\n", e.what());
      return 3;
    }
  }
  if (argc > 1 && std::string(argv[1]) == "json") {
    try {
      return json_mode();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "dropin_test json: %s\n", e.what());
      return 3;
    }
  }
  if (argc > 1 && std::string(argv[1]) == "heatmap") {
    try {
      return heatmap();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "dropin_test heatmap: %s\n", e.what());
      return 3;
    }
  }
  try {
    const SynthResult s = synthesize(SynthConfig{});
    const Dataset d = make_dataset(s.features, s.runtimes);
    const std::uint64_t seed = derive_seed(1, "forest");
    // forest.hpp:511 entry point
    const Forest f = fit(d, ForestParams{500, 6, 5, seed});
    const std::string js = f.to_json().dump();
    // tuner.hpp:247-253 objective path: PreparedDataset + fit(prepared, params, jobs)
    const PreparedDataset prep(d, ResponseTransform::Log10);
    const double obj = fit(prep, ParamsPoint{505, 30, 9}.to_forest_params(seed), 8).oob.error_pct;
    // experiments.hpp:383 evaluate (the reference's loop over folds, our fit/predict)
    const EvaluateResult ev = evaluate(d, ForestParams{50, 6, 5, 0}, seed);
    double mape = 0;
    for (std::size_t i = 0; i < d.rows.size(); ++i)
      mape += 100.0 * std::abs(ev.predicted_time_s[i] - d.rows[i].measured_time_s) /
              d.rows[i].measured_time_s;
    mape /= static_cast<double>(d.rows.size());
    // model round trip through the canonical JSON (forest.hpp:524-604)
    const Forest g = Forest::from_json(nlohmann::json::parse(js));
    const bool same = g.to_json().dump() == js &&
                      g.predict_time(d.predictor_row(7)) == f.predict_time(d.predictor_row(7));
    // oob_error recomputes OOB from trees + in-bag lists (forest.hpp:518)
    const OobStats o2 = oob_error(f, d);
    std::printf(
        "{\"json_fnv\": %llu, \"json_size\": %zu, \"oob_error_pct\": %.17g, \"r2\": %.17g, "
        "\"oob_recomputed\": %.17g, \"obj_505_30_9\": %.17g, \"c3_50_mape\": %.17g, "
        "\"pairs\": %llu, \"pairs_correct\": %llu, \"roundtrip\": %s}\n",
        static_cast<unsigned long long>(fnv1a64(js)), js.size(), f.oob.error_pct,
        f.oob.r_squared, o2.error_pct, obj, mape,
        static_cast<unsigned long long>(ev.rank.pairs),
        static_cast<unsigned long long>(ev.rank.pairs_correct), same ? "true" : "false");
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "dropin_test: %s\n", e.what());
    return 3;
  }
}
