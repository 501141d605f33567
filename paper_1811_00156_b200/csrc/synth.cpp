// Host-side synthetic AIWC table generator (the bench's input generator).
//
// Restates the reference's synthetic data path so that the GPU forest sees exactly
// the tables the reference fits (bit-identical doubles, identical canonical row
// order):
//   stream keys   derive_seed(seed, "device"|"kernel"|"ks"|"noise", i)   synth.hpp:135,145,170,246
//   latent model  g(f) and time_for()                                     synth.hpp:87-104
//   feature recipe per (kernel, size)                                     synth.hpp:150-239
//   quant9 (9-significant-digit round trip through "%.9g")                synth.hpp:117, csv.hpp:17
//   join + canonical sort (kernel, size, device, application)             dataset.hpp:101-115, 280-318
//   predictors = 27 features ++ one-hot(sorted devices)                   dataset.hpp:117-138
//   response  = log10(seconds)                                            dataset.hpp:85-87
// Host C++ only (this is input generation: "reused as-is on the host").
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "aiwc_cuda.h"
#include "host_common.hpp"

namespace aiwc_b200 {

namespace {

constexpr int kFeat = 27;

double q9(double x) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.9g", x);
  return std::strtod(buf, nullptr);
}

std::string two(uint64_t v) {
  std::string s = std::to_string(v);
  return s.size() < 2 ? "0" + s : s;
}

// splitmix64 stream with the reference's uniform/bounded/normal helpers (rng.hpp:41-74)
struct Stream {
  uint64_t s;
  explicit Stream(uint64_t key) : s(key) {}
  uint64_t next() { return host_mix64(s += kGoldenGamma); }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double in(double lo, double hi) { return lo + unit() * (hi - lo); }
  uint64_t below(uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * n) >> 64);
  }
  int64_t between(int64_t lo, int64_t hi) {
    return lo + static_cast<int64_t>(below(static_cast<uint64_t>(hi - lo + 1)));
  }
  double gauss() {
    double a = unit();
    const double b = unit();
    while (a <= 0.0) a = unit();
    return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * 3.14159265358979323846 * b);
  }
};

// feature slots (features.hpp:27-45 order)
enum : int {
  F_OPDIV = 0, F_INSTR, F_WI, F_BARRIERS, F_MIN_ITB, F_MAX_ITB, F_MED_ITB, F_SIMD_MAX,
  F_SIMD_MEAN, F_SIMD_SD, F_FOOT, F_FOOT90, F_GMAE, F_LMAE0, F_TUBI = 23, F_BR90,
  F_YOKOTA, F_AVGLIN
};

struct KernelTraits {
  double base_instr, mem_frac, uniq_frac, locality, lmae_slope, simd_max, yokota_base,
      wi_base;
  int64_t opdiv, phases, branch_sites;
};

KernelTraits draw_traits(uint64_t seed, uint64_t k) {
  static const double kSimd[5] = {1, 2, 4, 8, 16};
  Stream r(host_derive_seed(seed, "kernel", k));
  KernelTraits t{};
  t.base_instr = std::pow(10.0, r.in(std::log10(3e3), std::log10(3e5)));
  t.opdiv = r.between(2, 8);
  t.mem_frac = r.in(0.05, 0.35);
  t.uniq_frac = r.in(0.02, 0.8);
  t.locality = r.in(0.45, 0.98);
  t.lmae_slope = r.in(0.04, 0.10);
  t.phases = r.unit() < 0.45 ? 0 : r.between(1, 6);
  t.simd_max = kSimd[r.below(5)];
  const bool branchy = r.unit() >= 0.2;
  t.branch_sites = branchy ? r.between(2, 40) : 0;
  t.yokota_base = r.in(0.05, 0.95);
  t.wi_base = std::pow(2.0, static_cast<double>(r.between(6, 10)));
  return t;
}

std::array<double, kFeat> make_features(const KernelTraits& t, uint64_t seed, uint64_t k,
                                        uint64_t size_idx) {
  Stream r(host_derive_seed(seed, "ks", k * 8 + size_idx));
  std::array<double, kFeat> f{};
  const double im = std::pow(8.0, static_cast<double>(size_idx));
  const double wm = std::pow(4.0, static_cast<double>(size_idx));
  f[F_INSTR] = std::round(t.base_instr * im * std::pow(10.0, r.in(-0.05, 0.05)));
  f[F_WI] = std::min(std::round(t.wi_base * wm), f[F_INSTR]);
  f[F_OPDIV] = static_cast<double>(t.opdiv);
  const double per_item = f[F_INSTR] / f[F_WI];
  if (t.phases == 0) {
    f[F_BARRIERS] = 0;
    f[F_MIN_ITB] = f[F_MAX_ITB] = f[F_MED_ITB] = std::round(per_item);
  } else {
    f[F_BARRIERS] = f[F_WI] * static_cast<double>(t.phases);
    const double med = per_item / static_cast<double>(t.phases + 1);
    f[F_MED_ITB] = std::round(med * 2.0) / 2.0;
    f[F_MIN_ITB] = std::min(std::floor(med * r.in(0.5, 0.95)), f[F_MED_ITB]);
    f[F_MAX_ITB] = std::max(std::ceil(med * r.in(1.05, 2.0)), f[F_MED_ITB]);
  }
  f[F_SIMD_MAX] = t.simd_max;
  if (t.simd_max <= 1.0) {
    f[F_SIMD_MEAN] = 1.0;
    f[F_SIMD_SD] = 0.0;
  } else {
    f[F_SIMD_MEAN] = q9(r.in(1.0 + 0.3 * (t.simd_max - 1.0), t.simd_max));
    const double cap = std::sqrt((t.simd_max - f[F_SIMD_MEAN]) * (f[F_SIMD_MEAN] - 1.0));
    f[F_SIMD_SD] = q9(r.in(0.0, cap));
  }
  const double accesses = f[F_INSTR] * t.mem_frac;
  f[F_FOOT] = std::max(1.0, std::round(accesses * t.uniq_frac));
  f[F_FOOT90] = std::max(1.0, std::round(f[F_FOOT] * r.in(0.2, 0.9)));
  f[F_GMAE] = q9(t.locality * std::log2(std::max(f[F_FOOT], 1.0)));
  if (f[F_FOOT] <= 1.0) f[F_GMAE] = 0.0;
  for (int l = 0; l < 10; ++l)
    f[F_LMAE0 + l] =
        q9(f[F_GMAE] * std::max(0.0, 1.0 - t.lmae_slope * static_cast<double>(l + 1)));
  if (t.branch_sites != 0) {
    f[F_TUBI] = static_cast<double>(t.branch_sites);
    f[F_BR90] = std::max(
        1.0, std::round(static_cast<double>(t.branch_sites) * r.in(0.3, 0.95)));
    const double yok = std::clamp(t.yokota_base + r.in(-0.05, 0.05), 0.0, 1.0);
    f[F_YOKOTA] = q9(yok);
    f[F_AVGLIN] = q9(yok * r.in(0.55, 0.95));
  }
  return f;
}

struct Device {
  std::string name;
  double factor, branch_aff, simd_aff;
};

double latent_g(const std::array<double, kFeat>& f) {
  return std::pow(f[F_INSTR] / 4e6, 0.72) * (1.0 + 0.22 * f[F_GMAE]) *
         (1.0 + 0.9 * f[F_AVGLIN]) * std::pow(std::max(f[F_SIMD_MEAN], 1.0), -0.45) *
         (1.0 + 0.15 * std::log10(1.0 + f[F_FOOT]));
}

struct Row {
  uint32_t kernel_num;  // generation index
  uint32_t size;
  uint32_t device;  // generation index
  double seconds;
};

}  // namespace

const std::vector<std::string>& feature_names() {
  static const std::vector<std::string> names = [] {
    std::vector<std::string> n = {"opcode_diversity_90", "total_instruction_count",
                                  "work_items", "total_barriers_hit", "min_itb",
                                  "max_itb", "median_itb", "max_simd_width",
                                  "mean_simd_width", "sd_simd_width",
                                  "total_memory_footprint", "ninety_memory_footprint",
                                  "global_memory_address_entropy"};
    for (int i = 1; i <= 10; ++i)
      n.push_back("local_memory_address_entropy_" + std::to_string(i));
    n.insert(n.end(), {"total_unique_branch_instructions", "ninety_branch_instructions",
                       "yokota_branch_entropy", "average_linear_branch_entropy"});
    return n;
  }();
  return names;
}

Table synthesize_table(uint64_t K, uint64_t D, double noise, uint64_t seed) {
  if (K < 1 || D < 1) throw Status(AIWC_EEXEC, "synth config counts must be >= 1");
  if (noise < 0) throw Status(AIWC_EEXEC, "synth noise must be >= 0");
  static const double kSizeBase[4] = {2.0e-3, 2.4e-3, 2.9e-3, 3.5e-3};
  std::vector<Device> dev(D);
  for (uint64_t d = 0; d < D; ++d) {
    Stream r(host_derive_seed(seed, "device", d));
    dev[d].name = "dev" + two(d);
    dev[d].factor =
        q9(std::pow(10.0, -0.9 + 0.13 * static_cast<double>(d) + r.in(-0.015, 0.015)));
    dev[d].branch_aff = q9(r.in(-0.25, 0.25));
    dev[d].simd_aff = q9(r.in(-0.18, 0.18));
  }
  std::vector<std::array<double, kFeat>> feats(K * 4);
  std::vector<Row> rows;
  rows.reserve(K * 4 * D);
  for (uint64_t k = 0; k < K; ++k) {
    const KernelTraits t = draw_traits(seed, k);
    for (uint64_t s = 0; s < 4; ++s) {
      auto& f = feats[k * 4 + s];
      f = make_features(t, seed, k, s);
      const double g = latent_g(f);
      for (uint64_t d = 0; d < D; ++d) {
        Stream r(host_derive_seed(seed, "noise", (k * 4 + s) * D + d));
        const double z = noise > 0 ? r.gauss() : 0.0;
        const double inter = 1.0 + dev[d].branch_aff * f[F_AVGLIN] +
                             dev[d].simd_aff * (f[F_SIMD_MEAN] / 16.0);
        const double secs = q9(kSizeBase[s] * dev[d].factor * g * inter *
                               std::pow(10.0, noise * z));
        if (!(secs > 0)) throw Status(AIWC_EPARSE, "measured time must be positive");
        rows.push_back({static_cast<uint32_t>(k), static_cast<uint32_t>(s),
                        static_cast<uint32_t>(d), secs});
      }
    }
  }
  // canonical order: (kernel name, size, device name, application) -- names compare
  // as std::string (so "kern10" < "kern100" < "kern11")
  std::vector<std::string> kname(K), app(K);
  for (uint64_t k = 0; k < K; ++k) {
    kname[k] = "kern" + two(k);
    app[k] = "app" + two(k % 11);
  }
  std::vector<uint32_t> dev_rank(D), ker_rank(K);
  {
    std::vector<uint32_t> idx(D);
    for (uint32_t i = 0; i < D; ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(),
              [&](uint32_t a, uint32_t b) { return dev[a].name < dev[b].name; });
    for (uint32_t i = 0; i < D; ++i) dev_rank[idx[i]] = i;
    std::vector<uint32_t> kid(K);
    for (uint32_t i = 0; i < K; ++i) kid[i] = i;
    std::sort(kid.begin(), kid.end(),
              [&](uint32_t a, uint32_t b) { return kname[a] < kname[b]; });
    for (uint32_t i = 0; i < K; ++i) ker_rank[kid[i]] = i;
  }
  std::sort(rows.begin(), rows.end(), [&](const Row& a, const Row& b) {
    if (a.kernel_num != b.kernel_num) return ker_rank[a.kernel_num] < ker_rank[b.kernel_num];
    if (a.size != b.size) return a.size < b.size;
    return dev_rank[a.device] < dev_rank[b.device];
  });
  Table tb;
  tb.n = rows.size();
  tb.p = static_cast<uint32_t>(kFeat + D);
  tb.kernels = static_cast<uint32_t>(K);
  tb.col.assign(static_cast<size_t>(tb.p) * tb.n, 0.0);
  tb.y.resize(tb.n);
  tb.seconds.resize(tb.n);
  tb.kernel_of_row.resize(tb.n);
  for (uint64_t i = 0; i < tb.n; ++i) {
    const Row& r = rows[i];
    const auto& f = feats[r.kernel_num * 4 + r.size];
    for (int c = 0; c < kFeat; ++c) tb.col[static_cast<size_t>(c) * tb.n + i] = f[c];
    tb.col[static_cast<size_t>(kFeat + dev_rank[r.device]) * tb.n + i] = 1.0;
    tb.seconds[i] = r.seconds;
    tb.y[i] = std::log10(r.seconds);
    tb.kernel_of_row[i] = ker_rank[r.kernel_num];
  }
  // schema fingerprint (dataset.hpp:180-190): names joined by '|' + "response:log10"
  std::string blob;
  for (const auto& nm : feature_names()) blob += nm + "|";
  std::vector<std::string> dnames;
  for (const auto& d : dev) dnames.push_back(d.name);
  std::sort(dnames.begin(), dnames.end());
  for (const auto& d : dnames) blob += "device=" + d + "|";
  blob += "response:log10";
  tb.fingerprint = host_fnv1a64(blob.data(), blob.size());
  return tb;
}

}  // namespace aiwc_b200

using namespace aiwc_b200;

struct aiwc_table {
  Table t;
};

extern "C" {

int aiwc_synth(uint64_t kernel_count, uint64_t device_count, double noise, uint64_t seed,
               aiwc_table** out) {
  return guard([&] {
    if (!out) throw Status(AIWC_EARG, "out is NULL");
    *out = new aiwc_table{synthesize_table(kernel_count, device_count, noise, seed)};
  });
}

int aiwc_table_free(aiwc_table* t) {
  delete t;
  return AIWC_OK;
}

int aiwc_table_info(const aiwc_table* t, uint64_t* n, uint32_t* p, uint32_t* kernels,
                    uint64_t* fingerprint) {
  return guard([&] {
    if (!t) throw Status(AIWC_EARG, "table is NULL");
    if (n) *n = t->t.n;
    if (p) *p = t->t.p;
    if (kernels) *kernels = t->t.kernels;
    if (fingerprint) *fingerprint = t->t.fingerprint;
  });
}

int aiwc_table_export(const aiwc_table* t, double* col, double* y, double* seconds,
                      uint32_t* kernel_of_row) {
  return guard([&] {
    if (!t) throw Status(AIWC_EARG, "table is NULL");
    const Table& b = t->t;
    if (col) std::memcpy(col, b.col.data(), b.col.size() * sizeof(double));
    if (y) std::memcpy(y, b.y.data(), b.n * sizeof(double));
    if (seconds) std::memcpy(seconds, b.seconds.data(), b.n * sizeof(double));
    if (kernel_of_row)
      std::memcpy(kernel_of_row, b.kernel_of_row.data(), b.n * sizeof(uint32_t));
  });
}

}  // extern "C"
