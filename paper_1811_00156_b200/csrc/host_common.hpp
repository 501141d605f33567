// Host-side shared pieces of libaiwc_cuda.so: status/exception plumbing behind the
// C-ABI (error taxonomy of error.hpp:8-54 mapped to int codes), splitmix64 seed
// helpers (rng.hpp:13-35) and the synthetic table type.
#pragma once

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "aiwc_cuda.h"

namespace aiwc_b200 {

constexpr uint64_t kGoldenGamma = 0x9e3779b97f4a7c15ull;

inline uint64_t host_mix64(uint64_t x) {
  x += kGoldenGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

inline uint64_t host_fnv1a64(const char* s, size_t len) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < len; ++i) {
    h ^= static_cast<unsigned char>(s[i]);
    h *= 0x100000001b3ull;
  }
  return h;
}

inline uint64_t host_derive_seed(uint64_t seed, const char* tag, uint64_t index) {
  return host_mix64(seed ^ host_fnv1a64(tag, std::strlen(tag)) ^ host_mix64(index));
}

// Thrown inside the library, converted to a status code at the C boundary.
struct Status {
  int code;
  std::string msg;
  Status(int c, std::string m) : code(c), msg(std::move(m)) {}
};

void set_last_error(const std::string& m);

template <typename F>
int guard(F&& f) {
  try {
    f();
    return AIWC_OK;
  } catch (const Status& s) {
    set_last_error(s.msg);
    return s.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return AIWC_EEXEC;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return AIWC_EEXEC;
  }
}

struct Table {
  uint64_t n = 0;
  uint32_t p = 0;
  uint32_t kernels = 0;
  uint64_t fingerprint = 0;
  std::vector<double> col;  // p*n column-major
  std::vector<double> y;
  std::vector<double> seconds;
  std::vector<uint32_t> kernel_of_row;
};

const std::vector<std::string>& feature_names();
Table synthesize_table(uint64_t kernels, uint64_t devices, double noise, uint64_t seed);

}  // namespace aiwc_b200
