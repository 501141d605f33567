// C-ABI entry points of libaiwc_cuda.so (declared in include/aiwc_cuda.h).
//
// Host driver around the sm_100a kernels: PreparedDataset upload (presort + ranks),
// fit (grow_kernel launch over persistent per-tree CTAs, pool compaction, OOB),
// forest export/import, OOB, predict and hold-one-kernel-out evaluate.
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <cuda_runtime.h>
#include <sys/mman.h>

#include "aiwc_cuda.h"
#include "forest_kernels.cuh"
#include "grow.cuh"
#include "host_common.hpp"

namespace aiwc_b200 {

namespace {
thread_local std::string g_last_error;
}
std::atomic<uint64_t> g_launches{0};  // kernels launched by this library (bench evidence)

void set_last_error(const std::string& m) { g_last_error = m; }

#define CK(expr)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw Status(AIWC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Idle large device blocks per device, kept for the next fit.  Every C4 fit allocates
// ~45 GB of per-fit buffers (in-bag draws, OOB leaves, node pool, compacted forest);
// taken from and returned to the stream-ordered pool they fragmented it, and a later
// fit's allocation could stall 0.1-1.3 s while the pool mapped fresh memory
// (profiles/r2_bench_v3_phases.txt: 0.1-1.3 s compaction allocs before).  Blocks of at least kCacheMin bytes are recycled here
// instead: a request takes the smallest idle block of 1x-1.125x its size.
constexpr size_t kCacheMin = size_t{1} << 30;  // C4-scale buffers; small fits use the pool
struct BlockCache {
  std::mutex mu;
  std::vector<std::pair<char*, size_t>> idle;
  size_t bytes = 0;
};
inline BlockCache& block_cache(int dev) {
  static BlockCache c[64];
  return c[dev & 63];
}
inline size_t cache_idle_bytes(int dev) {
  BlockCache& c = block_cache(dev);
  std::lock_guard<std::mutex> g(c.mu);
  return c.bytes;
}
inline void cache_flush(int dev) {
  BlockCache& c = block_cache(dev);
  std::lock_guard<std::mutex> g(c.mu);
  for (auto& b : c.idle) cudaFreeAsync(b.first, 0);
  c.idle.clear();
  c.bytes = 0;
}
inline char* cache_take(int dev, size_t need, size_t* got) {
  {
    BlockCache& c = block_cache(dev);
    std::lock_guard<std::mutex> g(c.mu);
    size_t best = SIZE_MAX;
    for (size_t i = 0; i < c.idle.size(); ++i)
      if (c.idle[i].second >= need && c.idle[i].second <= need + need / 8 &&
          (best == SIZE_MAX || c.idle[i].second < c.idle[best].second))
        best = i;
    if (best != SIZE_MAX) {
      char* q = c.idle[best].first;
      *got = c.idle[best].second;
      c.bytes -= *got;
      c.idle.erase(c.idle.begin() + static_cast<long>(best));
      return q;
    }
  }
  char* q = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&q), need, 0) != cudaSuccess) {
    cudaGetLastError();
    cache_flush(dev);  // idle blocks back to the pool, then once more
    if (cudaMallocAsync(reinterpret_cast<void**>(&q), need, 0) != cudaSuccess) {
      cudaGetLastError();
      throw Status(AIWC_ECUDA, "out of device memory (" + std::to_string(need >> 20) + " MB)");
    }
  }
  *got = need;
  return q;
}
inline void cache_give(int dev, char* q, size_t bytes) {
  BlockCache& c = block_cache(dev);
  std::lock_guard<std::mutex> g(c.mu);
  c.idle.emplace_back(q, bytes);
  c.bytes += bytes;
  // at most 16 idle blocks (a C4 fit cycles 11: in-bag, OOB leaves, 5 node-pool
  // arrays, 4 forest arrays): the oldest go back to the pool
  while (c.idle.size() > 16) {
    cudaFreeAsync(c.idle.front().first, 0);
    c.bytes -= c.idle.front().second;
    c.idle.erase(c.idle.begin());
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  bool owned = true;  // false: a view into memory another object owns (never freed here)
  int cache_dev = -1;  // >= 0: a recycled block of block_cache(cache_dev), blk_bytes long
  size_t blk_bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t c) { alloc(c); }
  void view(T* q, size_t c) {
    release();
    p = q;
    count = c;
    owned = false;
  }
  // stream-ordered allocation from the device's default pool (kept warm, see
  // warm_pool): fits in tuning loops allocate/free without device-wide syncs.  Every
  // API call synchronises its stream before returning, so a buffer is idle when freed.
  void alloc(size_t c) {
    release();
    if (c) CK(cudaMallocAsync(reinterpret_cast<void**>(&p), c * sizeof(T), 0));
    count = c;
  }
  // large per-fit buffers: recycled through the device's block cache
  void alloc_cached(size_t c, int dev) {
    release();
    count = c;
    if (!c) return;
    if (c * sizeof(T) < kCacheMin) {
      CK(cudaMallocAsync(reinterpret_cast<void**>(&p), c * sizeof(T), 0));
      return;
    }
    p = reinterpret_cast<T*>(cache_take(dev, c * sizeof(T), &blk_bytes));
    cache_dev = dev;
  }
  void release() {
    if (p && owned) {
      if (cache_dev >= 0)
        cache_give(cache_dev, reinterpret_cast<char*>(p), blk_bytes);
      else
        cudaFreeAsync(p, 0);
    }
    p = nullptr;
    count = 0;
    owned = true;
    cache_dev = -1;
    blk_bytes = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept
      : p(o.p), count(o.count), owned(o.owned), cache_dev(o.cache_dev), blk_bytes(o.blk_bytes) {
    o.p = nullptr;
    o.count = 0;
    o.owned = true;
    o.cache_dev = -1;
    o.blk_bytes = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p;
    count = o.count;
    owned = o.owned;
    cache_dev = o.cache_dev;
    blk_bytes = o.blk_bytes;
    o.p = nullptr;
    o.count = 0;
    o.owned = true;
    o.cache_dev = -1;
    o.blk_bytes = 0;
    return *this;
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw Status(AIWC_ECUDA, "no CUDA device available (libaiwc_cuda has no CPU fallback)");
    if (dev < 0 || dev >= count)
      throw Status(AIWC_EARG, "device index " + std::to_string(dev) + " out of range");
    cudaGetDevice(&prev);
    CK(cudaSetDevice(dev));
    warm_pool(dev);
  }
  // keep freed pool memory cached instead of returning it to the driver
  static void warm_pool(int dev) {
    static std::once_flag flags[64];
    if (dev < 0 || dev >= 64) return;
    std::call_once(flags[dev], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    });
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s) cudaStreamDestroy(s);
  }
};

// 64 pinned uint32 flags, recycled through a process-wide free list
struct PinnedFlags {
  uint32_t* p = nullptr;
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<uint32_t*>& pool() {
    static std::vector<uint32_t*> v;
    return v;
  }
  PinnedFlags() {
    {
      std::lock_guard<std::mutex> g(mu());
      if (!pool().empty()) {
        p = pool().back();
        pool().pop_back();
        return;
      }
    }
    CK(cudaMallocHost(reinterpret_cast<void**>(&p), 64 * 4));
  }
  ~PinnedFlags() {
    std::lock_guard<std::mutex> g(mu());
    pool().push_back(p);
  }
  uint32_t* get() const { return p; }
};

// pinned host buffers recycled process-wide (cudaMallocHost pins pages: milliseconds)
struct PinnedPool {
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<std::pair<char*, size_t>>& free_list() {
    static std::vector<std::pair<char*, size_t>> v;
    return v;
  }
  static std::pair<char*, size_t> take(size_t bytes) {
    {
      std::lock_guard<std::mutex> g(mu());
      auto& v = free_list();
      size_t best = SIZE_MAX;  // best fit: a small request must not take a forest mirror
      for (size_t i = 0; i < v.size(); ++i)
        if (v[i].second >= bytes && (best == SIZE_MAX || v[i].second < v[best].second))
          best = i;
      if (best != SIZE_MAX) {
        auto r = v[best];
        v.erase(v.begin() + static_cast<long>(best));
        return r;
      }
    }
    char* p = nullptr;
    // small buffers get headroom for reuse; large ones (forest mirrors) are sized to fit
    const size_t cap = bytes >= (size_t{1} << 30)
                           ? (bytes + (size_t{2} << 20) - 1) & ~((size_t{2} << 20) - 1)
                           : std::max<size_t>(bytes + bytes / 2, size_t{1} << 20);
    CK(cudaMallocHost(reinterpret_cast<void**>(&p), cap));
    return {p, cap};
  }
  static void give(std::pair<char*, size_t> b) {
    if (!b.first) return;
    std::lock_guard<std::mutex> g(mu());
    auto& v = free_list();
    v.push_back(b);
    // at most 48 GB of idle pinned host memory (forest mirrors are ~14 GB at C4): the
    // oldest blocks are unpinned first
    size_t idle = 0;
    for (auto& x : v) idle += x.second;
    while (idle > (size_t{48} << 30) && v.size() > 1) {
      idle -= v.front().second;
      cudaFreeHost(v.front().first);
      v.erase(v.begin());
    }
  }
  static void release_all() {
    std::lock_guard<std::mutex> g(mu());
    for (auto& x : free_list()) cudaFreeHost(x.first);
    free_list().clear();
  }
};

// host threads for the pinned <-> pageable copies (AIWC_COPY_THREADS, default 16)
unsigned copy_threads() {
  static const unsigned n = [] {
    unsigned v = 16;
    if (const char* e = std::getenv("AIWC_COPY_THREADS")) v = static_cast<unsigned>(std::atoi(e));
    return std::max(1u, std::min(v, std::max(1u, std::thread::hardware_concurrency())));
  }();
  return n;
}

// Persistent host copy workers (the pinned <-> pageable copies): a job is split into
// parts run by the workers and the calling thread; one job at a time.  Round 1 started
// 16 fresh threads per 64 MB chunk (2,500 thread starts per 10 GB export).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool(copy_threads() - 1);  // never destroyed (exit-safe)
    return *p;
  }
  // f(i) for i < n, spread over the workers and the caller; returns when all are done
  void run(unsigned n, const std::function<void(unsigned)>& f) {
    std::lock_guard<std::mutex> job_lock(job_mu_);
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      parts_ = n;
      next_ = 0;
      pending_ = n;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  explicit CopyPool(unsigned workers) {
    for (unsigned i = 0; i < workers; ++i)
      th_.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          {
            std::unique_lock<std::mutex> g(mu_);
            cv_.wait(g, [&] { return gen_ != seen; });
            seen = gen_;
          }
          work();
        }
      });
    for (auto& t : th_) t.detach();
  }
  void work() {
    for (;;) {
      unsigned i;
      const std::function<void(unsigned)>* f;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (!job_ || next_ >= parts_) return;
        i = next_++;
        f = job_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> th_;
  const std::function<void(unsigned)>* job_ = nullptr;
  unsigned parts_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
};

// memcpy of `len` bytes split over the copy pool
void par_memcpy(char* d, const char* p, size_t len) {
  const unsigned nt = copy_threads();
  if (nt <= 1 || len < (size_t{1} << 20)) {
    std::memcpy(d, p, len);
    return;
  }
  const size_t part = ((len + nt - 1) / nt + 63) & ~size_t{63};
  CopyPool::get().run(nt, [=](unsigned t) {
    const size_t b = size_t{t} * part;
    if (b < len) std::memcpy(d + b, p + b, std::min(part, len - b));
  });
}

// Device -> pageable host copy through two pinned bounce buffers (allocated once per
// process): the DMA of chunk i+1 overlaps the multi-threaded host copy of chunk i, so
// large exports (10 GB of C4 nodes) run at PCIe speed instead of the driver's pageable
// path.  Small copies go straight through cudaMemcpy.
void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  constexpr size_t kChunk = size_t{64} << 20;
  constexpr int kBufs = 4;  // DMA runs up to three chunks ahead of the host copies
  if (bytes < (size_t{8} << 20)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return;
  }
  // AIWC_HUGE=1: ask for transparent huge pages on the destination ("madvise" mode, 512x
  // fewer faults on a fresh buffer).  Off by default: measured no faster on a clean host,
  // and with THP defrag "madvise" a fragmented host memory turns the faults into direct
  // compaction stalls
  static const bool huge = std::getenv("AIWC_HUGE") != nullptr;
  if (huge) {
    constexpr uintptr_t kHuge = uintptr_t{2} << 20;
    const uintptr_t b = (reinterpret_cast<uintptr_t>(dst) + kHuge - 1) & ~(kHuge - 1);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(dst) + bytes) & ~(kHuge - 1);
    if (e > b) madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);  // a hint only
  }
  static std::mutex mu;
  static char* pin[kBufs] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (!pin[0])
    for (int k = 0; k < kBufs; ++k) CK(cudaMallocHost(reinterpret_cast<void**>(&pin[k]), kChunk));
  cudaEvent_t ev[kBufs];
  for (int k = 0; k < kBufs; ++k) CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
  struct EvG {
    cudaEvent_t* e;
    ~EvG() {
      for (int k = 0; k < kBufs; ++k) cudaEventDestroy(e[k]);
    }
  } eg{ev};
  const size_t nchunk = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t i) {
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    CK(cudaMemcpyAsync(pin[i % kBufs], static_cast<const char*>(src) + off, len,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ev[i % kBufs], s));
  };
  for (size_t i = 0; i + 1 < kBufs && i < nchunk; ++i) issue(i);
  for (size_t i = 0; i < nchunk; ++i) {
    // buffer (i + kBufs - 1) % kBufs was drained in iteration i - 1
    if (i + kBufs - 1 < nchunk) issue(i + kBufs - 1);
    CK(cudaEventSynchronize(ev[i % kBufs]));
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    par_memcpy(static_cast<char*>(dst) + off, pin[i % kBufs], len);
  }
}

// Pageable host -> device copy through two pinned bounce buffers: the multi-threaded
// host copy into one buffer overlaps the DMA out of the other.  Returns when the data
// is on the device (the stream is synchronised).
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  constexpr size_t kChunk = size_t{64} << 20;
  if (bytes < (size_t{8} << 20)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    return;
  }
  static std::mutex mu;
  static char* pin[2] = {nullptr, nullptr};
  std::lock_guard<std::mutex> lock(mu);
  if (!pin[0]) {
    CK(cudaMallocHost(reinterpret_cast<void**>(&pin[0]), kChunk));
    CK(cudaMallocHost(reinterpret_cast<void**>(&pin[1]), kChunk));
  }
  cudaEvent_t ev[2];
  CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  struct EvG {
    cudaEvent_t* e;
    ~EvG() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } eg{ev};
  const size_t nchunk = (bytes + kChunk - 1) / kChunk;
  for (size_t i = 0; i < nchunk; ++i) {
    if (i >= 2) CK(cudaEventSynchronize(ev[i & 1]));  // DMA out of this buffer finished
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    par_memcpy(pin[i & 1], static_cast<const char*>(src) + off, len);
    CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, pin[i & 1], len, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(ev[i & 1], s));
  }
  CK(cudaStreamSynchronize(s));
}

}  // namespace aiwc_b200

using namespace aiwc_b200;

// ---------------------------------------------------------------------------------
// Slot arena: one per device, holds the wide grower's tree slots between fits; released
// when the device's last dataset context is freed.
// ---------------------------------------------------------------------------------
namespace aiwc_b200 {
struct SlotArena {
  std::mutex mu;
  DevBuf<char> buf;
  bool busy = false;
  int ctxs = 0;
};
SlotArena& slot_arena(int dev) {
  static SlotArena arenas[64];
  return arenas[dev & 63];
}
size_t slot_arena_size(int dev) {
  SlotArena& a = slot_arena(dev);
  std::lock_guard<std::mutex> g(a.mu);
  return a.busy ? 0 : a.buf.count;
}
// exclusive use of the device's arena for one fit (grown to `bytes` if needed), or a
// temporary block when another fit holds it
struct SlotLease {
  SlotArena* ar = nullptr;
  DevBuf<char> own;
  char* p = nullptr;
  SlotLease(int dev, size_t bytes, bool exact = false) {
    SlotArena& a = slot_arena(dev);
    {
      std::lock_guard<std::mutex> g(a.mu);
      if (!a.busy) {
        a.busy = true;
        ar = &a;
      }
    }
    if (ar) {
      try {
        if (ar->buf.count < bytes || (exact && ar->buf.count > bytes)) {
          ar->buf.release();
          ar->buf.alloc(bytes);
        }
      } catch (...) {
        std::lock_guard<std::mutex> g(ar->mu);
        ar->busy = false;
        throw;
      }
      p = ar->buf.p;
    } else {
      own.alloc(bytes);
      p = own.p;
    }
  }
  ~SlotLease() {
    if (ar) {
      std::lock_guard<std::mutex> g(ar->mu);
      ar->busy = false;
    }
  }
};
}  // namespace aiwc_b200

// ---------------------------------------------------------------------------------
// PreparedDataset on the device
// ---------------------------------------------------------------------------------
struct aiwc_ctx {
  uint64_t uid = 0;  // process-unique id (a forest's cached OOB leaves name their dataset)
  int device = 0;
  uint64_t n = 0;
  uint32_t p = 0;
  uint32_t rank_bytes = 2;
  std::vector<double> y;  // host copy (OOB finalize runs the reference's row-order sums)
  uint32_t nlisted = 0, order_stride = 0;
  DevBuf<double> col, dy, vals;
  DevBuf<uint32_t> order, listed;
  DevBuf<int32_t> list_of;
  DevBuf<uint8_t> rank;
  DevBuf<uint64_t> vals_off;
  // Concurrent aiwc_fit calls on this dataset (the reference's heatmap / loko / tune
  // threads, experiments.hpp:104-110, 175-181) queue here; one caller at a time leads and
  // grows every queued request's trees in ONE launch sequence (fit_batch).
  struct FitRequest;
  struct FitQueue {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<FitRequest*> pending;
    bool leader = false;
    size_t returning = 0;  // callers of the last batch that have not queued again yet
  } q;
  // fits also stream their in-bag draws into a pinned host mirror while later batches
  // grow (aiwc_ctx_set_host_mirror): the forest's host view then only moves its nodes
  bool host_mirror = false;
  // grow scratch + launch stream, reused across fits on this dataset (serialised by `mu`)
  std::mutex mu;
  cudaStream_t stream = nullptr;
  ~aiwc_ctx() {
    if (stream) cudaStreamDestroy(stream);
  }

  DevData view() const {
    return DevData{n, p, rank_bytes, nlisted, order_stride, col.p, dy.p, order.p, rank.p,
                   vals.p, vals_off.p, list_of.p, listed.p};
  }
};

struct aiwc_ctx::FitRequest {
  uint32_t num_trees, mtry, mns, tb, te;
  uint64_t seed;
  int compute_oob;
  aiwc_forest* out = nullptr;
  int status = AIWC_OK;
  std::string msg;
  bool done = false;
};

// ---------------------------------------------------------------------------------
// Forest
// ---------------------------------------------------------------------------------
struct aiwc_forest {
  int device = 0;
  uint32_t cells = 1;  // forests held (aiwc_fit_cells): trees of forest c are [c*T, (c+1)*T)
  uint64_t n = 0;  // training rows (inbag / oob arrays)
  uint32_t trees = 0, tree_begin = 0;
  uint32_t num_trees = 0, mtry = 0, mns = 0;
  uint64_t seed = 0;
  std::vector<uint64_t> off;  // trees+1, tree order
  DevBuf<int32_t> feature, left;
  DevBuf<double> thr, value;
  DevBuf<PredNode> packed;  // 16-byte predict nodes: built on first use (ensure_packed)
  std::mutex pk_mu;
  DevBuf<uint64_t> d_off;
  DevBuf<uint32_t> inbag;    // trees x n (may be empty)
  DevBuf<uint32_t> oobleaf;  // trees x n tree-local OOB leaf index, kInBag = in bag
  uint64_t oob_ctx = 0;      // uid of the aiwc_ctx whose rows oobleaf walks (0: none)
  bool has_oob = false;
  aiwc_oob_stats oob{};
  // measurement: grow-kernel device time (CUDA events on its stream), whole fit time,
  // sum over split nodes of their rows (the algorithmic-bytes unit)
  double grow_ms = 0, fit_ms = 0;
  uint64_t split_rows = 0;
  uint32_t grow_launches = 0;
  // largest split column (-2 = not yet computed), for the schema-width check of predict
  std::mutex mf_mu;
  int32_t max_feature = -2;
  // binned, chunked copy for the shared-memory predict path (built on first predict)
  struct Chunk {
    uint64_t node0, leaf0, root0;
    uint32_t nnodes, nleaves, ntrees;
  };
  std::mutex bin_mu;
  bool bin_ready = false, bin_ok = false;
  uint32_t bin_p = 0, bin_bytes = 1;
  std::vector<Chunk> chunks;
  DevBuf<BinNode> bnodes;
  DevBuf<uint32_t> bnodes4;  // packed 4-byte nodes (node_bytes == 4)
  int node_bytes = 8;
  PredFmt fmt{};  // their field layout
  DevBuf<double> bleaves, bthr;
  DevBuf<uint32_t> broots, bthr_off;
  // host copy of the node SoA + in-bag draws, made by a batched fit for each of its
  // forests in one transfer (the batch's callers export them without device calls)
  bool host_cached = false;
  const int32_t *h_feature = nullptr, *h_left = nullptr;  // into the parent's pinned copy
  const double *h_thr = nullptr, *h_value = nullptr;
  const uint32_t* h_inbag = nullptr;
  std::pair<char*, size_t> pinned{nullptr, 0};  // (parent) that copy, back to PinnedPool
  // a forest split out of a batched fit views its parent's device arrays
  std::shared_ptr<aiwc_forest> parent;
  DevBuf<uint64_t> aux;  // (parent) the children's rebased per-tree node offsets
  // few-row predictions (the reference's per-row predict_response / predict_time loops,
  // experiments.hpp:399-402): a stream, device buffers and pinned staging kept per forest
  std::mutex sm_mu;
  cudaStream_t sm_stream = nullptr;
  DevBuf<double> sm_rows, sm_out;
  std::pair<char*, size_t> sm_pin{nullptr, 0};  // from PinnedPool
  // pinned host mirror of the node SoA (+ right children) and in-bag draws, built on the
  // first aiwc_forest_host_view: [thr N][value N][feature N][left N][right N][inbag T*n]
  std::mutex view_mu;
  std::pair<char*, size_t> view_pin{nullptr, 0};  // from PinnedPool
  std::pair<char*, size_t> inbag_pin{nullptr, 0};  // in-bag mirror filled during the fit
  ~aiwc_forest() {
    if (sm_stream) cudaStreamDestroy(sm_stream);
    PinnedPool::give(sm_pin);
    PinnedPool::give(pinned);
    PinnedPool::give(view_pin);
    PinnedPool::give(inbag_pin);
  }
};

namespace {
void check_row_width(aiwc_forest* f, uint32_t p, cudaStream_t s);  // below, with predict

// 16-byte predict nodes of a fitted forest, built on first use (OOB walks of imported
// forests, the L2 predict paths): a fit does not pay their 16 B/node of allocation and
// writes (6 GB per 1000 C4 trees) unless something walks them.
void ensure_packed(aiwc_forest* f, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(f->pk_mu);
  if (f->packed.p) return;
  const uint64_t N = f->off.back();
  f->packed.alloc(N);
  DevBuf<uint32_t> bad(1);
  CK(cudaMemsetAsync(bad.p, 0, 4, s));
  pack_check_kernel<<<std::min<uint32_t>(f->trees, 148u * 16u), 256, 0, s>>>(
      f->d_off.p, f->trees, f->feature.p, f->thr.p, f->left.p, f->value.p, f->packed.p, bad.p);
  CK(cudaGetLastError());
  g_launches += 1;
  CK(cudaStreamSynchronize(s));
}
}  // namespace

extern "C" {

const char* aiwc_last_error(void) { return g_last_error.c_str(); }

const char* aiwc_version(void) { return "aiwc-b200 1 sm_100a"; }

int aiwc_device_count(int* out) {
  return guard([&] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
    cudaGetLastError();
    if (out) *out = c;
  });
}

uint64_t aiwc_derive_seed(uint64_t seed, const char* tag, uint64_t index) {
  return host_derive_seed(seed, tag, index);
}

int aiwc_ctx_create(const double* col, const double* y, uint64_t n, uint32_t p, int device,
                    aiwc_ctx** out) {
  return guard([&] {
    if (!col || !y || !out) throw Status(AIWC_EARG, "NULL argument");
    if (n < 2) throw Status(AIWC_EEXEC, "dataset must have at least 2 rows");
    if (p < 1 || p > 1024) throw Status(AIWC_EARG, "predictor count must be in [1, 1024]");
    if (n >= (uint64_t{1} << 31)) throw Status(AIWC_EARG, "too many rows (max 2^31-1)");
    DeviceGuard dg(device);
    auto ctx = std::make_unique<aiwc_ctx>();
    static std::atomic<uint64_t> next_uid{1};
    ctx->uid = next_uid.fetch_add(1);
    ctx->device = device;
    ctx->n = n;
    ctx->p = p;
    ctx->y.assign(y, y + n);
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    const cudaStream_t s = ctx->stream;
    ctx->col.alloc(size_t{p} * n);
    ctx->dy.alloc(n);
    h2d(ctx->col.p, col, size_t{p} * n * 8, s);
    h2d(ctx->dy.p, y, n * 8, s);
    {  // the reference rejects nothing here, but a non-finite value has no total order
      DevBuf<unsigned long long> bad(2);
      CK(cudaMemsetAsync(bad.p, 0, 16, s));
      CK(count_nonfinite(ctx->col.p, size_t{p} * n, bad.p, s));
      CK(count_nonfinite(ctx->dy.p, n, bad.p + 1, s));
      unsigned long long hb[2];
      CK(cudaMemcpyAsync(hb, bad.p, 16, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      g_launches += 2;
      if (hb[0]) throw Status(AIWC_EEXEC, "non-finite predictor value");
      if (hb[1]) throw Status(AIWC_EEXEC, "non-finite response value");
    }
    // presort on the device (presort.cu): argsorts, dense ranks, distinct values
    DevBuf<uint32_t> sorted(size_t{p} * n), rank32(size_t{p} * n), counts(p);
    DevBuf<double> vals_tmp(size_t{p} * n);
    uint64_t nl = 0;
    CK(gpu_presort(ctx->col.p, n, p, s, sorted.p, rank32.p, vals_tmp.p, counts.p, &nl));
    g_launches += nl;
    std::vector<uint32_t> cnt(p);
    CK(cudaMemcpyAsync(cnt.data(), counts.p, p * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<uint64_t> voff(p + 1, 0);
    uint64_t maxk = 0;
    for (uint32_t c = 0; c < p; ++c) {
      voff[c + 1] = voff[c] + cnt[c];
      maxk = std::max<uint64_t>(maxk, cnt[c]);
    }
    ctx->rank_bytes = maxk <= 65536 ? 2 : 4;
    // listed columns: >= 3 distinct values (two-level columns are read off the payload)
    std::vector<int32_t> list_of(p, -1);
    std::vector<uint32_t> listed;
    for (uint32_t c = 0; c < p; ++c)
      if (cnt[c] >= 3) {
        list_of[c] = static_cast<int32_t>(listed.size());
        listed.push_back(c);
      }
    ctx->nlisted = static_cast<uint32_t>(listed.size());
    ctx->order_stride = static_cast<uint32_t>((n + 15) & ~uint64_t{15});
    const size_t osz = std::max<size_t>(size_t{ctx->nlisted} * ctx->order_stride, 16);
    ctx->order.alloc(osz);
    CK(cudaMemsetAsync(ctx->order.p, 0, osz * 4, s));
    for (uint32_t i = 0; i < ctx->nlisted; ++i)
      CK(cudaMemcpyAsync(ctx->order.p + size_t{i} * ctx->order_stride,
                         sorted.p + size_t{listed[i]} * n, n * 4, cudaMemcpyDeviceToDevice, s));
    ctx->rank.alloc(size_t{p} * n * ctx->rank_bytes);
    if (ctx->rank_bytes == 2) {
      CK(narrow_ranks(rank32.p, size_t{p} * n, reinterpret_cast<uint16_t*>(ctx->rank.p), s));
      g_launches += 1;
    } else {
      CK(cudaMemcpyAsync(ctx->rank.p, rank32.p, size_t{p} * n * 4, cudaMemcpyDeviceToDevice, s));
    }
    ctx->vals.alloc(std::max<uint64_t>(voff[p], 1));
    for (uint32_t c = 0; c < p; ++c)
      CK(cudaMemcpyAsync(ctx->vals.p + voff[c], vals_tmp.p + size_t{c} * n, cnt[c] * 8,
                         cudaMemcpyDeviceToDevice, s));
    ctx->list_of.alloc(p);
    ctx->listed.alloc(std::max<size_t>(listed.size(), 1));
    ctx->vals_off.alloc(voff.size());
    CK(cudaMemcpyAsync(ctx->list_of.p, list_of.data(), p * 4, cudaMemcpyHostToDevice, s));
    if (!listed.empty())
      CK(cudaMemcpyAsync(ctx->listed.p, listed.data(), listed.size() * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->vals_off.p, voff.data(), voff.size() * 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));  // the temporaries above are freed on return
    {
      SlotArena& ar = slot_arena(device);
      std::lock_guard<std::mutex> g(ar.mu);
      ++ar.ctxs;
    }
    *out = ctx.release();
  });
}

int aiwc_ctx_free(aiwc_ctx* ctx) {
  if (!ctx) return AIWC_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  {  // the device's last dataset: hand the slot arena back to the pool
    SlotArena& ar = slot_arena(ctx->device);
    std::lock_guard<std::mutex> g(ar.mu);
    if (--ar.ctxs <= 0 && !ar.busy) {
      ar.ctxs = 0;
      ar.buf.release();
      cache_flush(ctx->device);
    }
  }
  delete ctx;
  cudaSetDevice(prev);
  return AIWC_OK;
}

int aiwc_ctx_set_host_mirror(aiwc_ctx* ctx, int on) {
  return guard([&] {
    if (!ctx) throw Status(AIWC_EARG, "ctx is NULL");
    std::lock_guard<std::mutex> lock(ctx->mu);
    ctx->host_mirror = on != 0;
  });
}

int aiwc_release_cached(int device) {
  return guard([&] {
    DeviceGuard dg(device);
    {
      SlotArena& ar = slot_arena(device);
      std::lock_guard<std::mutex> g(ar.mu);
      if (!ar.busy) ar.buf.release();
    }
    cache_flush(device);
    PinnedPool::release_all();  // idle pinned host buffers (forest mirrors, staging)
    CK(cudaDeviceSynchronize());
    cudaMemPool_t mp;
    if (cudaDeviceGetDefaultMemPool(&mp, device) == cudaSuccess) cudaMemPoolTrimTo(mp, 0);
  });
}

int aiwc_ctx_info(const aiwc_ctx* ctx, uint64_t* n, uint32_t* p, int* device) {
  return guard([&] {
    if (!ctx) throw Status(AIWC_EARG, "ctx is NULL");
    if (n) *n = ctx->n;
    if (p) *p = ctx->p;
    if (device) *device = ctx->device;
  });
}

}  // extern "C"

namespace {

// Per-row tree-ordered sums -> OobStats with the reference's row-order loops
// (forest.hpp:396-453); host side so the reduction order is literally the same.
aiwc_oob_stats finalize_oob(const double* y, uint64_t n, const double* sum,
                            const uint32_t* count) {
  aiwc_oob_stats st{};
  double mean = 0;
  for (uint64_t i = 0; i < n; ++i) mean += y[i];
  mean /= static_cast<double>(n);
  double var = 0;
  bool constant = true;
  for (uint64_t i = 0; i < n; ++i) {
    var += (y[i] - mean) * (y[i] - mean);
    if (y[i] != y[0]) constant = false;
  }
  var /= static_cast<double>(n);
  st.response_variance = var;
  if (constant) {
    st.degenerate = 1;
    return st;
  }
  double mse = 0;
  uint64_t ev = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (!count[i]) continue;
    const double pred = sum[i] / static_cast<double>(count[i]);
    mse += (pred - y[i]) * (pred - y[i]);
    ++ev;
  }
  if (ev == 0) throw Status(AIWC_EEXEC, "no out-of-bag rows: every row was in every bag");
  mse /= static_cast<double>(ev);
  st.mse = mse;
  st.rows_evaluated = ev;
  st.error_pct = 100.0 * mse / var;
  st.r_squared = 1.0 - mse / var;
  return st;
}

void oob_accumulate_device(aiwc_forest* f, double* row_sum, uint32_t* row_count,
                           cudaStream_t s) {
  const uint64_t n = f->n;
  DevBuf<double> ds(n);
  DevBuf<uint32_t> dc(n);
  CK(cudaMemcpyAsync(ds.p, row_sum, n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dc.p, row_count, n * 4, cudaMemcpyHostToDevice, s));
  oob_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      f->oobleaf.p, f->d_off.p, f->value.p, f->trees, n, ds.p, dc.p);
  CK(cudaGetLastError());
  g_launches += 1;
  CK(cudaMemcpyAsync(row_sum, ds.p, n * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(row_count, dc.p, n * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

int pick_threads(uint64_t n) {
  if (const char* e = std::getenv("AIWC_GROW_NT")) return std::atoi(e) == 512 ? 512 : 256;
  return n >= 65536 ? 512 : 256;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

// One fit: trees [tree_begin, tree_end) of a num_trees forest, or, with `cells`, the
// cells->n forests (grid cells, batched concurrent fits): forest c grows its trees
// [tb[c], te[c]) with its own mtry / mns / seed, all in one launch; its trees follow
// those of forest c-1 in the result.
struct CellSpec {
  uint32_t n;
  const uint32_t* mtry;
  const uint32_t* mns;
  const uint64_t* seed;
  const uint32_t* tb;
  const uint32_t* te;
  // hold-out folds: forest c trains on the nrows[c] table rows rows[rows_off[c] ..];
  // no in-bag lists or OOB leaves are kept (evaluate predicts the held-out rows only)
  const uint32_t* nrows = nullptr;
  const uint32_t* rows = nullptr;
  const uint64_t* rows_off = nullptr;
};

void fit_body(aiwc_ctx* ctx, uint32_t num_trees, uint32_t mtry, uint32_t min_node_size,
              uint64_t seed, uint32_t tree_begin, uint32_t tree_end, int compute_oob,
              const CellSpec* cells, aiwc_forest** out) {
  std::lock_guard<std::mutex> lock(ctx->mu);
  const auto t_start = std::chrono::steady_clock::now();
  DeviceGuard dg(ctx->device);
  struct {
    cudaStream_t s;
  } st{ctx->stream};
  const uint64_t n = ctx->n;
  const uint32_t p = ctx->p;
  const uint32_t T = tree_end - tree_begin;
  const int nt = pick_threads(n);

  int dev = ctx->device, sms = 0, max_optin = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  SlotLayout L = make_layout(n, p, ctx->nlisted, mtry, min_node_size, false);
  const size_t bits_smem = (grow_bits_words(n, L.stride) + grow_pref_words(n, L.stride)) * 4;
  // static shared memory of grow_kernel: scans + per-warp FP64 stages (< 12 KB)
  const bool smem_bits = bits_smem + 12288 <= static_cast<size_t>(max_optin) &&
                         std::getenv("AIWC_GROW_GBITS") == nullptr;
  const size_t dyn = smem_bits ? bits_smem : 0;
  if (!smem_bits) L = make_layout(n, p, ctx->nlisted, mtry, min_node_size, true);

  GrowArgs a{};
  a.d = ctx->view();
  a.mtry = mtry;
  a.mns = min_node_size;
  a.seed = seed;
  a.tag_tree = host_fnv1a64("tree", 4);
  a.tree_begin = tree_begin;
  a.tree_end = tree_end;
  a.L = L;
  a.bits_in_smem = smem_bits ? 1 : 0;
  DevBuf<uint32_t> cell_m, cell_n, tcell, tidx, fold_n, fold_rows;
  DevBuf<uint64_t> cell_s, fold_off;
  const bool folds = cells && cells->rows;
  if (cells) {
    std::vector<uint32_t> hc, ht;
    for (uint32_t c = 0; c < cells->n; ++c)
      for (uint32_t t = cells->tb[c]; t < cells->te[c]; ++t) {
        hc.push_back(c);
        ht.push_back(t);
      }
    if (hc.size() != T) throw Status(AIWC_EARG, "cell tree ranges do not add up");
    cell_m.alloc(cells->n);
    cell_n.alloc(cells->n);
    cell_s.alloc(cells->n);
    tcell.alloc(T);
    tidx.alloc(T);
    CK(cudaMemcpy(cell_m.p, cells->mtry, cells->n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(cell_n.p, cells->mns, cells->n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(cell_s.p, cells->seed, cells->n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(tcell.p, hc.data(), size_t{T} * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(tidx.p, ht.data(), size_t{T} * 4, cudaMemcpyHostToDevice));
    a.cell_mtry = cell_m.p;
    a.cell_mns = cell_n.p;
    a.cell_seed = cell_s.p;
    a.tree_cell = tcell.p;
    a.tree_t = tidx.p;
    if (folds) {
      const uint64_t total_rows = cells->rows_off[cells->n];
      fold_n.alloc(cells->n);
      fold_off.alloc(cells->n + 1);
      fold_rows.alloc(total_rows);
      CK(cudaMemcpy(fold_n.p, cells->nrows, cells->n * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(fold_off.p, cells->rows_off, (cells->n + 1) * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(fold_rows.p, cells->rows, total_rows * 4, cudaMemcpyHostToDevice));
      a.cell_nrows = fold_n.p;
      a.cell_rows = fold_rows.p;
      a.cell_rows_off = fold_off.p;
    }
  }

  // large tables grow batches of trees level-synchronously with one grid-wide kernel
  // per phase (grow_wide.cuh); small ones keep one persistent CTA per tree
  // The batched level-synchronous grower (grow_wide.cuh) for large tables, and for small
  // tables grown 64+ trees at a time (then in one batch: measured 13 -> 9 ms for 1000 C1
  // trees); the CTA-per-tree grower for a few small trees
  const bool small_table = n < 65536;
  bool wide = !small_table || T >= 64;
  if (const char* e = std::getenv("AIWC_GROW_WIDE")) wide = std::atoi(e) != 0;
  if (folds) wide = true;  // only the batched grower maps fold rows
  if (wide) {
    L = make_layout(n, p, ctx->nlisted, mtry, min_node_size, true);
    a.L = L;
    a.bits_in_smem = 0;
  }
  int per_sm = 0;
  if (wide) {
    // large tables: up to 4 trees per SM per batch (bounded by memory below); small ones:
    // every tree in one batch
    per_sm = small_table ? static_cast<int>((T + sms - 1) / sms) : 4;
    if (const char* e = std::getenv("AIWC_WIDE_PER_SM")) per_sm = std::max(1, std::atoi(e));
  }
  else
    CK(launch_grow(nt, ctx->rank_bytes, a, 0, dyn, st.s, &per_sm));
  if (per_sm < 1) throw Status(AIWC_ECUDA, "grow kernel does not fit on an SM");
  const bool tprof = std::getenv("AIWC_PROFILE_PHASES") != nullptr;
  auto tmark = [&](const char* what) {
    if (!tprof) return;
    static thread_local auto last = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[aiwc setup] %s %.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  };
  tmark("start");
  // outputs first: in-bag draws, OOB leaf values, node pool
  auto f = std::make_unique<aiwc_forest>();
  f->device = dev;
  f->n = n;
  f->trees = T;
  f->tree_begin = tree_begin;
  f->num_trees = num_trees;
  f->mtry = mtry;
  f->mns = min_node_size;
  f->seed = seed;
  // every (tree, row) entry of both is written by the grower (no fill needed)
  if (!folds) {
    f->inbag.alloc_cached(size_t{T} * n, dev);
    f->oobleaf.alloc_cached(size_t{T} * n, dev);
  }
  // in-bag host mirror: each batch's draws go to pinned memory on a copy stream while the
  // next batches grow (the wide grower writes a batch's draws in its first kernel)
  cudaStream_t cstream = nullptr;
  struct CsGuard {
    cudaStream_t& s;
    ~CsGuard() {
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    }
  } csg{cstream};
  if (ctx->host_mirror && !folds && !cells && f->inbag.p) {
    f->inbag_pin = PinnedPool::take(size_t{T} * n * 4);
    CK(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
  }
  f->oob_ctx = ctx->uid;
  tmark("inbag+oobleaf");
  a.inbag = f->inbag.p;
  a.oobleaf = f->oobleaf.p;

  uint64_t cap = uint64_t{T} * std::min<uint64_t>(L.nodes_cap, std::max<uint64_t>(1024, L.stride));
  int slots = static_cast<int>(std::min<uint64_t>(T, uint64_t(per_sm) * sms));
  // node pool (28 B/node) plus the compacted forest built from it after growth
  // (feature, left, thr, value, PredNode: 40 B/node) stay outside the slot scratch
  const size_t pool_bytes = cap * (28 + 40);
  // cudaMemGetInfo can stall for tens of milliseconds: small fits (a grid search's
  // thousands of C1-size fits) skip the free-memory budget when they need under 1/16
  // of the device
  static size_t total_mem[64] = {};
  size_t free_b = 0, total_b = 0;
  if (dev < 64 && total_mem[dev] == 0) {
    CK(cudaMemGetInfo(&free_b, &total_b));
    total_mem[dev] = total_b;
  }
  const size_t dev_total = dev < 64 ? total_mem[dev] : 0;
  const bool small = dev_total && pool_bytes + size_t(slots) * L.bytes < dev_total / 16;
  if (small) {
    free_b = dev_total;  // ample: the budget below keeps every slot
  } else {
    CK(cudaMemGetInfo(&free_b, &total_b));
    // memory parked in the stream-ordered pool (and this ctx's scratch, which is
    // reused or replaced) is available too; cudaMemGetInfo does not count it
    cudaMemPool_t mp;
    uint64_t reserved = 0, used_now = 0;
    if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess &&
        cudaMemPoolGetAttribute(mp, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
        cudaMemPoolGetAttribute(mp, cudaMemPoolAttrUsedMemCurrent, &used_now) == cudaSuccess &&
        reserved > used_now)
      free_b += reserved - used_now;
    free_b += slot_arena_size(dev) + cache_idle_bytes(dev);
  }
  const size_t budget = free_b > pool_bytes + (size_t{2} << 30) ? free_b - pool_bytes - (size_t{2} << 30) : 0;
  // memory-limited (e.g. the caller still holds an earlier forest): the arena must shrink
  // to what this fit uses, since the budget counted all of it as available
  const bool tight = budget / L.bytes < static_cast<size_t>(slots);
  slots = static_cast<int>(std::min<size_t>(slots, budget / L.bytes));
  if (slots < 1) throw Status(AIWC_ECUDA, "not enough device memory for one tree slot");
  const size_t need = size_t(slots) * L.bytes;
  tmark("budget");
  // the slots live in the device's slot arena (kept between fits: a 100+ GB block
  // re-allocated every fit fragmented the pool around the forests' own allocations and
  // the next fit stalled for seconds while the pool grew); a second fit running on the
  // device at the same time gets its own temporary block
  SlotLease lease(dev, need, tight);
  tmark("scratch");
  a.scratch = lease.p;
  int nlanes = 1;
  if (wide) {
    // concurrent batches (streams + host threads): 2 -> 4 measured +3 % at C4; a small
    // table's single batch keeps one lane
    // (round 2, after the list-pass change: 2 / 3 / 4 / 6 / 8 lanes -> 3.39 / 3.39 /
    // 3.42 / 3.46 / 3.49 s per 1000 C4 trees)
    nlanes = small_table ? 1 : 3;
    if (const char* e = std::getenv("AIWC_WIDE_LANES")) nlanes = std::max(1, std::atoi(e));
    nlanes = std::max(1, std::min(nlanes, slots));
  }
  const size_t per_lane = wide ? size_t(slots) / nlanes : 0;
  DevBuf<TreeState> wts(wide ? slots : 0);
  DevBuf<uint32_t> woff(wide ? 5 * nlanes * (per_lane + 1) : 0), wactive(wide ? nlanes : 0),
      wctr(wide ? 4 * nlanes : 0);
  // per-lane "trees still splitting" flags read back every level: a pinned buffer per
  // fit, taken from a process-wide pool (cudaMallocHost / cudaFreeHost synchronise
  // and cost milliseconds -- too much for the many small fits of a grid search)
  PinnedFlags h_active;
  std::vector<cudaStream_t> lane_streams;
  struct StreamsGuard {
    std::vector<cudaStream_t>& v;
    ~StreamsGuard() {
      for (auto s : v) cudaStreamDestroy(s);
    }
  } lsg{lane_streams};
  for (int k = 1; k < nlanes; ++k) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    lane_streams.push_back(s);
  }

  DevBuf<uint32_t> queue(1), tree_cnt(T);
  DevBuf<int> err(1);
  DevBuf<uint64_t> tree_off(T);
  a.queue = queue.p;
  a.tree_off = tree_off.p;
  a.tree_cnt = tree_cnt.p;
  a.err = err.p;
  DevBuf<int32_t> pf, pl;
  DevBuf<double> pt, pv;
  DevBuf<uint32_t> pr;
  DevBuf<unsigned long long> used(1), split_rows(1), prof;
  a.split_rows = split_rows.p;
  const bool want_prof = std::getenv("AIWC_PROFILE_PHASES") != nullptr;
  if (want_prof) {
    prof.alloc(16);
    CK(cudaMemset(prof.p, 0, 16 * 8));
    a.prof = prof.p;
  }
  std::vector<uint32_t> cnt(T);
  cudaEvent_t ev0, ev1, evf0, evf1;
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  CK(cudaEventCreate(&evf0));
  CK(cudaEventCreate(&evf1));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  };
  cudaEvent_t evs[4] = {ev0, ev1, evf0, evf1};
  EvGuard eg{evs};
  CK(cudaEventRecord(evf0, st.s));
      tmark("streams+events+pool");
  const auto t_grow0 = std::chrono::steady_clock::now();
  for (int attempt = 0; attempt < 2; ++attempt) {
    pf.alloc_cached(cap, dev);
    pl.alloc_cached(cap, dev);
    pt.alloc_cached(cap, dev);
    pv.alloc_cached(cap, dev);
    pr.alloc_cached(cap, dev);
    a.pool_feature = pf.p;
    a.pool_left = pl.p;
    a.pool_thr = pt.p;
    a.pool_value = pv.p;
    a.pool_rank = pr.p;
    a.pool_used = used.p;
    a.pool_cap = cap;
    CK(cudaMemsetAsync(queue.p, 0, 4, st.s));
    CK(cudaMemsetAsync(err.p, 0, 4, st.s));
    CK(cudaMemsetAsync(used.p, 0, 8, st.s));
    CK(cudaMemsetAsync(split_rows.p, 0, 8, st.s));
    CK(cudaEventRecord(ev0, st.s));
    // lane streams start after these resets (and the counters' earlier uses) on st.s
    for (cudaStream_t ls : lane_streams) CK(cudaStreamWaitEvent(ls, ev0, 0));
    if (wide) {
      // batched multi-kernel grower: K concurrent lanes (stream + host thread), each
      // growing batches of `per` trees level-synchronously.  While one batch sits in
      // the sequential tail of a level (a few long chains on huge nodes), the other
      // lanes' kernels fill the SMs.
      const int K = nlanes;
      // a batch's trees are gridDim.y of the per-row kernels: at most 65,535
      const uint32_t per = std::min<uint32_t>(static_cast<uint32_t>(slots / K), 65535u);
      // rows from which a node's chains run in 16-lane groups (w_chains_warp) instead of
      // 4-lane groups (w_chains_grp); measured at C4: 2K / 4K / 8K / 16K / 32K / 64K ->
      // 3.45 / 3.44 / 3.45 / 3.41 / 3.41 / 3.42 s per 1000 trees, all nodes 4-lane +7 %
      uint32_t big_min = 16384;
      if (const char* e = std::getenv("AIWC_BIG_MIN")) big_min = static_cast<uint32_t>(std::atoll(e));
      // CTA-per-chain / CTA-per-route for nodes >= coop_min rows: shorter critical
      // paths, more warps per node -- a win only when a lane's batch is too small to
      // keep the GPU busy (measured at C4: 64 trees +5 %, 200 trees -6 %, 1000 -7 %)
      // lanes per chain for big nodes: 32 (a warp each) or 16 / 8 (lane groups)
      uint32_t lane_max = 16;  // rows below which a node's chains run one lane each (measured)
      if (const char* e = std::getenv("AIWC_LANE_MAX")) lane_max = static_cast<uint32_t>(std::atoi(e));
      uint32_t big_lanes = 16;
      if (const char* e = std::getenv("AIWC_BIG_LANES")) big_lanes = static_cast<uint32_t>(std::atoi(e));
      if (big_lanes != 8 && big_lanes != 16) big_lanes = 32;
      uint32_t coop_min = per <= 48 ? 32768u : 0xffffffffu;
      if (const char* e = std::getenv("AIWC_COOP_MIN")) coop_min = static_cast<uint32_t>(std::atoll(e));
      coop_min = std::max(coop_min, big_min);
      if (std::getenv("AIWC_VERBOSE"))
        std::fprintf(stderr, "[aiwc wide] trees=%u slots=%d lanes=%d per=%u slot_bytes=%zu\n", T, slots,
                     K, per, L.bytes);
      std::vector<cudaError_t> lane_err(K, cudaSuccess);
      std::vector<std::thread> lanes;
      for (int k = 0; k < K; ++k) {
        lanes.emplace_back([&, k] {
          cudaSetDevice(dev);
          const cudaStream_t ls = k == 0 ? st.s : lane_streams[k - 1];
          for (uint32_t t0 = k * per; t0 < T; t0 += K * per) {
            WideArgs w{};
            w.g = a;
            w.g.scratch = a.scratch + size_t{k} * per * L.bytes;
            w.ts = wts.p + size_t{k} * per;
            w.B = std::min<uint32_t>(per, T - t0);
            w.big_min = big_min;
            w.coop_min = coop_min;
            w.pair_big = big_lanes;
            w.lane_max = lane_max;
            w.t0 = t0;
            for (int i = 0; i < 5; ++i)
              w.off[i] = woff.p + (size_t{k} * 5 + i) * (per + 1);
            w.active = wactive.p + k;
            w.task_ctr = wctr.p + 4 * k;
            uint64_t nl = 0;
            cudaError_t e = run_wide(ctx->rank_bytes, w, ls, sms, h_active.get() + k, &nl);
            g_launches += nl;
            if (e == cudaSuccess) e = cudaStreamSynchronize(ls);
            if (e == cudaSuccess && cstream)  // this batch's draws to the host mirror
              e = cudaMemcpyAsync(f->inbag_pin.first + size_t{t0} * n * 4,
                                  f->inbag.p + size_t{t0} * n, size_t{w.B} * n * 4,
                                  cudaMemcpyDeviceToHost, cstream);
            if (e != cudaSuccess) {
              lane_err[k] = e;
              return;
            }
          }
        });
      }
      for (auto& th : lanes) th.join();
      for (cudaError_t e : lane_err)
        if (e != cudaSuccess) throw Status(AIWC_ECUDA, std::string("wide grower: ") + cudaGetErrorString(e));
    } else {
      CK(launch_grow(nt, ctx->rank_bytes, a, slots, dyn, st.s, nullptr));
      g_launches += 1;
      if (cstream) {
        CK(cudaStreamSynchronize(st.s));
        CK(cudaMemcpyAsync(f->inbag_pin.first, f->inbag.p, size_t{T} * n * 4,
                           cudaMemcpyDeviceToHost, cstream));
      }
    }
    CK(cudaEventRecord(ev1, st.s));
    f->grow_launches += 1;
    int herr = 0;
    unsigned long long hused = 0;
    CK(cudaMemcpyAsync(&herr, err.p, 4, cudaMemcpyDeviceToHost, st.s));
    CK(cudaMemcpyAsync(&hused, used.p, 8, cudaMemcpyDeviceToHost, st.s));
    CK(cudaStreamSynchronize(st.s));
    {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ev0, ev1));
      f->grow_ms += ms;
    }
    if (herr == 1 && attempt == 0) {  // pool overflow: exact size is now known
      cap = hused;
      continue;
    }
    if (herr == 2) throw Status(AIWC_EEXEC, "in-bag row count exceeded the slot bound");
    if (herr == 3) throw Status(AIWC_EEXEC, "frontier/node capacity exceeded");
    if (herr) throw Status(AIWC_EEXEC, "grow kernel error " + std::to_string(herr));
    break;
  }
  CK(cudaMemcpy(cnt.data(), tree_cnt.p, size_t{T} * 4, cudaMemcpyDeviceToHost));
  if (want_prof) {
    unsigned long long h[16];
    CK(cudaMemcpy(h, prof.p, 16 * 8, cudaMemcpyDeviceToHost));
    static const char* names[14] = {"bootstrap", "bitmap", "payload0", "lists0+root",
                                    "-", "elig", "sample", "chains", "decide", "route",
                                    "segtab", "paypass", "listpass", "emit+oob"};
    double tot = 0;
    for (int i = 0; i < 14; ++i) tot += static_cast<double>(h[i]);
    std::fprintf(stderr, "[aiwc grow phases] slots=%d trees=%u total=%.3g cycles:", slots, T, tot);
    for (int i = 0; i < 14; ++i)
      if (h[i]) std::fprintf(stderr, " %s=%.1f%%", names[i], 100.0 * h[i] / tot);
    std::fprintf(stderr, "\n");
  }
  f->off.assign(T + 1, 0);
  for (uint32_t t = 0; t < T; ++t) f->off[t + 1] = f->off[t] + cnt[t];
  const uint64_t N = f->off[T];
  const auto t_alloc0 = std::chrono::steady_clock::now();
  f->feature.alloc_cached(N, dev);
  f->left.alloc_cached(N, dev);
  f->thr.alloc_cached(N, dev);
  f->value.alloc_cached(N, dev);
  f->d_off.alloc(T + 1);
  const auto t_alloc1 = std::chrono::steady_clock::now();
  CK(cudaMemcpyAsync(f->d_off.p, f->off.data(), (T + 1) * 8, cudaMemcpyHostToDevice, st.s));
  compact_kernel<<<T, 256, 0, st.s>>>(pf.p, pt.p, pl.p, pv.p, tree_off.p, f->d_off.p,
                                      f->feature.p, f->thr.p, f->left.p, f->value.p, nullptr);
  CK(cudaGetLastError());
  g_launches += 1;
  CK(cudaMemcpyAsync(&f->split_rows, split_rows.p, 8, cudaMemcpyDeviceToHost, st.s));
  CK(cudaStreamSynchronize(st.s));
  const auto t_compact = std::chrono::steady_clock::now();
  if (want_prof)
    std::fprintf(stderr, "[aiwc compact] alloc %.1f ms, kernel+sync %.1f ms\n",
                 std::chrono::duration<double, std::milli>(t_alloc1 - t_alloc0).count(),
                 std::chrono::duration<double, std::milli>(t_compact - t_alloc1).count());
  if (compute_oob && tree_begin == 0 && tree_end == num_trees) {
    std::vector<double> sum(n, 0.0);
    std::vector<uint32_t> count(n, 0);
    oob_accumulate_device(f.get(), sum.data(), count.data(), st.s);
    f->oob = finalize_oob(ctx->y.data(), n, sum.data(), count.data());
    f->has_oob = true;
  }
  if (want_prof) {
    const auto now = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[aiwc fit host] setup %.1f ms, grow+compact %.1f ms, oob %.1f ms\n",
                 ms(t_start, t_grow0), ms(t_grow0, t_compact), ms(t_compact, now));
  }
  CK(cudaEventRecord(evf1, st.s));
  CK(cudaEventSynchronize(evf1));
  {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, evf0, evf1));
    f->fit_ms = ms;
  }
  *out = f.release();
}

}  // namespace

extern "C" {

namespace {

// Forest c of a multi-forest fit (trees [t0, t1) of F) as a forest of its own: views of
// F's node SoA, in-bag draws and OOB leaves (F stays alive while any child does);
// d_off = the child's slice of F->aux (offsets rebased to the child's first node).
aiwc_forest* split_cell(const std::shared_ptr<aiwc_forest>& F, uint32_t t0, uint32_t t1,
                        uint64_t aux0, const aiwc_ctx::FitRequest& r) {
  auto f = std::make_unique<aiwc_forest>();
  const uint64_t n = F->n, b = F->off[t0], N = F->off[t1] - b;
  const uint32_t T = t1 - t0;
  f->parent = F;
  f->device = F->device;
  f->n = n;
  f->trees = T;
  f->tree_begin = r.tb;
  f->num_trees = r.num_trees;
  f->mtry = r.mtry;
  f->mns = r.mns;
  f->seed = r.seed;
  f->grow_ms = F->grow_ms;
  f->fit_ms = F->fit_ms;
  f->grow_launches = F->grow_launches;
  f->off.resize(T + 1);
  for (uint32_t t = 0; t <= T; ++t) f->off[t] = F->off[t0 + t] - b;
  f->feature.view(F->feature.p + b, N);
  f->left.view(F->left.p + b, N);
  f->thr.view(F->thr.p + b, N);
  f->value.view(F->value.p + b, N);
  f->d_off.view(F->aux.p + aux0, T + 1);
  f->inbag.view(F->inbag.p + size_t{t0} * n, size_t{T} * n);
  f->oobleaf.view(F->oobleaf.p + size_t{t0} * n, size_t{T} * n);
  f->oob_ctx = F->oob_ctx;
  return f.release();
}

// One queued batch: a lone request is a plain fit; several grow as the forests of one
// multi-forest launch (each tree keyed by its own forest's seed and index, so every
// forest equals its standalone fit bit for bit) and are then split apart.
void fit_batch(aiwc_ctx* ctx, const std::vector<aiwc_ctx::FitRequest*>& batch) {
  auto fail_all = [&](int rc, const std::string& m) {
    for (auto* r : batch) {
      if (r->out) {
        aiwc_forest_free(r->out);
        r->out = nullptr;
      }
      r->status = rc;
      r->msg = m;
    }
  };
  try {
    if (batch.size() == 1) {
      auto* r = batch[0];
      fit_body(ctx, r->num_trees, r->mtry, r->mns, r->seed, r->tb, r->te, r->compute_oob,
               nullptr, &r->out);
      return;
    }
    const uint32_t k = static_cast<uint32_t>(batch.size());
    std::vector<uint32_t> m(k), mn(k), tb(k), te(k);
    std::vector<uint64_t> sd(k);
    uint32_t mmax = 0, nmin = UINT32_MAX, total = 0;
    for (uint32_t i = 0; i < k; ++i) {
      m[i] = batch[i]->mtry;
      mn[i] = batch[i]->mns;
      sd[i] = batch[i]->seed;
      tb[i] = batch[i]->tb;
      te[i] = batch[i]->te;
      mmax = std::max(mmax, m[i]);
      nmin = std::min(nmin, mn[i]);
      total += te[i] - tb[i];
    }
    const CellSpec cs{k, m.data(), mn.data(), sd.data(), tb.data(), te.data()};
    aiwc_forest* F = nullptr;
    using clk = std::chrono::steady_clock;
    const auto c0 = clk::now();
    fit_body(ctx, total, mmax, nmin, sd[0], 0, total, 0, &cs, &F);
    const auto c1 = clk::now();
    const std::shared_ptr<aiwc_forest> Fs(F, [](aiwc_forest* x) { aiwc_forest_free(x); });
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    const cudaStream_t st = ctx->stream;
    const uint64_t n = F->n;
    // children's rebased node offsets, one upload
    std::vector<uint64_t> aux;
    std::vector<uint32_t> t0s(k + 1, 0);
    for (uint32_t i = 0; i < k; ++i) t0s[i + 1] = t0s[i] + (te[i] - tb[i]);
    for (uint32_t i = 0; i < k; ++i)
      for (uint32_t t = t0s[i]; t <= t0s[i + 1]; ++t) aux.push_back(F->off[t] - F->off[t0s[i]]);
    F->aux.alloc(aux.size());
    CK(cudaMemcpyAsync(F->aux.p, aux.data(), aux.size() * 8, cudaMemcpyHostToDevice, st));
    // small batches (tuning loops on paper-sized tables): the whole batch's nodes and
    // in-bag draws come to the host in one transfer each, so the callers' exports are
    // plain copies
    const uint64_t N = F->off.back();
    const size_t cbytes = N * 24 + size_t{total} * n * 4;
    const bool cache = cbytes < (size_t{256} << 20);
    int32_t *hf = nullptr, *hl = nullptr;
    double *ht = nullptr, *hv = nullptr;
    uint32_t* hi = nullptr;
    if (cache) {  // straight DMA into a pinned buffer the batch forest owns
      F->pinned = PinnedPool::take(cbytes);
      ht = reinterpret_cast<double*>(F->pinned.first);
      hv = ht + N;
      hf = reinterpret_cast<int32_t*>(hv + N);
      hl = hf + N;
      hi = reinterpret_cast<uint32_t*>(hl + N);
      CK(cudaMemcpyAsync(ht, F->thr.p, N * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hv, F->value.p, N * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hf, F->feature.p, N * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hl, F->left.p, N * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hi, F->inbag.p, size_t{total} * n * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    const auto c2 = clk::now();
    std::vector<aiwc_forest*> kids(k, nullptr);
    uint64_t a0 = 0;
    for (uint32_t i = 0; i < k; ++i) {
      const uint32_t t0 = t0s[i], t1 = t0s[i + 1];
      aiwc_forest* f = split_cell(Fs, t0, t1, a0, *batch[i]);
      a0 += t1 - t0 + 1;
      kids[i] = f;
      batch[i]->out = f;
      if (cache) {
        const uint64_t b = F->off[t0], e = F->off[t1];
        f->h_feature = hf + b;
        f->h_left = hl + b;
        f->h_thr = ht + b;
        f->h_value = hv + b;
        f->h_inbag = hi + size_t{t0} * n;
        f->host_cached = true;
      }
    }
    const auto c3 = clk::now();
    // OOB statistics of every forest that asks for them: one tree-ordered reduction per
    // forest into one buffer, one transfer, the reference's row-order finalisation each
    DevBuf<double> sums(size_t{k} * n);
    DevBuf<uint32_t> cnts(size_t{k} * n);
    CK(cudaMemsetAsync(sums.p, 0, size_t{k} * n * 8, st));
    CK(cudaMemsetAsync(cnts.p, 0, size_t{k} * n * 4, st));
    bool any = false;
    for (uint32_t i = 0; i < k; ++i) {
      const auto& r = *batch[i];
      if (!(r.compute_oob && r.tb == 0 && r.te == r.num_trees)) continue;
      any = true;
      oob_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
          kids[i]->oobleaf.p, kids[i]->d_off.p, kids[i]->value.p, kids[i]->trees, n,
          sums.p + size_t{i} * n, cnts.p + size_t{i} * n);
      CK(cudaGetLastError());
      g_launches += 1;
    }
    if (any) {
      std::vector<double> hs(size_t{k} * n);
      std::vector<uint32_t> hc(size_t{k} * n);
      CK(cudaMemcpyAsync(hs.data(), sums.p, hs.size() * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hc.data(), cnts.p, hc.size() * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (uint32_t i = 0; i < k; ++i) {
        const auto& r = *batch[i];
        if (!(r.compute_oob && r.tb == 0 && r.te == r.num_trees)) continue;
        try {
          kids[i]->oob = finalize_oob(ctx->y.data(), n, hs.data() + size_t{i} * n,
                                      hc.data() + size_t{i} * n);
          kids[i]->has_oob = true;
        } catch (const Status& e) {  // this forest alone (no out-of-bag rows)
          aiwc_forest_free(kids[i]);
          batch[i]->out = nullptr;
          batch[i]->status = e.code;
          batch[i]->msg = e.msg;
        }
      }
    }
    CK(cudaStreamSynchronize(st));
    if (std::getenv("AIWC_VERBOSE")) {
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "[aiwc batch split] fit_body %.2f, aux+host copy %.2f, children %.2f, oob %.2f ms\n",
                   ms(c0, c1), ms(c1, c2), ms(c2, c3), ms(c3, clk::now()));
    }
  } catch (const Status& e) {
    fail_all(e.code, e.msg);
  } catch (const std::exception& e) {
    fail_all(AIWC_EEXEC, e.what());
  }
}

// Queue a fit on ctx and return when it is grown.  The first caller to find no leader
// leads: it takes every queued request and runs them as one batch -- after waiting (up to
// AIWC_BATCH_WINDOW_US, default 20000) until every caller served by the previous batch has
// queued again, so the threads of a tuning loop (one fit per step each) keep meeting in
// one batch per step; a caller that stops costs one window.  The others sleep until their
// request is done.  AIWC_FIT_BATCH=0 runs every fit alone.
void submit_fit(aiwc_ctx* ctx, aiwc_ctx::FitRequest& req) {
  static const bool batching = [] {
    const char* e = std::getenv("AIWC_FIT_BATCH");
    return !(e && std::atoi(e) == 0);
  }();
  static const auto window = std::chrono::microseconds([] {
    const char* e = std::getenv("AIWC_BATCH_WINDOW_US");
    return e ? std::atoll(e) : 20000ll;
  }());
  auto& q = ctx->q;
  std::unique_lock<std::mutex> lk(q.mu);
  q.pending.push_back(&req);
  if (q.returning) --q.returning;
  q.cv.notify_all();
  while (!req.done) {
    if (q.leader) {
      q.cv.wait(lk);
      continue;
    }
    q.leader = true;
    const auto tw = std::chrono::steady_clock::now();
    if (batching && q.returning &&
        !q.cv.wait_for(lk, window, [&] { return q.returning == 0; }))
      q.returning = 0;  // some caller stopped fitting
    const auto tw1 = std::chrono::steady_clock::now();
    std::vector<aiwc_ctx::FitRequest*> batch;
    if (batching) {
      batch.swap(q.pending);
    } else {  // one at a time, own request first
      batch.push_back(&req);
      q.pending.erase(std::find(q.pending.begin(), q.pending.end(), &req));
    }

    lk.unlock();
    fit_batch(ctx, batch);
    if (std::getenv("AIWC_VERBOSE"))
      std::fprintf(stderr, "[aiwc batch] %zu fits: waited %.2f ms, ran %.2f ms\n", batch.size(),
                   std::chrono::duration<double, std::milli>(tw1 - tw).count(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw1).count());
    lk.lock();
    for (auto* r : batch) r->done = true;
    if (batching) q.returning += batch.size();
    q.leader = false;
    q.cv.notify_all();
  }
  if (req.status != AIWC_OK) throw Status(req.status, req.msg);
}

}  // namespace

int aiwc_fit(aiwc_ctx* ctx, uint32_t num_trees, uint32_t mtry, uint32_t min_node_size,
             uint64_t seed, uint32_t tree_begin, uint32_t tree_end, int compute_oob,
             aiwc_forest** out) {
  return guard([&] {
    if (!ctx || !out) throw Status(AIWC_EARG, "NULL argument");
    // parameter checks of forest.hpp:482-490
    if (ctx->n < 2) throw Status(AIWC_EEXEC, "dataset must have at least 2 rows");
    if (num_trees < 1) throw Status(AIWC_EEXEC, "num_trees must be >= 1");
    if (min_node_size < 1) throw Status(AIWC_EEXEC, "min_node_size must be >= 1");
    if (mtry < 1 || mtry > ctx->p)
      throw Status(AIWC_EEXEC, "mtry must be in [1, " + std::to_string(ctx->p) + "], got " +
                                   std::to_string(mtry));
    if (tree_begin >= tree_end || tree_end > num_trees)
      throw Status(AIWC_EARG, "bad tree range");
    aiwc_ctx::FitRequest req{num_trees, mtry, min_node_size, tree_begin, tree_end, seed,
                             compute_oob};
    submit_fit(ctx, req);
    *out = req.out;
  });
}

int aiwc_fit_cells(aiwc_ctx* ctx, uint32_t ncells, const uint32_t* mtry,
                   const uint32_t* min_node_size, uint32_t num_trees, uint64_t seed,
                   aiwc_forest** out) {
  return guard([&] {
    if (!ctx || !out || !mtry || !min_node_size || ncells == 0) throw Status(AIWC_EARG, "bad argument");
    if (ctx->n < 2) throw Status(AIWC_EEXEC, "dataset must have at least 2 rows");
    if (num_trees < 1) throw Status(AIWC_EEXEC, "num_trees must be >= 1");
    if (uint64_t{ncells} * num_trees >= (uint64_t{1} << 31)) throw Status(AIWC_EARG, "too many trees");
    uint32_t mmax = 0, nmin = UINT32_MAX;
    for (uint32_t c = 0; c < ncells; ++c) {  // the checks of forest.hpp:482-490 per cell
      if (min_node_size[c] < 1) throw Status(AIWC_EEXEC, "min_node_size must be >= 1");
      if (mtry[c] < 1 || mtry[c] > ctx->p)
        throw Status(AIWC_EEXEC, "mtry must be in [1, " + std::to_string(ctx->p) + "], got " +
                                     std::to_string(mtry[c]));
      mmax = std::max(mmax, mtry[c]);
      nmin = std::min(nmin, min_node_size[c]);
    }
    const std::vector<uint64_t> seeds(ncells, seed);
    const std::vector<uint32_t> tb(ncells, 0u), te(ncells, num_trees);
    const CellSpec cs{ncells, mtry, min_node_size, seeds.data(), tb.data(), te.data()};
    fit_body(ctx, num_trees, mmax, nmin, seed, 0, ncells * num_trees, 0, &cs, out);
    (*out)->cells = ncells;
  });
}

int aiwc_forest_free(aiwc_forest* f) {
  if (!f) return AIWC_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(f->device);
  delete f;
  cudaSetDevice(prev);
  return AIWC_OK;
}

int aiwc_forest_info(const aiwc_forest* f, uint32_t* trees, uint64_t* total_nodes,
                     uint32_t* tree_begin) {
  return guard([&] {
    if (!f) throw Status(AIWC_EARG, "forest is NULL");
    if (trees) *trees = f->trees;
    if (total_nodes) *total_nodes = f->off.back();
    if (tree_begin) *tree_begin = f->tree_begin;
  });
}

int aiwc_forest_node_counts(const aiwc_forest* f, uint64_t* counts) {
  return guard([&] {
    if (!f || !counts) throw Status(AIWC_EARG, "NULL argument");
    for (uint32_t t = 0; t < f->trees; ++t) counts[t] = f->off[t + 1] - f->off[t];
  });
}

int aiwc_forest_export(const aiwc_forest* f, uint64_t* offsets, int32_t* feature,
                       double* threshold, int32_t* left, int32_t* right, double* value) {
  return guard([&] {
    if (!f) throw Status(AIWC_EARG, "forest is NULL");
    const uint64_t N = f->off.back();
    if (offsets) std::copy(f->off.begin(), f->off.end(), offsets);
    if (f->host_cached) {  // a batched fit's forest: the batch's pinned host copy
      if (feature) par_memcpy(reinterpret_cast<char*>(feature), reinterpret_cast<const char*>(f->h_feature), N * 4);
      if (threshold) par_memcpy(reinterpret_cast<char*>(threshold), reinterpret_cast<const char*>(f->h_thr), N * 8);
      if (left) par_memcpy(reinterpret_cast<char*>(left), reinterpret_cast<const char*>(f->h_left), N * 4);
      if (right)
        for (uint64_t i = 0; i < N; ++i) right[i] = f->h_left[i] < 0 ? -1 : f->h_left[i] + 1;
      if (value) par_memcpy(reinterpret_cast<char*>(value), reinterpret_cast<const char*>(f->h_value), N * 8);
      return;
    }
    DeviceGuard dg(f->device);
    Stream st;
    if (feature) d2h(feature, f->feature.p, N * 4, st.s);
    if (threshold) d2h(threshold, f->thr.p, N * 8, st.s);
    if (left) d2h(left, f->left.p, N * 4, st.s);
    if (right) {  // right = left + 1 (BFS numbering, forest.hpp:310-311), -1 for leaves
      DevBuf<int32_t> r(N);
      right_child_kernel<<<static_cast<unsigned>(std::min<uint64_t>((N + 255) / 256, 1u << 20)),
                           256, 0, st.s>>>(f->left.p, N, r.p);
      CK(cudaGetLastError());
      g_launches += 1;
      d2h(right, r.p, N * 4, st.s);
    }
    if (value) d2h(value, f->value.p, N * 8, st.s);
  });
}

int aiwc_forest_host_view(aiwc_forest* f, const int32_t** feature, const double** threshold,
                          const int32_t** left, const int32_t** right, const double** value,
                          const uint32_t** inbag) {
  return guard([&] {
    if (!f) throw Status(AIWC_EARG, "forest is NULL");
    std::lock_guard<std::mutex> lock(f->view_mu);
    const uint64_t N = f->off.back();
    const bool has_inbag = f->inbag.p != nullptr || (f->host_cached && f->h_inbag);
    const bool fit_mirror = f->inbag_pin.first != nullptr;  // filled during the fit
    const size_t ib = has_inbag && !fit_mirror ? size_t{f->trees} * f->n * 4 : 0;
    auto parts = [&](char* b) {
      double* t = reinterpret_cast<double*>(b);
      double* v = t + N;
      int32_t* fe = reinterpret_cast<int32_t*>(v + N);
      int32_t* le = fe + N;
      int32_t* ri = le + N;
      uint32_t* in = reinterpret_cast<uint32_t*>(ri + N + (N & 1));
      return std::make_tuple(t, v, fe, le, ri, in);
    };
    if (!f->view_pin.first) {
      const size_t bytes = N * 28 + (N & 1) * 4 + ib + 16;
      const auto t0 = std::chrono::steady_clock::now();
      auto pin = PinnedPool::take(bytes);
      const auto t1 = std::chrono::steady_clock::now();
      struct Mark {
        std::chrono::steady_clock::time_point t0, t1;
        ~Mark() {
          if (std::getenv("AIWC_PROFILE_PHASES"))
            std::fprintf(stderr, "[aiwc host_view] pinned take %.1f ms, copies %.1f ms\n",
                         std::chrono::duration<double, std::milli>(t1 - t0).count(),
                         std::chrono::duration<double, std::milli>(
                             std::chrono::steady_clock::now() - t1).count());
        }
      } mark{t0, t1};
      auto [t, v, fe, le, ri, in] = parts(pin.first);
      try {
        if (f->host_cached) {  // a batched fit's small forest: already on the host
          std::memcpy(t, f->h_thr, N * 8);
          std::memcpy(v, f->h_value, N * 8);
          std::memcpy(fe, f->h_feature, N * 4);
          std::memcpy(le, f->h_left, N * 4);
          for (uint64_t i = 0; i < N; ++i) ri[i] = le[i] < 0 ? -1 : le[i] + 1;
          if (ib) std::memcpy(in, f->h_inbag, ib);
        } else {
          DeviceGuard dg(f->device);
          Stream st;
          // right children written by the device straight into the mapped pinned mirror
          // (no 1.5 GB device temporary); the other arrays by DMA
          if (N) {
            right_child_kernel<<<static_cast<unsigned>(std::min<uint64_t>((N + 255) / 256, 1u << 20)),
                                 256, 0, st.s>>>(f->left.p, N, ri);
            CK(cudaGetLastError());
            g_launches += 1;
          }
          CK(cudaMemcpyAsync(t, f->thr.p, N * 8, cudaMemcpyDeviceToHost, st.s));
          CK(cudaMemcpyAsync(v, f->value.p, N * 8, cudaMemcpyDeviceToHost, st.s));
          CK(cudaMemcpyAsync(fe, f->feature.p, N * 4, cudaMemcpyDeviceToHost, st.s));
          CK(cudaMemcpyAsync(le, f->left.p, N * 4, cudaMemcpyDeviceToHost, st.s));
          if (ib) CK(cudaMemcpyAsync(in, f->inbag.p, ib, cudaMemcpyDeviceToHost, st.s));
          CK(cudaStreamSynchronize(st.s));
        }
      } catch (...) {
        PinnedPool::give(pin);
        throw;
      }
      f->view_pin = pin;
    }
    auto [t, v, fe, le, ri, in] = parts(f->view_pin.first);
    if (threshold) *threshold = t;
    if (value) *value = v;
    if (feature) *feature = fe;
    if (left) *left = le;
    if (right) *right = ri;
    if (inbag)
      *inbag = fit_mirror ? reinterpret_cast<const uint32_t*>(f->inbag_pin.first)
                          : (ib ? in : nullptr);
  });
}

int aiwc_forest_export_inbag(const aiwc_forest* f, uint32_t* inbag) {
  return guard([&] {
    if (!f || !inbag) throw Status(AIWC_EARG, "NULL argument");
    if (!f->inbag.p) throw Status(AIWC_EEXEC, "forest holds no in-bag lists");
    if (f->host_cached) {
      par_memcpy(reinterpret_cast<char*>(inbag), reinterpret_cast<const char*>(f->h_inbag),
                 size_t{f->trees} * f->n * 4);
      return;
    }
    DeviceGuard dg(f->device);
    Stream st;
    d2h(inbag, f->inbag.p, size_t{f->trees} * f->n * 4, st.s);
  });
}

int aiwc_forest_oob_stats(const aiwc_forest* f, aiwc_oob_stats* out) {
  return guard([&] {
    if (!f || !out) throw Status(AIWC_EARG, "NULL argument");
    if (!f->has_oob) throw Status(AIWC_EEXEC, "forest has no OOB statistics (partial range?)");
    *out = f->oob;
  });
}

int aiwc_forest_import(uint32_t trees, const uint64_t* offsets, const int32_t* feature,
                       const double* threshold, const int32_t* left, const int32_t* right,
                       const double* value, const uint32_t* inbag, uint64_t n, int device,
                       aiwc_forest** out) {
  return guard([&] {
    if (!offsets || !feature || !threshold || !left || !value || !out || trees < 1)
      throw Status(AIWC_EARG, "NULL argument or zero trees");
    DeviceGuard dg(device);
    auto f = std::make_unique<aiwc_forest>();
    f->device = device;
    f->n = n;
    f->trees = trees;
    f->num_trees = trees;
    f->off.assign(offsets, offsets + trees + 1);
    const uint64_t N = f->off[trees];
    std::vector<PredNode> pk(N);
    for (uint32_t t = 0; t < trees; ++t) {
      const uint64_t b = f->off[t], e = f->off[t + 1];
      if (e <= b) throw Status(AIWC_EPARSE, "empty tree in model");
      for (uint64_t i = b; i < e; ++i) {
        const int64_t cnt = static_cast<int64_t>(e - b);
        if (feature[i] >= 0) {
          // BFS layout: right == left + 1, children after their parent and inside the
          // tree (a back edge would make every walk of the tree loop forever)
          if (left[i] <= static_cast<int64_t>(i - b) || left[i] + 1 >= cnt ||
              (right && right[i] != left[i] + 1))
            throw Status(AIWC_EPARSE, "model tree is not in canonical BFS layout");
        }
        pk[i] = PredNode{feature[i] >= 0 ? threshold[i] : value[i], feature[i], left[i]};
      }
    }
    f->feature.alloc(N);
    f->left.alloc(N);
    f->thr.alloc(N);
    f->value.alloc(N);
    f->packed.alloc(N);
    f->d_off.alloc(trees + 1);
    CK(cudaMemcpy(f->feature.p, feature, N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f->left.p, left, N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f->thr.p, threshold, N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f->value.p, value, N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f->packed.p, pk.data(), N * sizeof(PredNode), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f->d_off.p, f->off.data(), (trees + 1) * 8, cudaMemcpyHostToDevice));
    if (inbag && n) {
      f->inbag.alloc(size_t{trees} * n);
      CK(cudaMemcpy(f->inbag.p, inbag, size_t{trees} * n * 4, cudaMemcpyHostToDevice));
    }
    *out = f.release();
  });
}

int aiwc_forest_export_device(const aiwc_forest* f, int32_t* d_feature, double* d_threshold,
                              int32_t* d_left, double* d_value, uint32_t* d_inbag) {
  return guard([&] {
    if (!f) throw Status(AIWC_EARG, "forest is NULL");
    if (d_inbag && !f->inbag.p) throw Status(AIWC_EEXEC, "forest holds no in-bag lists");
    DeviceGuard dg(f->device);
    const uint64_t N = f->off.back();
    Stream st;
    if (d_feature) CK(cudaMemcpyAsync(d_feature, f->feature.p, N * 4, cudaMemcpyDeviceToDevice, st.s));
    if (d_threshold) CK(cudaMemcpyAsync(d_threshold, f->thr.p, N * 8, cudaMemcpyDeviceToDevice, st.s));
    if (d_left) CK(cudaMemcpyAsync(d_left, f->left.p, N * 4, cudaMemcpyDeviceToDevice, st.s));
    if (d_value) CK(cudaMemcpyAsync(d_value, f->value.p, N * 8, cudaMemcpyDeviceToDevice, st.s));
    if (d_inbag)
      CK(cudaMemcpyAsync(d_inbag, f->inbag.p, size_t{f->trees} * f->n * 4,
                         cudaMemcpyDeviceToDevice, st.s));
    CK(cudaStreamSynchronize(st.s));
  });
}

int aiwc_forest_import_device(uint32_t trees, const uint64_t* offsets, const int32_t* d_feature,
                              const double* d_threshold, const int32_t* d_left,
                              const double* d_value, const uint32_t* d_inbag, uint64_t n,
                              int device, aiwc_forest** out) {
  return guard([&] {
    if (!offsets || !d_feature || !d_threshold || !d_left || !d_value || !out || trees < 1)
      throw Status(AIWC_EARG, "NULL argument or zero trees");
    DeviceGuard dg(device);
    auto f = std::make_unique<aiwc_forest>();
    f->device = device;
    f->n = n;
    f->trees = trees;
    f->num_trees = trees;
    f->off.assign(offsets, offsets + trees + 1);
    for (uint32_t t = 0; t < trees; ++t)
      if (f->off[t + 1] <= f->off[t]) throw Status(AIWC_EPARSE, "empty tree in model");
    const uint64_t N = f->off[trees];
    f->feature.alloc(N);
    f->left.alloc(N);
    f->thr.alloc(N);
    f->value.alloc(N);
    f->packed.alloc(N);
    f->d_off.alloc(trees + 1);
    Stream st;
    CK(cudaMemcpyAsync(f->feature.p, d_feature, N * 4, cudaMemcpyDeviceToDevice, st.s));
    CK(cudaMemcpyAsync(f->left.p, d_left, N * 4, cudaMemcpyDeviceToDevice, st.s));
    CK(cudaMemcpyAsync(f->thr.p, d_threshold, N * 8, cudaMemcpyDeviceToDevice, st.s));
    CK(cudaMemcpyAsync(f->value.p, d_value, N * 8, cudaMemcpyDeviceToDevice, st.s));
    CK(cudaMemcpyAsync(f->d_off.p, f->off.data(), (trees + 1) * 8, cudaMemcpyHostToDevice, st.s));
    DevBuf<uint32_t> bad(1);
    CK(cudaMemsetAsync(bad.p, 0, 4, st.s));
    pack_check_kernel<<<std::min<uint32_t>(trees, 148u * 16u), 256, 0, st.s>>>(
        f->d_off.p, trees, f->feature.p, f->thr.p, f->left.p, f->value.p, f->packed.p, bad.p);
    CK(cudaGetLastError());
    g_launches += 1;
    if (d_inbag && n) {
      f->inbag.alloc(size_t{trees} * n);
      CK(cudaMemcpyAsync(f->inbag.p, d_inbag, size_t{trees} * n * 4, cudaMemcpyDeviceToDevice,
                         st.s));
    }
    uint32_t h_bad = 0;
    CK(cudaMemcpyAsync(&h_bad, bad.p, 4, cudaMemcpyDeviceToHost, st.s));
    CK(cudaStreamSynchronize(st.s));
    if (h_bad) throw Status(AIWC_EPARSE, "model tree is not in canonical BFS layout");
    *out = f.release();
  });
}

int aiwc_oob(aiwc_ctx* ctx, aiwc_forest* f, aiwc_oob_stats* out, double* row_sum,
             uint32_t* row_count) {
  return guard([&] {
    if (!ctx || !f || !out) throw Status(AIWC_EARG, "NULL argument");
    if (f->n != ctx->n) throw Status(AIWC_ESCHEMA, "forest and dataset row counts differ");
    if (f->device != ctx->device) throw Status(AIWC_EARG, "forest and dataset live on different devices");
    if (!f->inbag.p) throw Status(AIWC_EEXEC, "forest holds no in-bag lists");
    DeviceGuard dg(ctx->device);
    Stream st;
    const uint64_t n = ctx->n;
    check_row_width(f, ctx->p, st.s);  // split columns must exist in this dataset
    // the leaves cached by the fit walked its training context; any other dataset (same
    // row count) is walked afresh, as oob_error(forest, data) does (forest.hpp:518-522)
    if (!f->oobleaf.p || f->oob_ctx != ctx->uid) {
      f->oobleaf.alloc(size_t{f->trees} * n);
      f->oob_ctx = ctx->uid;
      DevBuf<uint8_t> flags(size_t{f->trees} * n);
      CK(cudaMemsetAsync(flags.p, 0, size_t{f->trees} * n, st.s));
      ensure_packed(f, st.s);
      for (uint32_t t0 = 0; t0 < f->trees; t0 += 65535u) {  // gridDim.y <= 65,535
        const dim3 grid(static_cast<unsigned>((n + 255) / 256), std::min(65535u, f->trees - t0));
        inbag_flags_kernel<<<grid, 256, 0, st.s>>>(f->inbag.p, t0, n, flags.p);
        oob_walk_kernel<<<grid, 256, 0, st.s>>>(f->packed.p, f->d_off.p, flags.p, ctx->col.p, n,
                                                t0, f->oobleaf.p);
        CK(cudaGetLastError());
        g_launches += 2;
      }
      CK(cudaStreamSynchronize(st.s));
    }
    std::vector<double> sum(n, 0.0);
    std::vector<uint32_t> count(n, 0);
    oob_accumulate_device(f, sum.data(), count.data(), st.s);
    *out = finalize_oob(ctx->y.data(), n, sum.data(), count.data());
    if (row_sum) std::copy(sum.begin(), sum.end(), row_sum);
    if (row_count) std::copy(count.begin(), count.end(), row_count);
  });
}

int aiwc_oob_accumulate(aiwc_ctx* ctx, aiwc_forest* f, double* row_sum, uint32_t* row_count) {
  return guard([&] {
    if (!ctx || !f || !row_sum || !row_count) throw Status(AIWC_EARG, "NULL argument");
    if (!f->oobleaf.p) throw Status(AIWC_EEXEC, "forest holds no OOB leaf values");
    if (f->n != ctx->n) throw Status(AIWC_ESCHEMA, "forest and dataset row counts differ");
    DeviceGuard dg(ctx->device);
    Stream st;
    oob_accumulate_device(f, row_sum, row_count, st.s);
  });
}

int aiwc_oob_accumulate_device(aiwc_ctx* ctx, aiwc_forest* f, double* d_row_sum,
                               uint32_t* d_row_count) {
  return guard([&] {
    if (!ctx || !f || !d_row_sum || !d_row_count) throw Status(AIWC_EARG, "NULL argument");
    if (!f->oobleaf.p) throw Status(AIWC_EEXEC, "forest holds no OOB leaf values");
    if (f->n != ctx->n) throw Status(AIWC_ESCHEMA, "forest and dataset row counts differ");
    if (f->device != ctx->device) throw Status(AIWC_EARG, "forest and dataset live on different devices");
    DeviceGuard dg(ctx->device);
    Stream st;
    const uint64_t n = f->n;
    oob_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st.s>>>(
        f->oobleaf.p, f->d_off.p, f->value.p, f->trees, n, d_row_sum, d_row_count);
    CK(cudaGetLastError());
    g_launches += 1;
    CK(cudaStreamSynchronize(st.s));
  });
}

int aiwc_oob_prefix(aiwc_ctx* ctx, aiwc_forest* f, const uint32_t* tree_counts, uint32_t k,
                    aiwc_oob_stats* out) {
  return guard([&] {
    if (!ctx || !f || !tree_counts || !out) throw Status(AIWC_EARG, "NULL argument");
    if (!f->oobleaf.p) throw Status(AIWC_EEXEC, "forest holds no OOB leaf values");
    if (f->n != ctx->n) throw Status(AIWC_ESCHEMA, "forest and dataset row counts differ");
    if (f->tree_begin != 0) throw Status(AIWC_EARG, "tree prefixes need a forest from tree 0");
    for (uint32_t i = 0; i < k; ++i)
      if (tree_counts[i] < 1 || tree_counts[i] > f->trees || (i && tree_counts[i] < tree_counts[i - 1]))
        throw Status(AIWC_EARG, "tree counts must ascend within [1, trees]");
    if (k == 0) return;
    DeviceGuard dg(ctx->device);
    Stream st;
    const uint64_t n = f->n;
    DevBuf<uint32_t> cps(k);
    DevBuf<double> sums(size_t{k} * n);
    DevBuf<uint32_t> counts(size_t{k} * n);
    CK(cudaMemcpyAsync(cps.p, tree_counts, k * 4, cudaMemcpyHostToDevice, st.s));
    oob_prefix_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st.s>>>(
        f->oobleaf.p, f->d_off.p, f->value.p, cps.p, k, n, sums.p, counts.p);
    CK(cudaGetLastError());
    g_launches += 1;
    std::vector<double> hs(size_t{k} * n);
    std::vector<uint32_t> hc(size_t{k} * n);
    CK(cudaMemcpyAsync(hs.data(), sums.p, hs.size() * 8, cudaMemcpyDeviceToHost, st.s));
    CK(cudaMemcpyAsync(hc.data(), counts.p, hc.size() * 4, cudaMemcpyDeviceToHost, st.s));
    CK(cudaStreamSynchronize(st.s));
    for (uint32_t i = 0; i < k; ++i)
      out[i] = finalize_oob(ctx->y.data(), n, hs.data() + size_t{i} * n, hc.data() + size_t{i} * n);
  });
}

int aiwc_oob_prefix_cells(aiwc_ctx* ctx, aiwc_forest* f, const uint32_t* tree_counts,
                          uint32_t k, aiwc_oob_stats* out) {
  return guard([&] {
    if (!ctx || !f || !tree_counts || !out) throw Status(AIWC_EARG, "NULL argument");
    if (!f->oobleaf.p) throw Status(AIWC_EEXEC, "forest holds no OOB leaf values");
    if (f->n != ctx->n) throw Status(AIWC_ESCHEMA, "forest and dataset row counts differ");
    const uint32_t T = f->trees / f->cells;
    for (uint32_t i = 0; i < k; ++i)
      if (tree_counts[i] < 1 || tree_counts[i] > T || (i && tree_counts[i] < tree_counts[i - 1]))
        throw Status(AIWC_EARG, "tree counts must ascend within [1, trees per forest]");
    if (k == 0) return;
    DeviceGuard dg(ctx->device);
    Stream st;
    const uint64_t n = f->n;
    DevBuf<uint32_t> cps(k);
    DevBuf<double> sums(size_t{k} * n);
    DevBuf<uint32_t> counts(size_t{k} * n);
    CK(cudaMemcpyAsync(cps.p, tree_counts, k * 4, cudaMemcpyHostToDevice, st.s));
    std::vector<double> hs(size_t{k} * n);
    std::vector<uint32_t> hc(size_t{k} * n);
    for (uint32_t c = 0; c < f->cells; ++c) {  // forest c: trees [c*T, (c+1)*T)
      oob_prefix_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st.s>>>(
          f->oobleaf.p + size_t{c} * T * n, f->d_off.p + size_t{c} * T, f->value.p, cps.p, k, n,
          sums.p, counts.p);
      CK(cudaGetLastError());
      g_launches += 1;
      CK(cudaMemcpyAsync(hs.data(), sums.p, hs.size() * 8, cudaMemcpyDeviceToHost, st.s));
      CK(cudaMemcpyAsync(hc.data(), counts.p, hc.size() * 4, cudaMemcpyDeviceToHost, st.s));
      CK(cudaStreamSynchronize(st.s));
      for (uint32_t i = 0; i < k; ++i)
        out[size_t{c} * k + i] = finalize_oob(ctx->y.data(), n, hs.data() + size_t{i} * n,
                                              hc.data() + size_t{i} * n);
    }
  });
}

int aiwc_oob_finalize(const double* y, uint64_t n, const double* row_sum,
                      const uint32_t* row_count, aiwc_oob_stats* out) {
  return guard([&] {
    if (!y || !row_sum || !row_count || !out) throw Status(AIWC_EARG, "NULL argument");
    *out = finalize_oob(y, n, row_sum, row_count);
  });
}

}  // extern "C"

namespace {

constexpr int kPredNT = kPredictThreads;
constexpr uint64_t kSmallQ = 4096;  // up to this many rows predict without binning
constexpr size_t kPredSmem = 220 * 1024;  // per-CTA budget: chunk nodes+leaves + bin tile

// Build the binned copy: per column the sorted distinct thresholds the forest uses,
// per node its threshold bin, trees packed into shared-memory-sized chunks.
void build_binned(aiwc_forest* f, uint32_t p) {
  std::lock_guard<std::mutex> lock(f->bin_mu);
  if (f->bin_ready && f->bin_p == p) return;
  f->bin_ready = true;
  f->bin_p = p;
  f->bin_ok = false;
  const uint64_t N = f->off.back();
  std::vector<int32_t> fe(N), le(N);
  std::vector<double> th(N), va(N);
  CK(cudaMemcpy(fe.data(), f->feature.p, N * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(le.data(), f->left.p, N * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(th.data(), f->thr.p, N * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(va.data(), f->value.p, N * 8, cudaMemcpyDeviceToHost));
  std::vector<std::vector<double>> T(p);
  for (uint64_t i = 0; i < N; ++i) {
    if (fe[i] < 0) continue;
    if (static_cast<uint32_t>(fe[i]) >= p || fe[i] >= 0xffff) return;  // schema too wide
    T[fe[i]].push_back(th[i]);
  }
  size_t maxT = 0;
  std::vector<uint32_t> toff(p + 1, 0);
  for (uint32_t c = 0; c < p; ++c) {
    auto& v = T[c];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    maxT = std::max(maxT, v.size());
    toff[c + 1] = toff[c] + static_cast<uint32_t>(v.size());
  }
  if (maxT >= 0xffff) return;
  f->bin_bytes = maxT < 0xff ? 1 : 2;
  // one tile of warp-transposed bins (whole 32-query groups)
  const size_t tile = bin_words(uint64_t{kPredNT} * kPredictQ, p, f->bin_bytes) * 4;
  if (tile + 4096 > kPredSmem) return;
  const size_t budget = kPredSmem - tile - 64;
  // a split node names its column by the byte offset of its bin in the warp-transposed
  // bin words (forest_kernels.cu): column c -> (c / E) * 128 + (c % E) * bin_bytes
  const uint32_t E = 4 / f->bin_bytes;
  auto boff = [&](uint32_t c) { return (c / E) * 128u + (c % E) * f->bin_bytes; };
  if (boff(p - 1) >= 0xffffu) return;
  // packed 4-byte nodes: the offset in 12 bits (0xfff = leaf), bb bits for the largest
  // threshold index, the rest for chunk-relative child / leaf indices
  auto bits = [](uint64_t v) {
    uint32_t b = 1;
    while ((uint64_t{1} << b) <= v) ++b;
    return b;
  };
  const uint32_t bbits = bits(maxT ? maxT - 1 : 0);
  const uint32_t chbits = 12 + bbits < 32 ? 32 - 12 - bbits : 0;
  const uint64_t chmax = chbits >= 32 ? UINT32_MAX : (uint64_t{1} << chbits);
  const bool node4 = chbits >= 12 && boff(p - 1) < 0xfffu && std::getenv("AIWC_PRED_NODE8") == nullptr;
  f->fmt = PredFmt{12, bbits, 12 + bbits, 0xfffu, (1u << bbits) - 1u};
  const size_t nb = node4 ? 4 : sizeof(BinNode);
  std::vector<double> thr_all;
  for (auto& v : T) thr_all.insert(thr_all.end(), v.begin(), v.end());
  std::vector<BinNode> nodes;
  std::vector<double> leaves;
  std::vector<uint32_t> roots;
  f->chunks.clear();
  aiwc_forest::Chunk ch{0, 0, 0, 0, 0, 0};
  for (uint32_t t = 0; t < f->trees; ++t) {
    const uint64_t b = f->off[t], e = f->off[t + 1];
    uint32_t nl = 0;
    for (uint64_t i = b; i < e; ++i) nl += fe[i] < 0;
    const size_t need = (ch.nnodes + (e - b)) * nb + 32 + (ch.nleaves + nl) * 8;
    const bool idx_full = node4 && (ch.nnodes + (e - b) >= chmax || ch.nleaves + nl >= chmax);
    if (ch.ntrees > 0 && (need > budget || idx_full)) {
      f->chunks.push_back(ch);
      ch = aiwc_forest::Chunk{nodes.size(), leaves.size(), roots.size(), 0, 0, 0};
    }
    if ((e - b) * nb + 16 + nl * 8 > budget) return;  // one tree too big
    if (node4 && (e - b >= chmax || nl >= chmax)) return;
    roots.push_back(ch.nnodes);
    for (uint64_t i = b; i < e; ++i) {
      const uint32_t local = static_cast<uint32_t>(i - b) + ch.nnodes;
      (void)local;
      if (fe[i] < 0) {
        nodes.push_back(BinNode{0xffff, 0, ch.nleaves});
        leaves.push_back(va[i]);
        ++ch.nleaves;
      } else {
        const auto& v = T[fe[i]];
        const uint32_t j = static_cast<uint32_t>(std::lower_bound(v.begin(), v.end(), th[i]) - v.begin());
        nodes.push_back(BinNode{static_cast<uint16_t>(boff(static_cast<uint32_t>(fe[i]))),
                                static_cast<uint16_t>(j), ch.nnodes + static_cast<uint32_t>(le[i])});
      }
    }
    ch.nnodes += static_cast<uint32_t>(e - b);
    ++ch.ntrees;
  }
  f->chunks.push_back(ch);
  f->node_bytes = 8;
  if (node4) {
    std::vector<uint32_t> n4(nodes.size());
    bool ok = true;
    const PredFmt& fm = f->fmt;
    for (size_t i = 0; i < nodes.size(); ++i) {
      const BinNode& v = nodes[i];
      if (v.child >= chmax) ok = false;
      n4[i] = v.feat == 0xffff ? (fm.cmask | (v.child << fm.sh))
                               : (v.feat | (uint32_t{v.j} << fm.cb) | (v.child << fm.sh));
    }
    if (ok) {
      f->node_bytes = 4;
      f->bnodes4.alloc(n4.size());
      CK(cudaMemcpy(f->bnodes4.p, n4.data(), n4.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  if (f->node_bytes == 4 && !node4) return;
  if (node4 && f->node_bytes != 4) return;  // packed chunks were sized for 4-byte nodes
  f->bnodes.alloc(nodes.size());
  f->bleaves.alloc(leaves.size());
  f->broots.alloc(roots.size());
  f->bthr.alloc(std::max<size_t>(thr_all.size(), 1));
  f->bthr_off.alloc(toff.size());
  CK(cudaMemcpy(f->bnodes.p, nodes.data(), nodes.size() * sizeof(BinNode), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(f->bleaves.p, leaves.data(), leaves.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(f->broots.p, roots.data(), roots.size() * 4, cudaMemcpyHostToDevice));
  if (!thr_all.empty())
    CK(cudaMemcpy(f->bthr.p, thr_all.data(), thr_all.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(f->bthr_off.p, toff.data(), toff.size() * 4, cudaMemcpyHostToDevice));
  f->bin_ok = true;
}

// scratch of the binned path for up to q rows (bins + running sums); kernels using it
// must have finished before it is freed (DevBuf frees on the legacy stream)
struct PredScratch {
  DevBuf<uint32_t> bins;  // warp-transposed (bin_words)
  DevBuf<double> sum;
  void reserve(uint64_t q, uint32_t p) {
    const uint64_t w = bin_words(q, p, 2);
    if (bins.count < w) bins.alloc(w);
    if (sum.count < q) sum.alloc(q);
  }
};

void predict_binned(aiwc_forest* f, const double* d_rows, uint64_t q, uint32_t p, double* d_out,
                    cudaStream_t s, PredScratch& sc) {
  sc.reserve(q, p);
  uint32_t* const bins = sc.bins.p;
  double* const sum = sc.sum.p;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, f->device));
  CK(launch_bin_queries(f->bin_bytes, d_rows, q, p, f->bthr.p, f->bthr_off.p, bins, s));
  g_launches += 1;
  const uint64_t tq = uint64_t{kPredNT} * kPredictQ;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(sms, (q + tq - 1) / tq));
  for (size_t k = 0; k < f->chunks.size(); ++k) {
    const auto& ch = f->chunks[k];
    const size_t smem = ((size_t{ch.nnodes} * f->node_bytes + 15) & ~size_t{15}) +
                        ((size_t{ch.nleaves} * 8 + 15) & ~size_t{15}) +
                        bin_words(uint64_t{kPredNT} * kPredictQ, p, f->bin_bytes) * 4;
    const void* nodes = f->node_bytes == 4 ? static_cast<const void*>(f->bnodes4.p + ch.node0)
                                           : static_cast<const void*>(f->bnodes.p + ch.node0);
    CK(launch_predict_chunk(f->bin_bytes, f->node_bytes, nodes, ch.nnodes,
                            f->bleaves.p + ch.leaf0, ch.nleaves, f->broots.p + ch.root0, ch.ntrees,
                            bins, q, p, sum, k == 0, k + 1 == f->chunks.size(),
                            static_cast<double>(f->trees), d_out, grid, smem, kPredSmem, f->fmt,
                            s));
    g_launches += 1;
  }
}

void build_binned_once(aiwc_forest* f, uint32_t p) { build_binned(f, p); }

// device rows -> device responses; binned shared-memory path when the forest fits,
// else the L2 walk (predict_kernel)
// Query rows must hold every column the forest splits on (the reference guarantees it
// through Forest::check_schema / make_row, forest.hpp:88-115); narrower rows are a
// schema error instead of out-of-bounds reads.
void check_row_width(aiwc_forest* f, uint32_t p, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(f->mf_mu);
  if (f->max_feature == -2) {
    const uint64_t N = f->off.back();
    DevBuf<int32_t> d(1);
    CK(cudaMemsetAsync(d.p, 0xff, 4, s));  // -1
    max_feature_kernel<<<static_cast<unsigned>(std::min<uint64_t>((N + 255) / 256, 148u * 16u)),
                         256, 0, s>>>(f->feature.p, N, d.p);
    CK(cudaGetLastError());
    g_launches += 1;
    int32_t h = -1;
    CK(cudaMemcpyAsync(&h, d.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    f->max_feature = h;
  }
  if (f->max_feature >= 0 && static_cast<uint32_t>(f->max_feature) >= p)
    throw Status(AIWC_ESCHEMA, "query rows have " + std::to_string(p) +
                                   " columns but the forest splits on column " +
                                   std::to_string(f->max_feature));
}

void predict_dispatch(aiwc_forest* f, const double* d_rows, uint64_t q, uint32_t p,
                      double* d_out, cudaStream_t s, PredScratch& sc) {
  check_row_width(f, p, s);
  if (q <= kSmallQ && !f->bin_ready) {  // a handful of rows: no binned copy
    ensure_packed(f, s);
    predict_small_kernel<<<static_cast<unsigned>((q + 7) / 8), 256, 0, s>>>(
        f->packed.p, f->d_off.p, f->trees, d_rows, q, p, d_out);
    CK(cudaGetLastError());
    g_launches += 1;
    return;
  }
  build_binned(f, p);
  if (f->bin_ok) {
    predict_binned(f, d_rows, q, p, d_out, s, sc);
    return;
  }
  ensure_packed(f, s);
  predict_kernel<<<static_cast<unsigned>((q + 255) / 256), 256, 0, s>>>(f->packed.p, f->d_off.p,
                                                                        f->trees, d_rows, q, p, d_out);
  CK(cudaGetLastError());
  g_launches += 1;
}

}  // namespace

extern "C" {

int aiwc_predict_device(aiwc_forest* f, const double* d_rows, uint64_t q, uint32_t p,
                        double* d_out) {
  return guard([&] {
    if (!f || (!d_rows && q) || (!d_out && q)) throw Status(AIWC_EARG, "NULL argument");
    if (q == 0) return;
    DeviceGuard dg(f->device);
    Stream st;
    PredScratch sc;
    predict_dispatch(f, d_rows, q, p, d_out, st.s, sc);
    CK(cudaStreamSynchronize(st.s));  // before sc is freed
  });
}

int aiwc_predict(aiwc_forest* f, const double* rows, uint64_t q, uint32_t p,
                 double* out_response) {
  return guard([&] {
    if (!f || (!rows && q) || (!out_response && q)) throw Status(AIWC_EARG, "NULL argument");
    if (q == 0) return;
    DeviceGuard dg(f->device);
    if (q <= kSmallQ && !f->bin_ready) {  // a few rows: cached stream + buffers, no binning
      std::lock_guard<std::mutex> lock(f->sm_mu);
      if (!f->sm_stream) CK(cudaStreamCreateWithFlags(&f->sm_stream, cudaStreamNonBlocking));
      const cudaStream_t s = f->sm_stream;
      const size_t need = (q * p + q) * 8;
      if (f->sm_pin.second < need) {
        PinnedPool::give(f->sm_pin);
        f->sm_pin = PinnedPool::take(need);
      }
      double* const pin = reinterpret_cast<double*>(f->sm_pin.first);
      if (f->sm_rows.count < q * p) f->sm_rows.alloc(std::max<size_t>(q * p, 64 * size_t{p}));
      if (f->sm_out.count < q) f->sm_out.alloc(std::max<uint64_t>(q, 64));
      std::memcpy(pin, rows, q * p * 8);
      CK(cudaMemcpyAsync(f->sm_rows.p, pin, q * p * 8, cudaMemcpyHostToDevice, s));
      PredScratch none;
      predict_dispatch(f, f->sm_rows.p, q, p, f->sm_out.p, s, none);
      CK(cudaMemcpyAsync(pin + q * p, f->sm_out.p, q * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      std::memcpy(out_response, pin + q * p, q * 8);
      return;
    }
    // row chunks on two streams: the upload of chunk i+1 (host copy into pinned memory,
    // DMA) overlaps the predict kernels of chunk i
    Stream st[2];
    const uint64_t chunk = std::max<uint64_t>(uint64_t{1} << 20, (q + 7) / 8);
    PredScratch sc[2];
    DevBuf<double> dr[2], dout(q);
    dr[0].alloc(std::min(q, chunk) * p);
    if (q > chunk) dr[1].alloc(chunk * p);
    if (q > kSmallQ) build_binned_once(f, p);  // a handful of rows: predict_small_kernel
    uint64_t i = 0;
    for (uint64_t r0 = 0; r0 < q; r0 += chunk, ++i) {
      const uint64_t rn = std::min(chunk, q - r0);
      const cudaStream_t s = st[i & 1].s;
      CK(cudaStreamSynchronize(s));  // chunk i-2's kernels are done with dr[i&1]
      h2d(dr[i & 1].p, rows + r0 * p, rn * p * 8, s);
      predict_dispatch(f, dr[i & 1].p, rn, p, dout.p + r0, s, sc[i & 1]);
    }
    CK(cudaStreamSynchronize(st[0].s));
    CK(cudaStreamSynchronize(st[1].s));
    d2h(out_response, dout.p, q * 8, st[0].s);
  });
}

int aiwc_rank(aiwc_forest* f, const double* features, uint64_t q, uint32_t nfeat,
              uint32_t ndev, double* out_response, uint32_t* out_best) {
  return guard([&] {
    if (!f || (q && (!features || !out_best))) throw Status(AIWC_EARG, "NULL argument");
    if (nfeat < 1 || ndev < 1) throw Status(AIWC_EARG, "nfeat and ndev must be >= 1");
    if (q == 0) return;
    DeviceGuard dg(f->device);
    Stream st;
    DevBuf<double> dfeat(q * nfeat), dresp(q * ndev);
    DevBuf<uint32_t> dbest(q);
    DevBuf<uint8_t> dtie(q);
    h2d(dfeat.p, features, q * nfeat * 8, st.s);
    // chunks of <= 2M device rows: expand make_row in HBM, score with the predict path
    const uint32_t p = nfeat + ndev;
    const uint64_t cq = std::max<uint64_t>(1, (uint64_t{1} << 21) / ndev);
    DevBuf<double> drows(std::min(q, cq) * ndev * p);
    PredScratch sc;
    if (q * ndev > kSmallQ) build_binned_once(f, p);
    for (uint64_t i0 = 0; i0 < q; i0 += cq) {
      const uint64_t nq = std::min(cq, q - i0);
      expand_rows_kernel<<<static_cast<unsigned>(
                               std::min<uint64_t>((nq * ndev * p + 255) / 256, 148u * 32u)),
                           256, 0, st.s>>>(dfeat.p + i0 * nfeat, nq, nfeat, ndev, drows.p);
      CK(cudaGetLastError());
      g_launches += 1;
      predict_dispatch(f, drows.p, nq * ndev, p, dresp.p + i0 * ndev, st.s, sc);
    }
    rank_best_kernel<<<static_cast<unsigned>(std::min<uint64_t>((q + 255) / 256, 148u * 64u)),
                       256, 0, st.s>>>(dresp.p, q, ndev, dbest.p, dtie.p);
    CK(cudaGetLastError());
    g_launches += 1;
    std::vector<uint8_t> tie(q);
    d2h(out_best, dbest.p, q * 4, st.s);
    d2h(tie.data(), dtie.p, q, st.s);
    std::vector<double> resp_buf;
    double* resp = out_response;
    if (!resp) {
      resp_buf.resize(q * ndev);
      resp = resp_buf.data();
      bool any = false;
      for (uint64_t i = 0; i < q && !any; ++i) any = tie[i];
      if (!any) return;
    }
    d2h(resp, dresp.p, q * ndev * 8, st.s);
    // exact tie-break of flagged queries: min (10^r, device column), tools/main.cpp:340-345
    for (uint64_t i = 0; i < q; ++i) {
      if (!tie[i]) continue;
      const double* r = resp + i * ndev;
      uint32_t b = 0;
      double sb = std::pow(10.0, r[0]);
      for (uint32_t d = 1; d < ndev; ++d) {
        const double sd = std::pow(10.0, r[d]);
        if (sd < sb) {
          sb = sd;
          b = d;
        }
      }
      out_best[i] = b;
    }
  });
}

int aiwc_evaluate(const double* col, const double* y, uint64_t n, uint32_t p,
                  const uint32_t* kernel_of_row, uint32_t K, uint32_t num_trees,
                  uint32_t mtry, uint32_t min_node_size, uint64_t seed, int device,
                  double* predicted_seconds) {
  return aiwc_evaluate_folds(col, y, n, p, kernel_of_row, K, 0, K, num_trees, mtry,
                             min_node_size, seed, device, predicted_seconds);
}

int aiwc_evaluate_folds(const double* col, const double* y, uint64_t n, uint32_t p,
                        const uint32_t* kernel_of_row, uint32_t K, uint32_t fold_begin,
                        uint32_t fold_end, uint32_t num_trees, uint32_t mtry,
                        uint32_t min_node_size, uint64_t seed, int device,
                        double* predicted_seconds) {
  return guard([&] {
    if (!col || !y || !kernel_of_row || !predicted_seconds)
      throw Status(AIWC_EARG, "NULL argument");
    if (fold_begin > fold_end || fold_end > K) throw Status(AIWC_EARG, "fold range out of [0, K]");
    // Every fold trains on the table minus its kernel's rows (experiments.hpp:393-397),
    // i.e. on a row subset of ONE dataset: the folds' forests grow together as one
    // multi-forest launch over a single device copy of the table (one presort), each
    // fold's trees drawing their bootstrap from the fold's own training rows; the
    // held-out rows are then predicted by their fold's trees in tree order.
    std::vector<uint32_t> fk, nrows, rows;
    std::vector<uint64_t> roff{0};
    std::vector<std::vector<uint64_t>> tests;
    for (uint32_t k = fold_begin; k < fold_end; ++k) {
      std::vector<uint64_t> test;
      for (uint64_t i = 0; i < n; ++i)
        if (kernel_of_row[i] == k) test.push_back(i);
      if (test.empty()) continue;
      for (uint64_t i = 0; i < n; ++i)
        if (kernel_of_row[i] != k) rows.push_back(static_cast<uint32_t>(i));
      nrows.push_back(static_cast<uint32_t>(rows.size() - roff.back()));
      roff.push_back(rows.size());
      fk.push_back(k);
      tests.push_back(std::move(test));
    }
    if (fk.empty()) return;
    // the checks of forest.hpp:482-490 on every fold's training set
    for (uint32_t nk : nrows)
      if (nk < 2) throw Status(AIWC_EEXEC, "dataset must have at least 2 rows");
    if (num_trees < 1) throw Status(AIWC_EEXEC, "num_trees must be >= 1");
    if (min_node_size < 1) throw Status(AIWC_EEXEC, "min_node_size must be >= 1");
    if (mtry < 1 || mtry > p)
      throw Status(AIWC_EEXEC, "mtry must be in [1, " + std::to_string(p) + "], got " +
                                   std::to_string(mtry));
    aiwc_ctx* ctx = nullptr;
    {
      const int rc = aiwc_ctx_create(col, y, n, p, device, &ctx);
      if (rc) throw Status(rc, g_last_error);
    }
    struct CtxG {
      aiwc_ctx* c;
      ~CtxG() { aiwc_ctx_free(c); }
    } cg{ctx};
    // folds per launch: node pools of at most ~8 GB
    const double stride = 0.6322 * static_cast<double>(n) + 8.0 * std::sqrt(static_cast<double>(n)) + 64.0;
    const double tree_bytes = std::max(1024.0, stride) * 68.0;
    const uint64_t cap_trees = std::max<uint64_t>(num_trees, static_cast<uint64_t>(8e9 / tree_bytes));
    const uint32_t per_launch = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(
        fk.size(), std::min<uint64_t>(cap_trees / num_trees, ((uint64_t{1} << 31) - 1) / num_trees))));
    for (uint32_t g0 = 0; g0 < fk.size(); g0 += per_launch) {
      const uint32_t G = std::min<uint32_t>(per_launch, static_cast<uint32_t>(fk.size()) - g0);
      std::vector<uint32_t> vm(G, mtry), vn(G, min_node_size), vtb(G, 0u), vte(G, num_trees);
      std::vector<uint64_t> vs(G), off(G + 1);
      for (uint32_t c = 0; c < G; ++c) {
        vs[c] = host_derive_seed(seed, "holdout", fk[g0 + c]);
        off[c] = roff[g0 + c] - roff[g0];
      }
      off[G] = roff[g0 + G] - roff[g0];
      CellSpec cs{G, vm.data(), vn.data(), vs.data(), vtb.data(), vte.data()};
      cs.nrows = nrows.data() + g0;
      cs.rows = rows.data() + roff[g0];
      cs.rows_off = off.data();
      aiwc_forest* F = nullptr;
      fit_body(ctx, G * num_trees, mtry, min_node_size, vs[0], 0, G * num_trees, 0, &cs, &F);
      const std::unique_ptr<aiwc_forest, int (*)(aiwc_forest*)> fg(F, aiwc_forest_free);
      // held-out rows, grouped by fold, row-major (Dataset::predictor_row)
      std::vector<uint64_t> qoff(G + 1, 0);
      for (uint32_t c = 0; c < G; ++c) qoff[c + 1] = qoff[c] + tests[g0 + c].size();
      const uint64_t Q = qoff[G];
      std::vector<double> hrows(Q * p), resp(Q);
      for (uint32_t c = 0; c < G; ++c)
        for (uint64_t j = 0; j < tests[g0 + c].size(); ++j)
          for (uint32_t k = 0; k < p; ++k)
            hrows[(qoff[c] + j) * p + k] = col[size_t{k} * n + tests[g0 + c][j]];
      {
        std::lock_guard<std::mutex> lock(ctx->mu);
        DeviceGuard dg(ctx->device);
        const cudaStream_t st = ctx->stream;
        DevBuf<double> drows(Q * p), dout(Q);
        CK(cudaMemcpyAsync(drows.p, hrows.data(), Q * p * 8, cudaMemcpyHostToDevice, st));
        ensure_packed(F, st);
        for (uint32_t c = 0; c < G; ++c) {  // fold c: trees [c T, (c+1) T) of F
          const uint64_t q = qoff[c + 1] - qoff[c];
          predict_small_kernel<<<static_cast<unsigned>((q + 7) / 8), 256, 0, st>>>(
              F->packed.p, F->d_off.p + size_t{c} * num_trees, num_trees, drows.p + qoff[c] * p,
              q, p, dout.p + qoff[c]);
          CK(cudaGetLastError());
          g_launches += 1;
        }
        CK(cudaMemcpyAsync(resp.data(), dout.p, Q * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
      for (uint32_t c = 0; c < G; ++c)  // from_response, dataset.hpp:89-91
        for (uint64_t j = 0; j < tests[g0 + c].size(); ++j)
          predicted_seconds[tests[g0 + c][j]] = std::pow(10.0, resp[qoff[c] + j]);
    }
  });
}

uint64_t aiwc_launch_count(void) { return g_launches.load(); }

int aiwc_forest_profile(const aiwc_forest* f, double* grow_ms, double* fit_ms,
                        uint64_t* split_rows, uint32_t* grow_launches) {
  return guard([&] {
    if (!f) throw Status(AIWC_EARG, "forest is NULL");
    if (grow_ms) *grow_ms = f->grow_ms;
    if (fit_ms) *fit_ms = f->fit_ms;
    if (split_rows) *split_rows = f->split_rows;
    if (grow_launches) *grow_launches = f->grow_launches;
  });
}

int aiwc_make_queries(const double* d_rows, uint64_t n, uint32_t p, uint64_t q, uint64_t seed,
                      int device, double* d_out) {
  return guard([&] {
    if (!d_rows || !d_out || n == 0) throw Status(AIWC_EARG, "bad argument");
    DeviceGuard dg(device);
    Stream st;
    const uint64_t tag = host_fnv1a64("query", 5);
    const uint64_t total = q * p;
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 1u << 20));
    make_queries_kernel<<<blocks, 256, 0, st.s>>>(d_rows, n, p, q, seed, tag, d_out);
    CK(cudaGetLastError());
    g_launches += 1;
    CK(cudaStreamSynchronize(st.s));
  });
}

}  // extern "C"
