// Host staging packer (tp_stage_pack): caller HWC images -> one pinned payload.
//
// The reference stages a request's buffers into its arena with one numpy copy per
// buffer on the calling thread (transfer.py:211-233, pack). On the B200 path that copy
// is the host half of the end-to-end critical path: a 64 x 1080p batch is 398 MB, and
// one thread copies it at ~8-10 GB/s, well under the ~55 GB/s the H2D link takes. This
// packer splits the batch into ~1 MB row chunks and copies them on a persistent pool of
// host threads, so the packing of batch i+1 keeps pace with the upload of batch i.
// With a row map (touched-row staging, tp_touched_rows) only the rows K2's stencil
// reads are copied, each to its compact slot; columns are always copied whole (a
// column gather would move 3-byte runs and saves 3% of a 1080p image).
//
// Host code only (compiled by nvcc's host compiler); no CUDA calls.

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <immintrin.h>
#include <sched.h>
#include <unistd.h>

#include "tileprep.h"
#include "tp_common.cuh"

namespace {

// A fixed pool of worker threads running one parallel-for at a time. Workers are
// created on first use and re-created after a fork (a forked child has none).
class Pool {
 public:
  static Pool& get() {
    static Pool* p = new Pool;  // never destroyed: joinable workers must not be torn down at exit
    return *p;
  }

  int size() {
    std::lock_guard<std::mutex> g(run_mu_);
    ensure();
    return static_cast<int>(workers_.size()) + 1;
  }

  // fn(task) for task in [0, n_tasks) on at most `threads` threads (the caller is one)
  void run(int64_t n_tasks, int threads, const std::function<void(int64_t)>& fn) {
    std::lock_guard<std::mutex> g(run_mu_);  // one parallel-for at a time
    ensure();
    const int helpers = std::max(0, std::min<int>(threads - 1, static_cast<int>(workers_.size())));
    next_.store(0);
    {
      std::lock_guard<std::mutex> l(mu_);
      fn_ = &fn;
      n_tasks_ = n_tasks;
      helpers_ = helpers;
      active_ = helpers;
      ++epoch_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> l(mu_);
    done_cv_.wait(l, [&] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  Pool() = default;

  void ensure() {
    const pid_t pid = getpid();
    if (pid == pid_ && !workers_.empty()) return;
    if (pid != pid_) {  // after fork: the parent's threads do not exist here
      for (auto& t : workers_) t.detach();
      workers_.clear();
      pid_ = pid;
    }
    cpu_set_t set;
    int cores = 0;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) cores = CPU_COUNT(&set);
    if (cores <= 0) cores = static_cast<int>(std::thread::hardware_concurrency());
    const int n = cores > 1 ? cores - 1 : 1;
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
  }

  void drain() {
    for (;;) {
      const int64_t t = next_.fetch_add(1);
      if (t >= n_tasks_) break;
      (*fn_)(t);
    }
  }

  void loop(int index) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return epoch_ != seen; });
        seen = epoch_;
        if (index >= helpers_) continue;  // not needed for this run
      }
      drain();
      std::lock_guard<std::mutex> l(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }

  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> workers_;
  pid_t pid_ = 0;
  uint64_t epoch_ = 0;
  const std::function<void(int64_t)>* fn_ = nullptr;
  int64_t n_tasks_ = 0;
  int helpers_ = 0, active_ = 0;
  std::atomic<int64_t> next_{0};
};

// Copy with non-temporal (streaming) stores: the staging slab is read next by the copy
// engine's DMA, not by this CPU, so writing around the caches saves the read-for-
// ownership of every destination line (a third of the memory traffic of a cached copy)
// and leaves the caller's data in cache.  AVX2 when the CPU has it, memcpy otherwise.
__attribute__((target("avx2"))) void copy_nt_avx2(uint8_t* dst, const uint8_t* src, size_t n) {
  size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  const size_t m = n & ~size_t(127);
  for (size_t i = 0; i < m; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  std::memcpy(dst + m, src + m, n - m);
}

bool have_avx2() {
  static const bool v = __builtin_cpu_supports("avx2");
  return v;
}

inline void copy_block(uint8_t* dst, const uint8_t* src, size_t n, bool nt) {
  if (nt) copy_nt_avx2(dst, src, n);
  else std::memcpy(dst, src, n);
}

struct Chunk {
  int32_t image;
  int32_t y0, y1;  // source rows [y0, y1)
};

constexpr int64_t kChunkBytes = 1 << 20;

}  // namespace

extern "C" {

TP_API int32_t tp_host_threads(void) { return Pool::get().size(); }

TP_API int tp_stage_pack(int32_t n, const uint8_t* const* src, const int64_t* src_stride,
                         const int32_t* wh, int32_t channels, const int32_t* row_map,
                         const int64_t* row_map_off, uint8_t* dst, const int64_t* dst_off,
                         int32_t threads) {
  if (n < 0 || (n > 0 && (!src || !src_stride || !wh || !dst || !dst_off)) || channels < 1 ||
      channels > 4 || (row_map && !row_map_off))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_stage_pack: bad arguments");
  std::vector<Chunk> chunks;
  for (int32_t k = 0; k < n; ++k) {
    const int64_t w = wh[2 * k], h = wh[2 * k + 1];
    if (w < 1 || h < 1 || !src[k] || src_stride[k] < w * channels)
      return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_stage_pack: image %d: bad size/stride", k);
    const int64_t row = w * channels;
    const int32_t rows_per = static_cast<int32_t>(std::max<int64_t>(1, kChunkBytes / row));
    for (int64_t y = 0; y < h; y += rows_per)
      chunks.push_back({k, static_cast<int32_t>(y), static_cast<int32_t>(std::min<int64_t>(h, y + rows_per))});
  }
  const int nthreads = threads > 0 ? threads : Pool::get().size();
  const bool nt = have_avx2() && getenv("TP_PACK_NO_NT") == nullptr;
  std::function<void(int64_t)> fn = [&](int64_t t) {
    const Chunk& c = chunks[static_cast<size_t>(t)];
    const int64_t w = wh[2 * c.image];
    const int64_t row = w * channels;
    const uint8_t* s = src[c.image];
    uint8_t* d = dst + dst_off[c.image];
    const int64_t st = src_stride[c.image];
    if (row_map) {
      const int32_t* m = row_map + row_map_off[c.image] + 1;  // m[y]: compact row or -1
      // runs of consecutive staged rows are one copy
      int32_t y = c.y0;
      while (y < c.y1) {
        if (m[y] < 0) {
          ++y;
          continue;
        }
        int32_t e = y + 1;
        while (e < c.y1 && m[e] == m[e - 1] + 1) ++e;
        if (st == row)
          copy_block(d + static_cast<int64_t>(m[y]) * row, s + y * st, static_cast<size_t>(e - y) * row, nt);
        else
          for (int32_t yy = y; yy < e; ++yy)
            copy_block(d + static_cast<int64_t>(m[yy]) * row, s + yy * st, row, nt);
        y = e;
      }
    } else if (st == row) {
      copy_block(d + c.y0 * row, s + c.y0 * st, (c.y1 - c.y0) * row, nt);
    } else {
      for (int32_t y = c.y0; y < c.y1; ++y) copy_block(d + y * row, s + y * st, row, nt);
    }
    if (nt) _mm_sfence();  // streaming stores visible before the caller uploads the slab
  };
  if (nthreads <= 1 || chunks.size() <= 1) {
    for (size_t t = 0; t < chunks.size(); ++t) fn(static_cast<int64_t>(t));
  } else {
    Pool::get().run(static_cast<int64_t>(chunks.size()), nthreads, fn);
  }
  return TP_OK;
}

}  // extern "C"
