// host_io.hpp -- host <-> device transfer runtime of the C ABI's host-buffer
// entry points (pipedp_*_solve*).
//
// The reference's API takes and returns std::vector (pageable host memory).  A
// plain cudaMemcpy into pageable memory goes through the driver's own bounce
// buffer at a few GB/s; tables here are up to tens of GiB (config 5b: 32 GiB),
// so the transfer path is its own small runtime:
//   * a per-thread, per-device cache of device buffers (grow-only) so repeated
//     calls do not pay cudaMalloc/cudaFree;
//   * pinned staging buffers (two 64 MiB chunks per thread/device): DMA of chunk
//     i+1 overlaps the host-side copy of chunk i;
//   * the host-side copy of a chunk is split over a persistent worker pool, so
//     the pageable side (first-touch faults included) runs at memory bandwidth.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace pipedp_host {

// Persistent pool for parallel host memcpy (never runs any DP arithmetic).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool();  // never destroyed: its detached workers outlive main
    return *pool;
  }
  int size() const { return (int)workers_.size() + 1; }
  // run fn(i) for i in [0, n) on the pool and the caller; returns when all done
  void parallel_for(int n, const std::function<void(int)>& fn) {
    if (n <= 1 || workers_.empty()) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel_for at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      n_ = n;
      next_ = 0;
      pending_ = n;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = (int)std::min(16u, hw) - 1;
    for (int i = 0; i < nt; ++i) workers_.emplace_back([this] { loop(); });
    for (auto& t : workers_) t.detach();
  }
  void work() {
    for (;;) {
      int i;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (!fn_ || next_ >= n_) return;
        i = next_++;
        f = fn_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0, next_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
};

inline void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = 1u << 20;  // >= 1 MiB per thread; every pool thread busy from 16 MiB on
  const int pieces = (int)std::min<size_t>((bytes + kPiece - 1) / kPiece, (size_t)CopyPool::get().size());
  if (pieces <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes + pieces - 1) / pieces;
  CopyPool::get().parallel_for(pieces, [&](int i) {
    const size_t lo = (size_t)i * per, hi = std::min(bytes, lo + per);
    if (lo < hi) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  });
}

// Touch every page of a pageable destination (one write per 4 KiB, split over
// the pool) so the later copy does not take the first-touch faults; run while
// the kernel that produces the data is still executing.
inline void parallel_prefault(void* dst, size_t bytes) {
  // one piece per pool thread, in whole 2 MiB units (a transparent huge page
  // is faulted by one thread, never two at once), at least 2 MiB
  constexpr size_t kPage = 4096, kUnit = 2u << 20;
  const size_t threads = (size_t)CopyPool::get().size();
  const size_t piece = std::max(kUnit, ((bytes + threads - 1) / threads + kUnit - 1) / kUnit * kUnit);
  const int pieces = (int)((bytes + piece - 1) / piece);
  CopyPool::get().parallel_for(pieces, [&](int i) {
    char* p = static_cast<char*>(dst) + (size_t)i * piece;
    const size_t len = std::min(piece, bytes - (size_t)i * piece);
    for (size_t o = 0; o < len; o += kPage) reinterpret_cast<volatile char*>(p)[o] = 0;
  });
}

// memset split over the pool (a large host flag array written while the
// kernels run)
inline void parallel_fill(void* dst, int value, size_t bytes) {
  constexpr size_t kPiece = 4u << 20;
  const int pieces = (int)((bytes + kPiece - 1) / kPiece);
  if (pieces <= 1) {
    std::memset(dst, value, bytes);
    return;
  }
  CopyPool::get().parallel_for(pieces, [&](int i) {
    const size_t lo = (size_t)i * kPiece;
    std::memset(static_cast<char*>(dst) + lo, value, std::min(kPiece, bytes - lo));
  });
}

// dst[i] = src[i] widened, split over the pool (the host half of a narrowed
// device -> host copy).
inline void parallel_widen(int64_t* dst, const int32_t* src, size_t count) {
  constexpr size_t kSlice = 32u << 10;  // values per slice (128 KiB of int32): a few MiB already spread over the pool
  const int pieces = (int)std::min<size_t>((count + kSlice - 1) / kSlice, (size_t)CopyPool::get().size());
  if (pieces <= 1) {
    for (size_t i = 0; i < count; ++i) dst[i] = src[i];
    return;
  }
  const size_t per = (count + pieces - 1) / pieces;
  CopyPool::get().parallel_for(pieces, [&](int i) {
    const size_t lo = (size_t)i * per, hi = std::min(count, lo + per);
    for (size_t j = lo; j < hi; ++j) dst[j] = src[j];
  });
}

// dst[i] = table[src[i]]: 16-bit ranks back to their int64 values
inline void parallel_lookup16(int64_t* dst, const uint16_t* src, size_t count, const int64_t* table) {
  constexpr size_t kSlice = 64u << 10;
  const int pieces = (int)std::min<size_t>((count + kSlice - 1) / kSlice, (size_t)CopyPool::get().size());
  if (pieces <= 1) {
    for (size_t i = 0; i < count; ++i) dst[i] = table[src[i]];
    return;
  }
  const size_t per = (count + pieces - 1) / pieces;
  CopyPool::get().parallel_for(pieces, [&](int i) {
    const size_t lo = (size_t)i * per, hi = std::min(count, lo + per);
    for (size_t j = lo; j < hi; ++j) dst[j] = table[src[j]];
  });
}

// Per-thread, per-device transfer workspace.
struct Workspace {
  static constexpr size_t kChunk = 64u << 20;
  int device = -1;
  cudaStream_t stream = nullptr;
  void* pinned[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  Buf bufs[6];

  cudaError_t init(int dev) {
    device = dev;
    cudaError_t e = cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaHostAlloc(&pinned[i], kChunk, cudaHostAllocDefault);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    }
    return e;
  }
  // device buffer `slot` with at least `bytes` (contents not preserved)
  cudaError_t buffer(int slot, size_t bytes, void** out) {
    Buf& b = bufs[slot];
    if (b.cap < bytes) {
      if (b.p) cudaFree(b.p);
      b.p = nullptr;
      b.cap = 0;
      cudaError_t e = cudaMalloc(&b.p, std::max<size_t>(bytes, 256));
      if (e != cudaSuccess) return e;
      b.cap = std::max<size_t>(bytes, 256);
    }
    *out = b.p;
    return cudaSuccess;
  }
  // pageable host -> device, staged and double-buffered; asynchronous w.r.t.
  // the device work queued after it on `stream` (returns once the host side is read)
  cudaError_t h2d(void* dst, const void* src, size_t bytes) {
    size_t off = 0;
    int i = 0;
    while (off < bytes) {
      const size_t len = std::min(kChunk, bytes - off);
      const int s = i & 1;
      cudaError_t e = cudaEventSynchronize(ev[s]);  // buffer s free again
      if (e != cudaSuccess) return e;
      parallel_memcpy(pinned[s], static_cast<const char*>(src) + off, len);
      e = cudaMemcpyAsync(static_cast<char*>(dst) + off, pinned[s], len, cudaMemcpyHostToDevice, stream);
      if (e == cudaSuccess) e = cudaEventRecord(ev[s], stream);
      if (e != cudaSuccess) return e;
      off += len;
      ++i;
    }
    return cudaSuccess;
  }
  // Device -> pageable host copy of a table that a running kernel is still
  // producing front to back.  `progress(&ready)` reports how many leading
  // bytes are final (it may itself issue small copies on `side`); chunks are
  // copied out as soon as they are final, so only the tail is left when the
  // kernel ends.  `done` is recorded on `stream` after the kernel: once it has
  // completed everything is final.  Synchronous.
  template <class Progress>
  cudaError_t d2h_streamed(void* dst, const void* src, size_t bytes, cudaEvent_t done, Progress progress) {
    constexpr size_t kPiece = 16u << 20;
    if (!side) {
      cudaError_t e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
    }
    const size_t nchunks = (bytes + kPiece - 1) / kPiece;
    size_t ready = 0, issued = 0, drained = 0;
    bool finished = false;
    static const bool trace = getenv("PIPEDP_TRACE_D2H") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
    long polls = 0;
    cudaEvent_t* evs = ev;
    auto drain = [&](size_t c) {  // chunk c: wait for its DMA, copy it out of pinned
      cudaError_t e = cudaEventSynchronize(evs[c & 1]);
      if (e != cudaSuccess) return e;
      const size_t off = c * kPiece, len = std::min(kPiece, bytes - off);
      parallel_memcpy(static_cast<char*>(dst) + off, pinned[c & 1], len);
      return cudaSuccess;
    };
    while (drained < nchunks) {
      // issue every final chunk that has a free pinned slot
      while (issued < nchunks && issued < drained + 2) {
        const size_t off = issued * kPiece, len = std::min(kPiece, bytes - off);
        if (!finished && ready < off + len) break;
        cudaError_t e = cudaMemcpyAsync(pinned[issued & 1], static_cast<const char*>(src) + off, len,
                                        cudaMemcpyDeviceToHost, side);
        if (e == cudaSuccess) e = cudaEventRecord(evs[issued & 1], side);
        if (e != cudaSuccess) return e;
        if (trace) fprintf(stderr, "d2h chunk %zu issued at %.2f ms (ready %zu MiB, finished %d, polls %ld)\n", issued,
                           ms(), ready >> 20, (int)finished, polls);
        ++issued;
      }
      if (drained < issued) {
        cudaError_t e = drain(drained++);
        if (e != cudaSuccess) return e;
        continue;
      }
      // nothing in flight: learn more progress
      if (!finished) {
        cudaError_t q = cudaEventQuery(done);
        if (q == cudaSuccess) {
          finished = true;
        } else if (q != cudaErrorNotReady) {
          return q;
        } else {
          const size_t before = ready;
          cudaError_t e = progress(&ready);
          ++polls;
          if (e != cudaSuccess) return e;
          // no new chunk final yet: back off (each poll is a device read the
          // running kernel's counters see as traffic)
          if (ready == before || ready < std::min(bytes, (issued + 1) * kPiece))
            std::this_thread::sleep_for(std::chrono::microseconds(200));
        }
      }
    }
    if (trace) fprintf(stderr, "d2h done at %.2f ms\n", ms());
    return cudaStreamSynchronize(stream);
  }
  cudaStream_t side = nullptr;  // second copy stream (d2h_streamed)
  unsigned long long* ctr = nullptr;  // pinned scratch for progress counters (8 words)
  cudaEvent_t armed = nullptr, done = nullptr;
  cudaError_t streaming_init() {
    cudaError_t e = cudaSuccess;
    if (!ctr) e = cudaHostAlloc(reinterpret_cast<void**>(&ctr), 64, cudaHostAllocDefault);
    if (e == cudaSuccess && !armed) e = cudaEventCreateWithFlags(&armed, cudaEventDisableTiming);
    if (e == cudaSuccess && !done) e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    if (e == cudaSuccess && !side) e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    return e;
  }

  // int64 host table from an int32 device copy (values proven to fit int32):
  // half the PCIe bytes, widened on the host while the next piece is in flight.
  cudaError_t d2h_widen(int64_t* dst, const int32_t* src, size_t count, cudaStream_t st = nullptr) {
    if (!st) st = stream;
    // pieces of 16 MiB of int32: the DMA of piece i+1 overlaps the widening of
    // piece i (the host side is the slower leg)
    static const size_t piece_bytes = std::min<size_t>(kChunk, size_t(16) << 20);
    const size_t per = piece_bytes / sizeof(int32_t);
    const size_t nchunks = (count + per - 1) / per;
    auto issue = [&](size_t c) {
      const size_t off = c * per, len = std::min(per, count - off);
      cudaError_t e = cudaMemcpyAsync(pinned[c & 1], src + off, len * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
      return e == cudaSuccess ? cudaEventRecord(ev[c & 1], st) : e;
    };
    if (nchunks == 0) return cudaStreamSynchronize(st);
    cudaError_t e = issue(0);
    for (size_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
      if (c + 1 < nchunks) e = issue(c + 1);
      if (e == cudaSuccess) e = cudaEventSynchronize(ev[c & 1]);
      if (e != cudaSuccess) break;
      const size_t off = c * per, len = std::min(per, count - off);
      parallel_widen(dst + off, static_cast<const int32_t*>(pinned[c & 1]), len);
    }
    return e;
  }

  // int64 host table from a device array of 16-bit ranks into `table`
  // (chunked min / max: every value is an init value) -- a quarter of the
  // PCIe bytes; pieces of 16 MiB, the DMA of piece i+1 overlapping the lookup of piece i
  cudaError_t d2h_lookup16(int64_t* dst, const uint16_t* src, size_t count, const int64_t* table,
                           cudaStream_t st = nullptr) {
    if (!st) st = stream;
    const size_t per = (size_t(16) << 20) / sizeof(uint16_t);
    const size_t nchunks = (count + per - 1) / per;
    auto issue = [&](size_t c) {
      const size_t off = c * per, len = std::min(per, count - off);
      cudaError_t e = cudaMemcpyAsync(pinned[c & 1], src + off, len * sizeof(uint16_t), cudaMemcpyDeviceToHost, st);
      return e == cudaSuccess ? cudaEventRecord(ev[c & 1], st) : e;
    };
    if (nchunks == 0) return cudaStreamSynchronize(st);
    cudaError_t e = issue(0);
    for (size_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
      if (c + 1 < nchunks) e = issue(c + 1);
      if (e == cudaSuccess) e = cudaEventSynchronize(ev[c & 1]);
      if (e != cudaSuccess) break;
      const size_t off = c * per, len = std::min(per, count - off);
      parallel_lookup16(dst + off, static_cast<const uint16_t*>(pinned[c & 1]), len, table);
    }
    return e;
  }

  // Mapped pinned words the device publishes progress into (grow-only).
  unsigned long long* prog_h = nullptr;
  unsigned long long* prog_d = nullptr;
  size_t prog_cap = 0;
  uint32_t prog_epoch = 0;
  cudaError_t progress_words(size_t count) {
    if (prog_cap >= count) return cudaSuccess;
    if (prog_h) cudaFreeHost(prog_h);
    prog_h = prog_d = nullptr;
    prog_cap = 0;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&prog_h), sizeof(unsigned long long) * count,
                                  cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&prog_d), prog_h, 0);
    if (e != cudaSuccess) return e;
    memset(prog_h, 0, sizeof(unsigned long long) * count);
    prog_cap = count;
    return cudaSuccess;
  }

  // Chunked min / max solve, ranks leaving the device while the chunks still
  // run.  Chunk g owns cells [a1 + g L, a1 + (g+1) L) of d_rank (the last one
  // ragged at n) and publishes (epoch << 32 | cells final) in prog_h[g]; the
  // cells every chunk has finished form a column band [lo, hi) of the G x L
  // view, copied by one strided DMA on `side` and turned into int64 values by
  // the pool (dst[c] = table[rank]) while the next band is in flight.  After
  // `done` (the launch's completion) the rest goes the same way.
  cudaError_t d2h_lookup16_chunks(int64_t* dst, const uint16_t* d_rank, int64_t a1, int64_t n, int64_t G, int64_t L,
                                  const int64_t* table, uint32_t epoch, cudaEvent_t done) {
    constexpr int64_t kMinBand = 4096;  // one publication step
    const int64_t max_band = std::max<int64_t>(1, (int64_t)(kChunk / (sizeof(uint16_t) * G)));
    const volatile unsigned long long* prog = prog_h;
    auto ready = [&]() -> int64_t {
      int64_t m = L;
      for (int64_t g = 0; g < G && m > 0; ++g) {
        const unsigned long long v = prog[g];
        const int64_t len = std::min(L, n - a1 - g * L);
        int64_t d = (uint32_t)(v >> 32) == epoch ? (int64_t)(v & 0xffffffffu) : 0;
        if (d >= len) d = L;
        m = std::min(m, d);
      }
      return m;
    };
    static const bool trace = getenv("PIPEDP_TRACE_D2H") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
    int64_t band[2][2] = {{0, 0}, {0, 0}};
    int64_t lo = 0;
    size_t issued = 0, drained = 0;
    bool fin = false;
    for (;;) {
      if (!fin) {
        const cudaError_t q = cudaEventQuery(done);
        if (q == cudaSuccess) fin = true;
        else if (q != cudaErrorNotReady) return q;
      }
      if (issued - drained < 2 && lo < L) {
        const int64_t hi = std::min(fin ? L : ready(), lo + max_band);
        if (hi > lo && (fin || hi == L || hi - lo >= kMinBand)) {
          const int sl = (int)(issued & 1);
          const size_t w = sizeof(uint16_t) * (size_t)(hi - lo);
          cudaError_t e = cudaMemcpy2DAsync(pinned[sl], w, d_rank + a1 + lo, sizeof(uint16_t) * (size_t)L, w,
                                            (size_t)G, cudaMemcpyDeviceToHost, side);
          if (e == cudaSuccess) e = cudaEventRecord(ev[sl], side);
          if (e != cudaSuccess) return e;
          if (trace) fprintf(stderr, "band [%lld, %lld) issued at %.3f ms (fin %d)\n", (long long)lo, (long long)hi, ms(), (int)fin);
          band[sl][0] = lo;
          band[sl][1] = hi;
          lo = hi;
          ++issued;
          continue;
        }
      }
      if (drained < issued) {
        const int sl = (int)(drained & 1);
        cudaError_t e = cudaEventSynchronize(ev[sl]);
        if (e != cudaSuccess) return e;
        const int64_t b0 = band[sl][0], w = band[sl][1] - b0;
        const uint16_t* src = static_cast<const uint16_t*>(pinned[sl]);
        const int pieces = (int)std::min<int64_t>(G, CopyPool::get().size());
        const int64_t per = (G + pieces - 1) / pieces;
        CopyPool::get().parallel_for(pieces, [&](int i) {
          for (int64_t g = i * per; g < std::min(G, (i + 1) * per); ++g) {
            const int64_t c0 = a1 + g * L + b0, cnt = std::min(w, n - c0);
            const uint16_t* r = src + g * w;
            int64_t* o = dst + c0;
            for (int64_t j = 0; j < cnt; ++j) o[j] = table[r[j]];
          }
        });
        if (trace) fprintf(stderr, "band [%lld, %lld) converted at %.3f ms\n", (long long)b0, (long long)(b0 + w), ms());
        ++drained;
        continue;
      }
      if (fin && lo >= L) return cudaSuccess;
      std::this_thread::yield();
    }
  }

  // device -> pageable host after the work queued on `stream`; synchronous
  cudaError_t d2h(void* dst, const void* src, size_t bytes) {
    // pieces of the whole 64 MiB staging buffer (smaller pieces measured
    // slower: per-call pool overhead outweighs the overlap)
    static const size_t piece = kChunk;
    const size_t nchunks = (bytes + piece - 1) / piece;
    auto issue = [&](size_t c) {
      const size_t off = c * piece, len = std::min(piece, bytes - off);
      cudaError_t e = cudaMemcpyAsync(pinned[c & 1], static_cast<const char*>(src) + off, len,
                                      cudaMemcpyDeviceToHost, stream);
      return e == cudaSuccess ? cudaEventRecord(ev[c & 1], stream) : e;
    };
    if (nchunks == 0) return cudaStreamSynchronize(stream);
    static const bool trace = getenv("PIPEDP_TRACE_D2H") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
    cudaError_t e = issue(0);
    for (size_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
      if (c + 1 < nchunks) e = issue(c + 1);  // overlaps the host copy of chunk c
      if (e == cudaSuccess) e = cudaEventSynchronize(ev[c & 1]);
      if (e != cudaSuccess) break;
      const double tw = trace ? ms() : 0;
      const size_t off = c * piece, len = std::min(piece, bytes - off);
      parallel_memcpy(static_cast<char*>(dst) + off, pinned[c & 1], len);
      if (trace) fprintf(stderr, "d2h piece %zu: ready at %.2f ms, host copy %.2f ms\n", c, tw, ms() - tw);
    }
    return e;
  }
};

// The calling thread's workspace for `device` (created on first use).
inline cudaError_t workspace(int device, Workspace** out) {
  thread_local std::vector<Workspace*> spaces;
  for (Workspace* w : spaces)
    if (w->device == device) {
      *out = w;
      return cudaSuccess;
    }
  auto* w = new Workspace();
  cudaError_t e = w->init(device);
  if (e != cudaSuccess) {
    delete w;  // partial resources are reclaimed at process exit
    return e;
  }
  spaces.push_back(w);
  *out = w;
  return cudaSuccess;
}

}  // namespace pipedp_host
