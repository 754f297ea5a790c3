// Host <-> device copies of the caller's field arrays at pinned-DMA speed (see hostio.cuh).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hostio.cuh"
#include "system.cuh"

namespace tlsph_cuda {
namespace {

constexpr size_t kPiece = size_t(8) << 20;  // pinned bytes per ring slot (largest pipeline piece)
constexpr int kRing = 3;                    // pinned pieces in flight
constexpr size_t kDirect = size_t(1) << 20; // below this the driver's own staged copy is as fast

// A fixed team of host threads splitting one memcpy (the copy rate of a single thread, ~9-15 GB/s
// on the GPU hosts measured by tools/h2d_probe, is well below the ~55 GB/s of pinned DMA). Workers
// spin on a job counter for a while after each job (pipeline pieces follow each other within tens
// of microseconds) and sleep on a condition variable when idle.
class CopyTeam {
 public:
  CopyTeam() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    team_ = std::min(8u, hw);
    for (unsigned k = 1; k < team_; ++k) workers_.emplace_back([this, k] { work(k); });
  }
  ~CopyTeam() {
    stop_.store(true);
    {
      std::lock_guard<std::mutex> g(mu_);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (team_ == 1 || bytes < (size_t(256) << 10)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    pending_.store(team_ - 1);
    {
      std::lock_guard<std::mutex> g(mu_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    part(0);
    while (pending_.load(std::memory_order_acquire) != 0) {
    }
  }

 private:
  void part(unsigned k) {
    const size_t per = (bytes_ / team_ + 63) & ~size_t(63);
    const size_t lo = std::min(bytes_, per * k), hi = std::min(bytes_, lo + per);
    if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void work(unsigned k) {
    unsigned long long seen = 0;
    for (;;) {
      // spin briefly for the next job, then sleep
      const auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(200)) {
      }
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return gen_.load() != seen; });
      }
      seen = gen_.load(std::memory_order_acquire);
      if (stop_.load()) return;
      part(k);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> workers_;
  unsigned team_ = 1;
  std::mutex mu_;
  std::condition_variable cv_;
  std::atomic<unsigned long long> gen_{0};
  std::atomic<unsigned> pending_{0};
  std::atomic<bool> stop_{false};
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
};

struct Staging {
  std::mutex mu;  // one pipelined transfer at a time per process
  CopyTeam team;
  char* ring[kRing] = {};
  cudaEvent_t ev[kRing] = {};
  int device = -1;
  void ensure(int dev) {
    if (ring[0] && device == dev) return;
    for (int k = 0; k < kRing; ++k) {
      if (ev[k]) cudaEventDestroy(ev[k]);
      if (ring[k]) cudaFreeHost(ring[k]);
      CK(cudaMallocHost(&ring[k], kPiece));
      CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    }
    device = dev;
  }
};

Staging& staging() {
  static Staging* s = new Staging();  // never destroyed: worker threads outlive static teardown order
  return *s;
}

// at least four pieces in flight for mid-sized transfers, 1..8 MB each
size_t piece_for(size_t bytes) {
  const size_t p = (bytes / 4 + 4095) & ~size_t(4095);
  return std::max(size_t(1) << 20, std::min(kPiece, p));
}

bool pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

void copy_to_device(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < kDirect || pinned(src)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  Staging& s = staging();
  std::lock_guard<std::mutex> g(s.mu);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  s.ensure(dev);
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const size_t piece = piece_for(bytes);
  for (size_t off = 0, k = 0; off < bytes; off += piece, ++k) {
    const size_t len = std::min(piece, bytes - off);
    const int b = static_cast<int>(k % kRing);
    if (k >= kRing) CK(cudaEventSynchronize(s.ev[b]));  // the DMA that last read this piece is done
    s.team.copy(s.ring[b], in + off, len);
    CK(cudaMemcpyAsync(out + off, s.ring[b], len, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(s.ev[b], st));
  }
  // the pieces must not be reused before their DMA ran
  for (int b = 0; b < kRing; ++b) CK(cudaEventSynchronize(s.ev[b]));
}

void copy_to_host(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < kDirect || pinned(dst)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return;
  }
  Staging& s = staging();
  std::lock_guard<std::mutex> g(s.mu);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  s.ensure(dev);
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const size_t piece = piece_for(bytes);
  const size_t pieces = (bytes + piece - 1) / piece;
  auto enqueue = [&](size_t k) {
    const size_t off = k * piece, len = std::min(piece, bytes - off);
    const int b = static_cast<int>(k % kRing);
    CK(cudaMemcpyAsync(s.ring[b], in + off, len, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s.ev[b], st));
  };
  for (size_t k = 0; k < std::min<size_t>(pieces, kRing - 1); ++k) enqueue(k);
  for (size_t k = 0; k < pieces; ++k) {
    if (k + kRing - 1 < pieces) enqueue(k + kRing - 1);  // its piece was emptied in iteration k-1
    const int b = static_cast<int>(k % kRing);
    CK(cudaEventSynchronize(s.ev[b]));
    const size_t off = k * piece, len = std::min(piece, bytes - off);
    s.team.copy(out + off, s.ring[b], len);
  }
}

}  // namespace tlsph_cuda
