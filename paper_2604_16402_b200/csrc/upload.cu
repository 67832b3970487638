// Host -> device upload of large pageable buffers (the build's input rows).
//
// A plain cudaMemcpyAsync from pageable memory runs at the speed of the
// driver's single-threaded copy into its pinned bounce buffers (~11 GB/s on
// the B200 hosts: 48 ms of a 1M x 128 build). Here the source is copied into a
// ring of pinned chunks by several host threads at once while the previous
// chunks are already on the wire, so the host-memory copy and the DMA overlap
// and the copy itself is parallel. Small buffers take the plain path.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "index.cuh"

namespace grab {

namespace {
constexpr size_t kChunk = 32ull << 20;  // bytes per pinned chunk
constexpr int kRing = 4;                // chunks in flight
constexpr size_t kMinParallel = 64ull << 20;

struct UploadRing {
  std::mutex mu;
  void* buf[kRing] = {};
  cudaEvent_t done[kRing] = {};
  bool ready = false;
};
UploadRing& ring() {
  static UploadRing r;  // process lifetime (pinned host memory is freed at exit)
  return r;
}
}  // namespace

void upload_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes < kMinParallel) {
    GRAB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  UploadRing& r = ring();
  std::lock_guard<std::mutex> g(r.mu);
  if (!r.ready) {
    for (int i = 0; i < kRing; ++i) {
      GRAB_CUDA(cudaHostAlloc(&r.buf[i], kChunk, cudaHostAllocDefault));
      GRAB_CUDA(cudaEventCreateWithFlags(&r.done[i], cudaEventDisableTiming));
      GRAB_CUDA(cudaEventRecord(r.done[i], st));
    }
    r.ready = true;
  }
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nthr = (int)std::min<unsigned>(8u, hw);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
    const int b = (int)(i % kRing);
    const size_t len = std::min(kChunk, bytes - off);
    GRAB_CUDA(cudaEventSynchronize(r.done[b]));  // the chunk's previous DMA has drained
    char* pin = static_cast<char*>(r.buf[b]);
    const size_t part = (len + nthr - 1) / nthr;
    std::vector<std::thread> th;
    for (int t = 1; t < nthr; ++t) {
      const size_t a = std::min(len, (size_t)t * part), e = std::min(len, a + part);
      if (a < e) th.emplace_back([=] { std::memcpy(pin + a, s + off + a, e - a); });
    }
    std::memcpy(pin, s + off, std::min(len, part));
    for (auto& x : th) x.join();
    GRAB_CUDA(cudaMemcpyAsync(d + off, pin, len, cudaMemcpyHostToDevice, st));
    GRAB_CUDA(cudaEventRecord(r.done[b], st));
  }
}

}  // namespace grab
