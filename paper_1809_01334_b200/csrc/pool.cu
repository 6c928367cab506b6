// pool.cu -- caching device allocator of librc.  Forests allocate large,
// long-lived buffers (records, scratch, per-leaf arrays); a caching pool lets
// a new forest (or a regrown buffer) reuse the blocks of a destroyed one
// instead of paying cudaMalloc/cudaFree of tens of GB each time.
//
// Reuse is stream-ordered: dfree records an event on the stream whose work
// may still read the block; a later dmalloc on the same stream reuses it at
// once (stream order), on another stream it makes that stream wait for the
// event first (cudaStreamWaitEvent, no host sync).  Blocks are keyed by
// device.  Best fit within 1.5x of the request; on an out-of-memory error the
// cached blocks are released (after their events complete) and the
// allocation retried once.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <unordered_map>

#include "rc_internal.cuh"

namespace rc {

namespace {
struct Cached {
  void* p;
  cudaStream_t stream;   // stream of the last use (the free)
  cudaEvent_t done;      // recorded on `stream` at the free; nullptr = no pending work
};
struct Key {
  int dev;
  size_t size;
  bool operator<(const Key& o) const { return dev != o.dev ? dev < o.dev : size < o.size; }
};
std::mutex g_mu;
std::multimap<Key, Cached> g_free;           // (device, size) -> cached block
std::unordered_map<void*, size_t> g_size;    // live and cached block sizes

void release_cached_locked() {
  for (auto& kv : g_free) {
    if (kv.second.done) {
      cudaEventSynchronize(kv.second.done);
      cudaEventDestroy(kv.second.done);
    }
    g_size.erase(kv.second.p);
    cudaFree(kv.second.p);
  }
  g_free.clear();
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace

cudaError_t dmalloc(void** p, size_t bytes, cudaStream_t s) {
  *p = nullptr;
  if (bytes == 0) bytes = 256;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_free.lower_bound(Key{dev, bytes});
  if (it != g_free.end() && it->first.dev == dev && it->first.size <= bytes + bytes / 2 + ((size_t)1 << 20)) {
    Cached c = it->second;
    g_free.erase(it);
    cudaError_t e = cudaSuccess;
    if (c.done) {
      if (c.stream != s) e = cudaStreamWaitEvent(s, c.done, 0);   // stream-ordered hand-over
      cudaEventDestroy(c.done);
    }
    if (e != cudaSuccess) {
      g_size.erase(c.p);
      cudaFree(c.p);
      return e;
    }
    *p = c.p;
    return cudaSuccess;
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();   // clear the error state
    release_cached_locked();
    e = cudaMalloc(p, bytes);
  }
  if (e != cudaSuccess) {
    *p = nullptr;
    return e;
  }
  g_size[*p] = bytes;
  return cudaSuccess;
}

void dfree(void* p, cudaStream_t s, bool idle) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_size.find(p);
  if (it == g_size.end()) {   // not from the pool
    cudaFree(p);
    return;
  }
  Cached c{p, s, nullptr};
  if (!idle) {
    if (cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(c.done, s) != cudaSuccess) {
      // cannot order the reuse: wait for the stream's work instead
      if (c.done) cudaEventDestroy(c.done);
      c.done = nullptr;
      cudaGetLastError();
      cudaStreamSynchronize(s);
    }
  }
  g_free.insert({Key{current_device(), it->second}, c});
}

size_t device_free_bytes() {
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& kv : g_free)
    if (kv.first.dev == dev) free_b += kv.first.size;   // cached blocks are released on demand
  return free_b;
}

void dtrim() {
  std::lock_guard<std::mutex> lk(g_mu);
  release_cached_locked();
}

}  // namespace rc

extern "C" rc_status rc_pool_trim(void) {
  rc::dtrim();
  return RC_OK;
}
