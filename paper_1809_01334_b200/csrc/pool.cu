// pool.cu -- caching device allocator of librc.  Forests allocate large,
// long-lived buffers (records, scratch, per-leaf arrays); a caching pool lets
// a new forest (or a regrown buffer) reuse the blocks of a destroyed one
// instead of paying cudaMalloc/cudaFree of tens of GB each time.  Best fit
// within 1.5x of the request; on an out-of-memory error the cached blocks
// are released and the allocation retried once.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <unordered_map>

#include "rc_internal.cuh"

namespace rc {

namespace {
std::mutex g_mu;
std::multimap<size_t, void*> g_free;         // size -> cached block
std::unordered_map<void*, size_t> g_size;    // live and cached block sizes

void release_cached_locked() {
  for (auto& kv : g_free) {
    g_size.erase(kv.second);
    cudaFree(kv.second);
  }
  g_free.clear();
}
}  // namespace

cudaError_t dmalloc(void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 256;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_free.lower_bound(bytes);
  if (it != g_free.end() && it->first <= bytes + bytes / 2 + ((size_t)1 << 20)) {
    *p = it->second;
    g_free.erase(it);
    return cudaSuccess;
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();   // clear the sticky-free error state
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

void dfree(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_size.find(p);
  if (it == g_size.end()) {   // not from the pool
    cudaFree(p);
    return;
  }
  g_free.insert({it->second, p});
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
