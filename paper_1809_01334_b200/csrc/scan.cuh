// scan.cuh -- device-wide exclusive prefix sums (int64 results), used for
// visible-leaf compaction, the chunk offsets of the pair generation and the
// per-pixel bucket offsets of the composite.  Three-phase reduce-then-scan:
// one 1024-thread block per 4096 items, recursive scan of the block sums.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rc {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// `in` and `out` may alias (in-place scan of int64 counts): no __restrict__ on
// them; every thread reads its own items before it writes them.
template <typename Tin>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tile(const Tin* in, int64_t* out, int64_t n,
                                                             int64_t* __restrict__ tile_sums) {
  __shared__ int64_t warp_sums[SCAN_THREADS / 32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t local = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t idx = base + k;
    v[k] = idx < n ? (int64_t)in[idx] : 0;
    local += v[k];
  }
  // inclusive warp scan of per-thread sums
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t ws = warp_sums[lane];
    int64_t wi = ws;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += y;
    }
    warp_sums[lane] = wi - ws;  // exclusive
    if (lane == 31 && tile_sums) tile_sums[blockIdx.x] = wi;
  }
  __syncthreads();
  int64_t run = warp_sums[warp] + incl - local;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t idx = base + k;
    if (idx < n) out[idx] = run;
    run += v[k];
  }
  // the last thread of the last tile writes the grand total (for single-tile scans)
  if (gridDim.x == 1 && threadIdx.x == SCAN_THREADS - 1) out[n] = run;
}

__global__ void k_scan_add(int64_t* __restrict__ out, int64_t n, const int64_t* __restrict__ tile_off);

}  // namespace rc
