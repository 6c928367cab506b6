// scan.cu -- host driver of the three-phase exclusive scan (see scan.cuh).
#include "rc_internal.cuh"
#include "scan.cuh"

namespace rc {

__global__ void k_scan_add(int64_t* __restrict__ out, int64_t n, const int64_t* __restrict__ tile_off) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t add = tile_off[blockIdx.x];
  for (int k = threadIdx.x; k < SCAN_TILE; k += blockDim.x) {
    int64_t idx = base + k;
    if (idx < n) out[idx] += add;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = tile_off[gridDim.x];
}

size_t scan_tmp_size(int64_t n) {
  size_t total = 0;
  int64_t m = n;
  while (m > SCAN_TILE) {
    int64_t nb = (m + SCAN_TILE - 1) / SCAN_TILE;
    total += 2 * (nb + 1);
    m = nb;
  }
  return total + 16;
}

template <typename Tin>
cudaError_t scan_exclusive(const Tin* in, int64_t* out, int64_t n, int64_t* tmp, cudaStream_t s) {
  if (n <= 0) {
    return cudaMemsetAsync(out, 0, sizeof(int64_t), s);
  }
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (nb == 1) {
    k_scan_tile<Tin><<<1, SCAN_THREADS, 0, s>>>(in, out, n, nullptr);
    ++g_launches;
    return cudaGetLastError();
  }
  int64_t* sums = tmp;
  int64_t* offs = tmp + nb + 1;
  k_scan_tile<Tin><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, sums);
  ++g_launches;
  cudaError_t err = scan_exclusive<int64_t>(sums, offs, nb, tmp + 2 * (nb + 1), s);
  if (err != cudaSuccess) return err;
  k_scan_add<<<(unsigned)nb, 256, 0, s>>>(out, n, offs);
  ++g_launches;
  return cudaGetLastError();
}

template cudaError_t scan_exclusive<int32_t>(const int32_t*, int64_t*, int64_t, int64_t*, cudaStream_t);
template cudaError_t scan_exclusive<int64_t>(const int64_t*, int64_t*, int64_t, int64_t*, cudaStream_t);

cudaError_t scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* tmp, cudaStream_t s) {
  return scan_exclusive<int64_t>(in, out, n, tmp, s);
}

}  // namespace rc
