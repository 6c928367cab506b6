// gen.cu -- GPU helpers of the synthetic scene generator (input generation
// only: no arithmetic of the raycasting method).  Used for the configs whose
// host generation would take minutes (C5: ~1.9e8 leaves, 512 bumps).
//
//  sg_shell_refine: refinement rule of SURVEY §8(c) R20 -- element centre on
//    the exact cubed-sphere shell (R21) closer than c 2^-level to a source.
//  sg_shell_bumps: nodal field f(x) = sum_i a_i exp(-|x - c_i|^2 / (2 s_i^2))
//    at the element-local GLL nodes mapped through the exact shell, in fp64,
//    rounded once to fp32; also max |f| (for F).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace {

constexpr double R_IN = 0.55, R_OUT = 1.0;
constexpr int MAXLEVEL = 18;
constexpr int MAXB = 1024;

__device__ void shell_point(int k, double t1, double t2, double t3, double x[3]) {
  const int a = k / 2, b = (a + 1) % 3, c = (a + 2) % 3;
  const double s = 1.0 - 2.0 * (k % 2);
  double p[3];
  p[a] = s;
  p[b] = 2.0 * t1 - 1.0;
  p[c] = s * (2.0 * t2 - 1.0);
  const double nrm = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
  const double r = R_IN + (R_OUT - R_IN) * t3;
  for (int q = 0; q < 3; ++q) x[q] = r * p[q] / nrm;
}

__global__ void k_refine(const int32_t* __restrict__ anchor, const int32_t* __restrict__ tree, int64_t n, int level,
                         const double* __restrict__ src, int nsrc, double c, uint8_t* __restrict__ flag) {
  __shared__ double S[MAXB * 3];
  for (int i = threadIdx.x; i < nsrc * 3; i += blockDim.x) S[i] = src[i];
  __syncthreads();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double h = ldexp(1.0, -level);
  double x[3];
  shell_point(tree[e], ldexp((double)anchor[3 * e], -MAXLEVEL) + 0.5 * h,
              ldexp((double)anchor[3 * e + 1], -MAXLEVEL) + 0.5 * h,
              ldexp((double)anchor[3 * e + 2], -MAXLEVEL) + 0.5 * h, x);
  double d2 = 1e300;
  for (int i = 0; i < nsrc; ++i) {
    const double dx = x[0] - S[3 * i], dy = x[1] - S[3 * i + 1], dz = x[2] - S[3 * i + 2];
    d2 = fmin(d2, dx * dx + dy * dy + dz * dz);
  }
  flag[e] = sqrt(d2) < c * h ? 1 : 0;
}

__global__ void k_bumps(const int32_t* __restrict__ anchor, const int32_t* __restrict__ tree,
                        const int8_t* __restrict__ level, int64_t n, int P, const double* __restrict__ bumps, int nb,
                        float* __restrict__ out, unsigned long long* __restrict__ fmax_bits) {
  __shared__ double B[MAXB * 5];   // cx, cy, cz, 1/(2 s^2), a
  for (int i = threadIdx.x; i < nb * 5; i += blockDim.x) B[i] = bumps[i];
  __syncthreads();
  const int np1 = P + 1, NP = np1 * np1 * np1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double fa = 0.0;
  if (idx < n * NP) {
    const int64_t e = idx / NP;
    const int q = (int)(idx % NP);
    const int k1 = q % np1, k2 = (q / np1) % np1, k3 = q / (np1 * np1);
    const double h = ldexp(1.0, -(int)level[e]);
    const double eta1 = (double)k1 / P, eta2 = (double)k2 / P, eta3 = (double)k3 / P;
    double x[3];
    shell_point(tree[e], ldexp((double)anchor[3 * e], -MAXLEVEL) + h * eta1,
                ldexp((double)anchor[3 * e + 1], -MAXLEVEL) + h * eta2,
                ldexp((double)anchor[3 * e + 2], -MAXLEVEL) + h * eta3, x);
    double f = 0.0;
    for (int i = 0; i < nb; ++i) {
      const double dx = x[0] - B[5 * i], dy = x[1] - B[5 * i + 1], dz = x[2] - B[5 * i + 2];
      f += B[5 * i + 4] * exp(-(dx * dx + dy * dy + dz * dz) * B[5 * i + 3]);
    }
    out[idx] = (float)f;
    fa = fabs(f);
  }
  // block max of |f| (non-negative doubles order like their bit patterns)
  for (int off = 16; off > 0; off >>= 1) fa = fmax(fa, __shfl_xor_sync(0xffffffffu, fa, off));
  if ((threadIdx.x & 31) == 0 && fa > 0.0) atomicMax(fmax_bits, (unsigned long long)__double_as_longlong(fa));
}

}  // namespace

extern "C" int sg_shell_refine(const int32_t* anchor, const int32_t* tree, int64_t n, int level, const double* src,
                               int nsrc, double c, uint8_t* flag, void* stream) {
  if (nsrc > MAXB) return -1;
  if (n == 0) return 0;
  k_refine<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(anchor, tree, n, level, src, nsrc, c, flag);
  return (int)cudaGetLastError();
}

extern "C" int sg_shell_bumps(const int32_t* anchor, const int32_t* tree, const int8_t* level, int64_t n, int P,
                              const double* bumps, int nb, float* out, unsigned long long* fmax_bits, void* stream) {
  if (nb > MAXB) return -1;
  const int NP = (P + 1) * (P + 1) * (P + 1);
  const int64_t total = n * NP;
  if (total == 0) return 0;
  k_bumps<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(anchor, tree, level, n, P, bumps, nb,
                                                                            out, fmax_bits);
  return (int)cudaGetLastError();
}
