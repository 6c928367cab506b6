// peaks.cu -- FP32 pipe peaks of this B200 for the segment kernel's roofline
// ("independent-chain FFMA, MUFU.EX2 and FMNMX across all
// SMs").  Each thread runs CH independent dependency chains of one
// instruction for ITERS iterations; the grid fills every SM.  Prints one JSON
// line: giga-instructions/s per pipe and the FFMA TFLOP/s (2 flops / FFMA).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;
constexpr int ITERS = 1 << 17;   // ~10 ms per launch: clocks settle, loop overhead < 1%

__global__ void k_ffma(float* out, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
#pragma unroll 32
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(a), "f"(b));
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void k_ex2(float* out) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = -1e-3f * (threadIdx.x + c);
#pragma unroll 32
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void k_fmnmx(float* out, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
#pragma unroll 32
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      asm volatile("min.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(a));
      asm volatile("max.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(b));
    }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double a, double b) {   // FP64 pipe (surface kernel's geometry)
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
#pragma unroll 32
  for (int i = 0; i < ITERS / 4; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(a), "d"(b));
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <class F>
static double run(F launch, double insts_per_thread, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();   // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 20; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return insts_per_thread * blocks * threads / (best * 1e-3) / 1e9;   // giga-instructions / s
}

int main() {
  int sms = 0, dev = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4096);
  const int threads = 512, blocks = sms * 4;   // 64 warps per SM
  const double ffma = run([&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-4f); }, (double)ITERS * CH, blocks,
                          threads);
  const double ex2 = run([&] { k_ex2<<<blocks, threads>>>(out); }, (double)ITERS * CH, blocks, threads);
  const double mnx = run([&] { k_fmnmx<<<blocks, threads>>>(out, 1e3f, -1e3f); }, (double)ITERS * CH * 2, blocks,
                         threads);
  const double dfma = run([&] { k_dfma<<<blocks, threads>>>(reinterpret_cast<double*>(out), 0.999, 1e-4); },
                          (double)(ITERS / 4) * CH, blocks, threads);
  cudaError_t e = cudaGetLastError();
  printf("{\"dfma_ginst_s\": %.1f, \"dfma_tflops\": %.3f, ", dfma, 2 * dfma / 1000.0);
  printf("\"sms\": %d, \"clock_attr_mhz\": %.0f, \"ffma_ginst_s\": %.1f, \"ffma_tflops\": %.2f, "
         "\"mufu_ex2_ginst_s\": %.1f, \"mufu_ex2_tops\": %.3f, \"fmnmx_ginst_s\": %.1f, \"fmnmx_tops\": %.3f, "
         "\"per_sm_per_clk_at_attr\": {\"ffma\": %.1f, \"ex2\": %.2f, \"fmnmx\": %.1f}, \"error\": \"%s\"}\n",
         sms, clk / 1000.0, ffma, 2 * ffma / 1000.0, ex2, ex2 / 1000.0, mnx, mnx / 1000.0,
         ffma * 1e9 / sms / (clk * 1e3), ex2 * 1e9 / sms / (clk * 1e3), mnx * 1e9 / sms / (clk * 1e3),
         cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
