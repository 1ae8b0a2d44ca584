// Pipe-peak microbenchmark for the roofline denominators the driver does not
// measure (MEASURED_PEAKS.json has HBM and bf16 only): FP64 DFMA, FP32 FFMA,
// MUFU.LG2 and FP64 divide throughput on this B200.  Prints one JSON line.
#include <cuda_runtime.h>
#include <stdio.h>

template <int CH>
__global__ void dfma_k(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
template <int CH>
__global__ void ffma_k(float* out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.678f) out[0] = s;
}
template <int CH>
__global__ void lg2_k(float* out, int iters) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = 1.5f + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __log2f(x[i]) + 2.0f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.678f) out[0] = s;
}
template <int CH>
__global__ void ddiv_k(double* out, int iters) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = 1.5 + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = 3.0 / x[i] + 1.0;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
template <int CH>
__global__ void dlog_k(double* out, int iters) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = 1.5 + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = log2(x[i]) + 2.0;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <class F>
static float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* dd; float* fd;
  cudaMalloc(&dd, 64); cudaMalloc(&fd, 64);
  const int blocks = sms * 8, threads = 256, it = 4096;
  const double nthr = (double)blocks * threads;
  float t;
  t = timeit([&] { dfma_k<8><<<blocks, threads>>>(dd, it, 1.0000001, 1e-9); });
  double dfma = nthr * it * 8 * 2 / (t * 1e-3) / 1e12;
  t = timeit([&] { ffma_k<8><<<blocks, threads>>>(fd, it, 1.0000001f, 1e-9f); });
  double ffma = nthr * it * 8 * 2 / (t * 1e-3) / 1e12;
  t = timeit([&] { lg2_k<8><<<blocks, threads>>>(fd, it / 4); });
  double lg2 = nthr * (it / 4) * 8 / (t * 1e-3) / 1e12;
  t = timeit([&] { ddiv_k<8><<<blocks, threads>>>(dd, it / 8); });
  double ddiv = nthr * (it / 8) * 8 / (t * 1e-3) / 1e12;
  t = timeit([&] { dlog_k<8><<<blocks, threads>>>(dd, it / 16); });
  double dlog = nthr * (it / 16) * 8 / (t * 1e-3) / 1e12;
  printf("{\"sms\": %d, \"clock_mhz_attr\": %d, \"fp64_fma_tflops\": %.3f, \"fp32_fma_tflops\": %.3f, "
         "\"mufu_lg2_tops\": %.4f, \"fp64_div_tops\": %.4f, \"fp64_log2_tops\": %.4f}\n",
         sms, clk / 1000, dfma, ffma, lg2, ddiv, dlog);
  return 0;
}
