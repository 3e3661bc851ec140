// Pipe-rate microbenchmark on sm_100a: FFMA (scalar), FFMA2 (fma.rn.f32x2),
// DFMA, HFMA2, LDG-free.  Prints per-SM ops/clk estimates from CUDA events
// and the measured SM clock.  Used to choose the arithmetic of the hot
// kernels.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ float2 ffma2(float2 x, float2 a, float2 b) {
  unsigned long long xr = *reinterpret_cast<unsigned long long*>(&x);
  unsigned long long ar = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long br = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(xr), "l"(ar), "l"(br));
  return *reinterpret_cast<float2*>(&d);
}

__global__ void k_ffma2(float* out, float a, float b) {
  float2 A = make_float2(a, a), B = make_float2(b, b);
  float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, 3), x2 = make_float2(4, 5), x3 = make_float2(6, 7);
  for (int i = 0; i < ITERS; ++i) {
    x0 = ffma2(x0, A, B); x1 = ffma2(x1, A, B); x2 = ffma2(x2, A, B); x3 = ffma2(x3, A, B);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0.x + x1.x + x2.x + x3.x + x0.y + x1.y + x2.y + x3.y;
}

__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_hfma2(float* out, float a, float b) {
  __half2 A = __float2half2_rn(a), B = __float2half2_rn(b);
  __half2 x0 = __float2half2_rn(threadIdx.x), x1 = x0, x2 = x0, x3 = x0, x4 = x0, x5 = x0, x6 = x0, x7 = x0;
  for (int i = 0; i < ITERS; ++i) {
    x0 = __hfma2(x0, A, B); x1 = __hfma2(x1, A, B); x2 = __hfma2(x2, A, B); x3 = __hfma2(x3, A, B);
    x4 = __hfma2(x4, A, B); x5 = __hfma2(x5, A, B); x6 = __hfma2(x6, A, B); x7 = __hfma2(x7, A, B);
  }
  float2 f = __half22float2(__hadd2(__hadd2(__hadd2(x0, x1), __hadd2(x2, x3)), __hadd2(__hadd2(x4, x5), __hadd2(x6, x7))));
  out[blockIdx.x * blockDim.x + threadIdx.x] = f.x + f.y;
}

template <class K, class T>
void run(const char* name, K kern, T* buf, double flops_per_thread, int sms) {
  const int blocks = sms * 8, threads = 256;
  kern<<<blocks, threads>>>(buf, (T)0.999, (T)0.001);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(buf, (T)0.999, (T)0.001);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fmas = 5.0 * blocks * threads * flops_per_thread;
  printf("%-6s %8.2f TFMA/s  (%.1f TFLOPS)  %.3f ms\n", name, fmas / (ms * 1e-3) / 1e12, 2 * fmas / (ms * 1e-3) / 1e12, ms / 5);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s: %d SMs, max clock %.0f MHz\n", p.name, p.multiProcessorCount, clk / 1e3);
  float* f;
  double* d;
  cudaMalloc(&f, sizeof(float) * p.multiProcessorCount * 8 * 256);
  cudaMalloc(&d, sizeof(double) * p.multiProcessorCount * 8 * 256);
  run("FFMA", k_ffma, f, 8.0 * ITERS, p.multiProcessorCount);
  run("FFMA2", k_ffma2, f, 8.0 * ITERS, p.multiProcessorCount);
  run("HFMA2", k_hfma2, f, 16.0 * ITERS, p.multiProcessorCount);
  run("DFMA", k_dfma, d, 8.0 * ITERS, p.multiProcessorCount);
  printf("per SM per clock at max clock: divide TFMA/s by (SMs * clock)\n");
  return 0;
}
