// Throughput of FFMA (register operands) vs FFMA2 (fma.rn.f32x2) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(r);
}
template <int ILP>
__global__ void k_ffma(float* out, int iters, float a0, float b0) {
  float v[ILP], a[ILP], b[ILP];
  for (int j = 0; j < ILP; ++j) { v[j] = threadIdx.x * 1e-3f + j; a[j] = a0 + j * 1e-9f; b[j] = b0 * (j + 1); }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) v[j] = fmaf(v[j], a[j], b[j]);
  float s = 0; for (int j = 0; j < ILP; ++j) s += v[j];
  if (s == 12345.f) out[0] = s;
}
template <int ILP>
__global__ void k_ffma2(float* out, int iters, float a0, float b0) {
  float2 v[ILP], a[ILP], b[ILP];
  for (int j = 0; j < ILP; ++j) { v[j] = make_float2(threadIdx.x * 1e-3f + j, j + 0.5f); a[j] = make_float2(a0 + j * 1e-9f, a0 - j * 1e-9f); b[j] = make_float2(b0 * (j + 1), b0 * (j + 2)); }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) v[j] = ffma2(v[j], a[j], b[j]);
  float s = 0; for (int j = 0; j < ILP; ++j) s += v[j].x + v[j].y;
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256, iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ffma<8><<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("FFMA  reg: %.1f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0); k_ffma2<8><<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 4.0 * 8 * iters * (double)blocks * threads;
    printf("FFMA2 reg: %.1f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  }
  return 0;
}
