// Microbenchmark: scalar FFMA vs packed FFMA2 (fma.rn.f32x2) issue/throughput on sm_100a.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/ubench_ffma2.cu -o /tmp/ub && /tmp/ub
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float s) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 0.25f);
  float t = 0; for (int i = 0; i < 8; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ffma2(float* out, float s) {
  float2 a[4];
  for (int i = 0; i < 4; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
  const float2 s2 = make_float2(s, s), c2 = make_float2(0.25f, 0.25f);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __ffma2_rn(a[i], s2, c2);
  float t = 0; for (int i = 0; i < 4; ++i) t += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
// 16 independent chains (scalar) vs 8 float2 chains, more ILP
__global__ void k_ffma16(float* out, float s) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.25f);
  float t = 0; for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ffma2_16(float* out, float s) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
  const float2 s2 = make_float2(s, s), c2 = make_float2(0.25f, 0.25f);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], s2, c2);
  float t = 0; for (int i = 0; i < 8; ++i) t += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
// scalar FFMA with a register (non-immediate) third operand, the K1 case
__global__ void k_ffma_reg(float* out, float s, float c) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, c);
  float t = 0; for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <typename K, typename... A>
void run(const char* name, K k, int flops_per_thread_iter, A... args) {
  float* d; cudaMalloc(&d, 148 * 8 * 1024 * sizeof(float));
  const int blocks = 148 * 8, threads = 256;
  k<<<blocks, threads>>>(d, args...);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 10; ++rep) k<<<blocks, threads>>>(d, args...);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fma = 10.0 * blocks * threads * (double)ITERS * flops_per_thread_iter;
  printf("%-12s %8.3f ms  %7.2f T FMA/s\n", name, ms, fma / (ms * 1e-3) / 1e12);
  cudaFree(d);
}
int main() {
  run("ffma x8", k_ffma, 8, 0.999f);
  run("ffma2 x4", k_ffma2, 8, 0.999f);
  run("ffma x16", k_ffma16, 16, 0.999f);
  run("ffma2 x8", k_ffma2_16, 16, 0.999f);
  run("ffma reg x16", k_ffma_reg, 16, 0.999f, 0.25f);
  return 0;
}
