// FFMA vs FFMA2 (packed fp32x2, sm_100a) throughput microbenchmark: 8 independent
// chains per thread, 148*8 CTAs x 256 threads; prints FLOP/s of each.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1(float* out, float a, float b, int iters) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, float a, float b, int iters) {
  float2 x[8];
  const float2 A = make_float2(a, a), Bv = make_float2(b, b);
  for (int j = 0; j < 8; ++j) x[j] = make_float2(threadIdx.x * 1e-3f + j, j * 0.5f);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __ffma2_rn(x[j], A, Bv);
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j].x + x[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int it = 20000; float ms;
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0); k1<<<148 * 8, 256>>>(o, 0.999f, 1e-3f, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA : %.1f TFLOP/s\n", 2.0 * 8 * it * 148 * 8 * 256 / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); k2<<<148 * 8, 256>>>(o, 0.999f, 1e-3f, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2: %.1f TFLOP/s\n", 4.0 * 8 * it * 148 * 8 * 256 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
