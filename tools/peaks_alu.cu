// Measures the FP64 / FP32 CUDA-core FMA peak and dependent-FMA latency on the
// local GPU (the roofline denominator for the ALU-bound RNEA path).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks_alu peaks_alu.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CHAINS>
__global__ void fma_tput(T* out, int iters, T a, T b) {
  T x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = (T)(threadIdx.x + c);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == (T)12345.678) out[threadIdx.x] = s;
}

template <typename T>
__global__ void fma_lat(T* out, long long* cyc, int iters, T a, T b) {
  T x = (T)threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <typename T, int CHAINS>
void run_tput(const char* name, int blocks_per_sm, int threads) {
  int dev; cudaGetDevice(&dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  T* out; cudaMalloc(&out, 1024 * sizeof(T));
  int iters = 1 << 16;
  int grid = p.multiProcessorCount * blocks_per_sm;
  fma_tput<T, CHAINS><<<grid, threads>>>(out, 1024, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_tput<T, CHAINS><<<grid, threads>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * CHAINS * (double)iters * grid * threads;
  printf("{\"kind\":\"tput\",\"type\":\"%s\",\"chains\":%d,\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
         name, CHAINS, blocks_per_sm, threads, ms, flops / ms / 1e9);
  cudaFree(out);
}

template <typename T>
void run_lat(const char* name) {
  T* out; long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(T)); cudaMalloc(&cyc, sizeof(long long));
  int iters = 4096;
  fma_lat<T><<<1, 32>>>(out, cyc, iters, (T)0.999, (T)0.001);
  fma_lat<T><<<1, 32>>>(out, cyc, iters, (T)0.999, (T)0.001);
  long long h; cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"kind\":\"latency\",\"type\":\"%s\",\"cycles_per_fma\":%.2f}\n", name, (double)h / (iters * 16.0));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu,\"regs_per_sm\":%d}\n",
         p.name, p.multiProcessorCount, p.clockRate, p.l2CacheSize, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  run_lat<double>("f64");
  run_lat<float>("f32");
  run_tput<double, 8>("f64", 4, 256);
  run_tput<double, 4>("f64", 1, 128);
  run_tput<double, 8>("f64", 1, 128);
  run_tput<double, 2>("f64", 1, 128);
  run_tput<double, 1>("f64", 1, 128);
  run_tput<double, 2>("f64", 2, 128);
  run_tput<double, 4>("f64", 2, 128);
  run_tput<double, 8>("f64", 8, 256);
  run_tput<float, 8>("f32", 4, 256);
  run_tput<float, 8>("f32", 8, 256);
  // sustained: ~2 s of f64 FMA to see the clock under load
  for (int r = 0; r < 10; ++r) run_tput<double, 8>("f64", 8, 256);
  return 0;
}
