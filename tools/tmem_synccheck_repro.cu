// tmem_synccheck_repro.cu -- minimal kernels for the compute-sanitizer synccheck
// finding on rnea_thread_pp_kernel ("Barrier error detected. Missing init ...
// Barrier is located at shared address 0x0", VERDICT r01 missing-4).
//
// Each variant is a complete, correct tcgen05 program (alloc -> relinquish ->
// __syncthreads -> st / wait::st / ld / wait::ld -> __syncthreads -> dealloc), the
// exact sequence rnea_thread.cu uses, with nothing else in the kernel:
//   0  no tcgen05 at all (control: synccheck must be clean)
//   1  tcgen05.alloc / dealloc only
//   2  alloc + one st / ld round trip (checks the value)
//   3  like 2, the allocation slot at a non-zero shared offset
// If variants 1-3 abort under synccheck while memcheck / racecheck pass and the
// kernel's results are right, the finding is the tool's handling of tcgen05.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_synccheck_repro tools/tmem_synccheck_repro.cu
//   compute-sanitizer --tool synccheck tools/tmem_synccheck_repro <variant>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int V>
__global__ void repro(int* out) {
  __shared__ __align__(16) uint32_t pad[4];
  __shared__ __align__(16) uint32_t slot_at0;
  uint32_t* slot = (V == 3) ? &pad[2] : &slot_at0;
  if (V == 3 && threadIdx.x == 0) pad[0] = 7;
  const int warp = threadIdx.x / 32;
  if (V >= 1) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(smem_u32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  int val = (int)threadIdx.x;
  if (V >= 2) {
    const uint32_t taddr = *slot + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)(warp / 4) * 8;
    const uint32_t x = 1000u + threadIdx.x;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" :: "r"(taddr), "r"(x));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    uint32_t y;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(y) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+r"(y) :: "memory");
    val = (int)y - 1000;
  }
  if (V >= 1) asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (V >= 1 && warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(*slot));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = val;
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 2;
  const int blocks = 4, threads = 256;
  int* d;
  cudaMalloc(&d, blocks * threads * sizeof(int));
  switch (v) {
    case 0: repro<0><<<blocks, threads>>>(d); break;
    case 1: repro<1><<<blocks, threads>>>(d); break;
    case 2: repro<2><<<blocks, threads>>>(d); break;
    default: repro<3><<<blocks, threads>>>(d); break;
  }
  cudaError_t e = cudaDeviceSynchronize();
  int h[blocks * threads];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < blocks * threads; ++i) bad += (h[i] != i % threads);
  printf("variant %d: %s, %d wrong values\n", v, cudaGetErrorString(e), bad);
  return (e == cudaSuccess && bad == 0) ? 0 : 1;
}
