// rd_async.cuh -- per-thread asynchronous global -> shared copies (cp.async,
// SASS LDGSTS) for the ABA kernel's input / workspace rings.  Each thread copies
// and later reads only its own shared-memory words, so a per-thread
// cp.async.wait_group is the only synchronisation a ring stage needs.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rd {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 4- or 8-byte copy through L1 (.ca: the only cache mode for sizes below 16)
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst_smem, const T* src) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "cp.async element");
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(smem_addr(dst_smem)), "l"(src),
               "n"((int)sizeof(T))
               : "memory");
}
// 16-byte copy straight from L2 (.cg): data written earlier in the same kernel
// by this thread (st.global writes through to L2) is read back coherently.
__device__ __forceinline__ void cp_async_16(void* dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

}  // namespace rd
