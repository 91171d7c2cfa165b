// gen.cu -- the seeded state generator of synth/__init__.py on the GPU.
//
// Input generation only: this file holds none of the method's arithmetic (no
// transforms, no recursion, no dynamics).  It evaluates the same counter-based
// splitmix64 hash as synth.uniform01, so a rank can generate its shard of the
// batch directly in device memory from the GLOBAL state indices (SURVEY §8(d)
// "States", §8(e)), bit-identical to the numpy generator the oracle side uses:
//
//   key  = splitmix64(seed)
//   key  = splitmix64(key ^ ((stream & 0xFFFF) << 48 | (link & 0xFFFFFFFF)))
//   z    = splitmix64(key ^ (idx * 0x9E3779B97F4A7C15))
//   u    = (z >> 11) * 2^-53                       in [0, 1)
//   x    = lo + (hi - lo) * u                      (two roundings, no FMA, as numpy)
//
// Output: x[i * ld + (b - b0)] for link i < n and global index b in [b0, b1),
// float64 or (rounded to nearest) float32.  C ABI, plain device pointers.
#include <cuda_runtime.h>
#include <cstdint>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void uniform_states_kernel(uint64_t seed, int stream, int n, int64_t b0, int64_t count, double lo,
                                      double span, T* __restrict__ out, int64_t ld) {
  const int i = blockIdx.y;                          // link
  const uint64_t key0 = splitmix64(seed);
  const uint64_t key = splitmix64(key0 ^ (((uint64_t)(stream & 0xFFFF) << 48) | ((uint64_t)(uint32_t)i)));
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = (uint64_t)(b0 + j);
    const uint64_t z = splitmix64(key ^ (idx * 0x9E3779B97F4A7C15ull));
    const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    const double x = __dadd_rn(lo, __dmul_rn(span, u));
    out[(int64_t)i * ld + j] = (T)x;
  }
}

template <typename T>
int launch(uint64_t seed, int stream, int n, int64_t b0, int64_t b1, double lo, double hi, T* out, int64_t ld,
           void* cuda_stream) {
  const int64_t count = b1 - b0;
  if (n < 1 || count < 0 || ld < count || !out) return 1;
  if (count == 0) return 0;
  const int threads = 256;
  int64_t gx = (count + threads - 1) / threads;
  if (gx > 4096) gx = 4096;
  dim3 grid((unsigned)gx, (unsigned)n);
  uniform_states_kernel<T><<<grid, threads, 0, reinterpret_cast<cudaStream_t>(cuda_stream)>>>(
      seed, stream, n, b0, count, lo, hi - lo, out, ld);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

extern "C" {
// U[lo, hi) draws of synth.uniform_states(seed, stream, n, b0, b1, lo, hi) into the
// DEVICE array out [n][ld] (row i, columns 0 .. b1-b0-1); asynchronous on stream.
// Returns 0, 1 on a bad argument, 3 on a launch failure.
int synth_uniform_states_f64(uint64_t seed, int stream, int n, int64_t b0, int64_t b1, double lo, double hi,
                             double* out, int64_t ld, void* cuda_stream) {
  return launch<double>(seed, stream, n, b0, b1, lo, hi, out, ld, cuda_stream);
}
int synth_uniform_states_f32(uint64_t seed, int stream, int n, int64_t b0, int64_t b1, double lo, double hi,
                             float* out, int64_t ld, void* cuda_stream) {
  return launch<float>(seed, stream, n, b0, b1, lo, hi, out, ld, cuda_stream);
}
}
