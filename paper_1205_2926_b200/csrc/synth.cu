// synth.cu -- device copy of the seeded counter-based input generator
// (definition in synth/__init__.py; test/bench infrastructure, no NTT arithmetic).
//   key  = mix64(seed ^ tensor_id * 0xD1B54A32D192ED03)
//   draw = mix64(key + (i*64 + attempt) * 0x9E3779B97F4A7C15)
//   [0,bound): top bitlen(bound) bits, rejection; attempt 63 falls back to v mod bound.
//   [0,2^bits): top `bits` bits of attempt 0.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace nttb {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

template <class W>
__global__ void k_synth(W* __restrict__ x, size_t count, uint64_t key, uint64_t start, uint64_t bound, unsigned shift) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t idx = start + i;
    uint64_t v = 0;
    if (bound) {
      for (unsigned a = 0; a < 64; ++a) {
        v = mix64(key + (idx * 64 + a) * 0x9E3779B97F4A7C15ull) >> shift;
        if (v < bound) break;
        if (a == 63) v %= bound;
      }
    } else {
      v = mix64(key + (idx * 64) * 0x9E3779B97F4A7C15ull) >> shift;
    }
    x[i] = (W)v;
  }
}

cudaError_t launch_synth(int wbytes, void* x, size_t count, uint64_t seed, uint64_t tensor_id, uint64_t start,
                         uint64_t bound, unsigned bits, cudaStream_t s) {
  if (!count) return cudaSuccess;
  const uint64_t key = mix64(seed ^ (tensor_id * 0xD1B54A32D192ED03ull));
  unsigned nb = bits;
  if (bound) {
    nb = 0;
    while (nb < 64 && (bound >> nb)) ++nb;  // bit length of bound
  }
  const unsigned shift = 64 - nb;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int th = 256;
  size_t g = (count + th - 1) / th;
  const size_t cap = (size_t)sms * 32;
  const unsigned grid = (unsigned)(g < cap ? g : cap);
  if (wbytes == 8) k_synth<uint64_t><<<grid, th, 0, s>>>((uint64_t*)x, count, key, start, bound, shift);
  else k_synth<uint32_t><<<grid, th, 0, s>>>((uint32_t*)x, count, key, start, bound, shift);
  return cudaGetLastError();
}

}  // namespace nttb
