// Integer-pipe microbenchmark for the roofline denominators of DESIGN.md §Roofline.
// Measures, on the live B200, the sustained warp-instruction throughput of the
// multiplier opcodes the lazy Shoup butterfly (§3, Alg. 3) compiles to,
// plus the throughput of the register-only Alg.3 butterfly itself (u32 and u64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_pipe_peak int_pipe_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int CH = 8;       // independent chains per thread
constexpr int ITERS = 4096;

__global__ void k_imad_lo(uint32_t* out, uint32_t a) {
  uint32_t v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = v[c] * a + (uint32_t)c;
  uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 0x12345678u) out[0] = s;
}
__global__ void k_imad_hi(uint32_t* out, uint32_t a) {
  uint32_t v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c + 0x9e3779b9u;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = __umulhi(v[c], a) ^ (uint32_t)c;
  uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 0x12345678u) out[0] = s;
}
__global__ void k_imad_wide(uint32_t* out, uint32_t a) {
  uint64_t v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = (uint64_t)(uint32_t)v[c] * a + v[c];
  uint64_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 0x12345678u) out[0] = (uint32_t)s;
}
__global__ void k_iadd3(uint32_t* out, uint32_t a) {
  uint32_t v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = v[c] + a + (uint32_t)i;
  uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 0x12345678u) out[0] = s;
}

// Alg. 3 butterfly, register-only, u32 (β = 2^32)
__global__ void k_bfly32(uint32_t* out, uint32_t p, uint32_t W, uint32_t Wp) {
  uint32_t x[CH], y[CH];
  const uint32_t p2 = 2 * p;
  for (int c = 0; c < CH; ++c) { x[c] = (threadIdx.x * 7 + c) % p; y[c] = (threadIdx.x * 13 + 3 * c) % p; }
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint32_t X = x[c], Y = y[c];
      uint32_t s = X + Y; s = (s >= p2) ? s - p2 : s;
      uint32_t T = X - Y + p2;
      uint32_t Q = __umulhi(Wp, T);
      uint32_t r = W * T - Q * p;
      x[c] = s; y[c] = r;
    }
  uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= x[c] ^ y[c];
  if (s == 0x12345678u) out[0] = s;
}
// Alg. 3 butterfly, register-only, u64 (β = 2^64)
__global__ void k_bfly64(uint32_t* out, uint64_t p, uint64_t W, uint64_t Wp) {
  uint64_t x[CH], y[CH];
  const uint64_t p2 = 2 * p;
  for (int c = 0; c < CH; ++c) { x[c] = (threadIdx.x * 7ull + c) % p; y[c] = (threadIdx.x * 13ull + 3 * c) % p; }
  for (int i = 0; i < ITERS / 4; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint64_t X = x[c], Y = y[c];
      uint64_t s = X + Y; s = (s >= p2) ? s - p2 : s;
      uint64_t T = X - Y + p2;
      uint64_t Q = __umul64hi(Wp, T);
      uint64_t r = W * T - Q * p;
      x[c] = s; y[c] = r;
    }
  uint64_t s = 0; for (int c = 0; c < CH; ++c) s ^= x[c] ^ y[c];
  if (s == 0x12345678u) out[0] = (uint32_t)s;
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  uint32_t* d; CK(cudaMalloc(&d, 64));
  const int sms = pr.multiProcessorCount;
  const int threads = 256, blocks = sms * 8;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %.0f, \"results\": [\n", pr.name, sms, clk_khz / 1e3);
  auto run = [&](const char* name, auto launch, double ops_per_thread_iter, int iters) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double ops = (double)blocks * threads * iters * ops_per_thread_iter;
    double per_s = ops / (ms * 1e-3);
    printf("  {\"op\": \"%s\", \"ms\": %.4f, \"thread_ops_per_s\": %.4e, \"thread_ops_per_clk_per_sm_at_attr_clock\": %.2f},\n",
           name, ms, per_s, per_s / sms / (clk_khz * 1e3));
  };
  run("imad_lo_u32", [&] { k_imad_lo<<<blocks, threads>>>(d, 3u); }, CH, ITERS);
  run("imad_hi_u32", [&] { k_imad_hi<<<blocks, threads>>>(d, 0x9e3779b9u); }, CH, ITERS);
  run("imad_wide_u32", [&] { k_imad_wide<<<blocks, threads>>>(d, 0x9e3779b9u); }, CH, ITERS);
  run("iadd3", [&] { k_iadd3<<<blocks, threads>>>(d, 7u); }, CH, ITERS);
  run("bfly_alg3_u32", [&] { k_bfly32<<<blocks, threads>>>(d, 998244353u, 258648936u, (uint32_t)(((uint64_t)258648936u << 32) / 998244353u)); }, CH, ITERS);
  const uint64_t p64 = 4179340454199820289ull, W64 = 3233568307201063014ull;
  const uint64_t Wp64 = (uint64_t)(((unsigned __int128)W64 << 64) / p64);
  run("bfly_alg3_u64", [&] { k_bfly64<<<blocks, threads>>>(d, p64, W64, Wp64); }, CH, ITERS / 4);
  CK(cudaGetLastError());
  printf("  {\"op\": \"end\"}\n]}\n");
  return 0;
}
