// Register-only throughput of the u64 Algorithm 3 butterfly with different
// instruction formulations of hi64(W' T) (the Shoup quotient) on sm_100a, bit-exact against
// the library formulation.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bfly_hi64 bfly_hi64.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t tail_plo1(uint64_t Q, uint64_t WT, uint32_t np1) {
  uint64_t r;
  asm("{\n\t.reg .u32 q0,q1,r0,r1;\n\tmov.b64 {q0,q1}, %1;\n\tmov.b64 {r0,r1}, %2;\n\t"
      "sub.cc.u32 r0, r0, q0;\n\tsubc.u32 r1, r1, q1;\n\tmad.lo.u32 r1, q0, %3, r1;\n\tmov.b64 %0, {r0,r1};\n\t}"
      : "=l"(r) : "l"(Q), "l"(WT), "r"(np1));
  return r;
}
// V1: one mul.hi + three mul.wide, carries with add.cc (ptxas: IADD3 with two carry-outs)
__device__ __forceinline__ uint64_t hi64_v1(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("{\n\t.reg .u32 a0,a1,b0,b1,h,m1l,m1h,m2l,m2h,hl,hh,s,c,q0,q1;\n\t.reg .u64 M1,M2,HH;\n\t"
      "mov.b64 {a0,a1}, %1;\n\tmov.b64 {b0,b1}, %2;\n\t"
      "mul.hi.u32 h, a0, b0;\n\t"
      "mul.wide.u32 M1, a0, b1;\n\tmul.wide.u32 M2, a1, b0;\n\tmul.wide.u32 HH, a1, b1;\n\t"
      "mov.b64 {m1l,m1h}, M1;\n\tmov.b64 {m2l,m2h}, M2;\n\tmov.b64 {hl,hh}, HH;\n\t"
      "add.cc.u32 s, h, m1l;\n\taddc.u32 c, 0, 0;\n\tadd.cc.u32 s, s, m2l;\n\taddc.u32 c, c, 0;\n\t"
      "add.cc.u32 q0, hl, m1h;\n\taddc.u32 q1, hh, 0;\n\tadd.cc.u32 q0, q0, m2h;\n\taddc.u32 q1, q1, 0;\n\t"
      "add.cc.u32 q0, q0, c;\n\taddc.u32 q1, q1, 0;\n\tmov.b64 %0, {q0,q1};\n\t}"
      : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// V2: 64-bit accumulate: mid = hi(a0 b0) + a0 b1 (fits 64 bits), mid2 = lo32(mid) + a1 b0, hi = a1 b1 + hi32(mid) + hi32(mid2)
__device__ __forceinline__ uint64_t hi64_v2(uint64_t a, uint64_t b) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  const uint64_t mid = (uint64_t)__umulhi(a0, b0) + (uint64_t)a0 * b1;
  const uint64_t mid2 = (uint64_t)(uint32_t)mid + (uint64_t)a1 * b0;
  return (uint64_t)a1 * b1 + (mid >> 32) + (mid2 >> 32);
}
// V3: mad chain (library mulhi_chain)
__device__ __forceinline__ uint64_t hi64_v3(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("{\n\t.reg .u32 a0,a1,b0,b1,t,m1,h0,h1;\n\tmov.b64 {a0,a1}, %1;\n\tmov.b64 {b0,b1}, %2;\n\t"
      "mul.hi.u32 t, a0, b0;\n\tmad.lo.cc.u32 t, a0, b1, t;\n\tmadc.hi.u32 m1, a0, b1, 0;\n\t"
      "mad.lo.cc.u32 t, a1, b0, t;\n\tmadc.hi.cc.u32 m1, a1, b0, m1;\n\taddc.u32 h1, 0, 0;\n\t"
      "mad.lo.cc.u32 h0, a1, b1, m1;\n\tmadc.hi.u32 h1, a1, b1, h1;\n\tmov.b64 %0, {h0,h1};\n\t}"
      : "=l"(r) : "l"(a), "l"(b));
  return r;
}
template <int V> __device__ __forceinline__ uint64_t hi64(uint64_t a, uint64_t b) {
  if constexpr (V == 0 || V == 4) return __umul64hi(a, b);
  else if constexpr (V == 5) return hi64_v3(a, b);
  else if constexpr (V == 1) return hi64_v1(a, b);
  else if constexpr (V == 2) return hi64_v2(a, b);
  else return hi64_v3(a, b);
}
// conditional subtraction by the carry of x + (2^64 - m): x >= m exactly when that add carries out
__device__ __forceinline__ uint64_t csub_cc(uint64_t x, uint64_t nm) {
  uint64_t r;
  asm("{\n\t.reg .u32 x0,x1,n0,n1,d0,d1,c;\n\t.reg .pred q;\n\t"
      "mov.b64 {x0,x1}, %1;\n\tmov.b64 {n0,n1}, %2;\n\t"
      "add.cc.u32 d0, x0, n0;\n\taddc.cc.u32 d1, x1, n1;\n\taddc.u32 c, 0, 0;\n\t"
      "setp.ne.u32 q, c, 0;\n\tselp.u32 d0, d0, x0, q;\n\tselp.u32 d1, d1, x1, q;\n\t"
      "mov.b64 %0, {d0,d1};\n\t}" : "=l"(r) : "l"(x), "l"(nm));
  return r;
}
template <int V>
__device__ __forceinline__ void bf(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t p2, uint32_t np1) {
  uint64_t s = X + Y;
  if constexpr (V >= 4) {
    s = csub_cc(s, 0 - p2);
  } else {
    const int64_t d = (int64_t)(s - p2);
    s = d < 0 ? s : (uint64_t)d;
  }
  const uint64_t T = X - Y + p2;
  const uint64_t Q = hi64<V>(wp, T);
  Y = tail_plo1(Q, w * T, np1);
  X = s;
}
template <int V, int NT>
__global__ void __launch_bounds__(NT) k(uint64_t* io, uint64_t p, uint64_t w, uint64_t wp, unsigned iters) {
  uint64_t x[8], y[8];
  const uint64_t p2 = 2 * p;
  const uint32_t np1 = 0u - (uint32_t)(p >> 32);
  const size_t base = ((size_t)blockIdx.x * NT + threadIdx.x) * 16;
  for (int c = 0; c < 8; ++c) { x[c] = io[base + c]; y[c] = io[base + 8 + c]; }
  for (unsigned i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) bf<V>(x[c], y[c], w, wp, p2, np1);
  for (int c = 0; c < 8; ++c) { io[base + c] = x[c]; io[base + 8 + c] = y[c]; }
}

int main() {
  const uint64_t p = 4179340454199820289ull, w = 3233568307201063014ull;
  const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int maxblocks = sms * 8;
  const size_t words = (size_t)maxblocks * 256 * 16;
  uint64_t *d, *d0, *ref;
  cudaMalloc(&d, words * 8);
  cudaMalloc(&d0, words * 8);
  cudaMalloc(&ref, words * 8);
  uint64_t* h = (uint64_t*)malloc(words * 8);
  for (size_t i = 0; i < words; ++i) h[i] = (i * 0x9E3779B97F4A7C15ull) % (2 * p);
  cudaMemcpy(d0, h, words * 8, cudaMemcpyHostToDevice);
  uint64_t* g = (uint64_t*)malloc(words * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const unsigned iters = 2048;
  bool have_ref = false;
  auto bench = [&](auto kern, int nt, int blocks_per_sm, const char* name) {
    const int grid = sms * blocks_per_sm;
    cudaMemcpy(d, d0, words * 8, cudaMemcpyDeviceToDevice);
    kern<<<grid, nt>>>(d, p, w, wp, 4);
    cudaMemcpy(g, d, (size_t)grid * nt * 16 * 8, cudaMemcpyDeviceToHost);
    bool same = true;
    if (!have_ref) { memcpy(h, g, (size_t)grid * nt * 16 * 8); have_ref = true; }
    else for (size_t i = 0; i < (size_t)grid * nt * 16 && i < words; ++i) same &= g[i] == h[i];
    for (int r = 0; r < 2; ++r) kern<<<grid, nt>>>(d, p, w, wp, iters);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<grid, nt>>>(d, p, w, wp, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bfly = 5.0 * grid * nt * 8 * iters;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"variant\": \"%s\", \"warps_per_sm\": %d, \"Gbfly_s\": %.1f, \"warp_cycles_per_bfly_at_1965\": %.2f, \"bitexact\": %s}\n",
           name, nt / 32 * blocks_per_sm, bfly / (ms * 1e-3) / 1e9,
           (double)sms * 4 * 1.965e9 * (ms * 1e-3) / (bfly / 32), same ? "true" : "false");
  };
  // reference: the same per-thread data size at 256 threads x 4 blocks (the first call sets the reference)
  // the first call (the largest grid) sets the reference every variant must reproduce bit for bit
  for (int bps : {8, 4, 2}) {
    bench(k<0, 256>, 256, bps, "V0 __umul64hi (library)");
    bench(k<1, 256>, 256, bps, "V1 mul.hi + 3 mul.wide + add.cc");
    bench(k<2, 256>, 256, bps, "V2 64-bit accumulate");
    bench(k<3, 256>, 256, bps, "V3 mad.lo.cc/madc.hi chain");
    bench(k<4, 256>, 256, bps, "V4 library hi64 + carry csub");
    bench(k<5, 256>, 256, bps, "V5 chain hi64 + carry csub");
  }
  return 0;
}
