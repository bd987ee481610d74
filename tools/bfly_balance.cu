// Register-only throughput of u64 Algorithm 3 butterfly formulations on
// sm_100a, to test the instruction-cost model of DESIGN.md §7: IMAD.WIDE/IMAD.HI do not overlap
// ALU work, plain IMAD does.  Variant B moves 64-bit add/sub high words and the conditional -2p
// onto the FMA pipe (IMAD.X with a runtime multiplier `one` ptxas cannot fold).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bfly_balance bfly_balance.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t tail_plo1(uint64_t Q, uint64_t WT, uint32_t np1) {
  uint64_t r;
  asm("{\n\t.reg .u32 q0,q1,r0,r1;\n\t"
      "mov.b64 {q0,q1}, %1;\n\tmov.b64 {r0,r1}, %2;\n\t"
      "sub.cc.u32 r0, r0, q0;\n\tsubc.u32 r1, r1, q1;\n\t"
      "mad.lo.u32 r1, q0, %3, r1;\n\t"
      "mov.b64 %0, {r0,r1};\n\t}"
      : "=l"(r) : "l"(Q), "l"(WT), "r"(np1));
  return r;
}

// A: library formulation (modarith.cuh)
__device__ __forceinline__ void bfA(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t p2, uint32_t np1,
                                    uint32_t one, uint64_t mp2) {
  const int64_t d = (int64_t)(X + Y - p2);
  const uint64_t s = d < 0 ? X + Y : (uint64_t)d;
  const uint64_t T = X - Y + p2;
  const uint64_t Q = __umul64hi(wp, T);
  Y = tail_plo1(Q, w * T, np1);
  X = s;
}

// B: X' = d + [d<0] 2p with d = X + Y - 2p; high words by IMAD.X (madc with runtime one),
// the add-back as IMAD of the 0/1 sign into 2p's words; tail's high word by madc.
__device__ __forceinline__ void bfB(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t p2, uint32_t np1,
                                    uint32_t one, uint64_t mp2) {
  uint64_t s, T;
  asm("{\n\t.reg .u32 x0,x1,y0,y1,a0,a1,m0,m1,d0,d1,sg,t0,t1;\n\t"
      "mov.b64 {x0,x1}, %2;\n\tmov.b64 {y0,y1}, %3;\n\tmov.b64 {a0,a1}, %4;\n\tmov.b64 {m0,m1}, %5;\n\t"
      // d = X + Y - 2p  (lo on ALU with carries, hi on FMA)
      "add.cc.u32 d0, x0, y0;\n\tmadc.lo.u32 d1, x1, %6, y1;\n\t"
      "add.cc.u32 d0, d0, m0;\n\tmadc.lo.u32 d1, d1, %6, m1;\n\t"
      // sign -> 0/1, add back sign * 2p
      "shr.u32 sg, d1, 31;\n\t"
      "mad.lo.cc.u32 d0, sg, a0, d0;\n\tmadc.lo.u32 d1, sg, a1, d1;\n\t"
      // T = X - Y + 2p = (X + 2p) - Y
      "add.cc.u32 t0, x0, a0;\n\tmadc.lo.u32 t1, x1, %6, a1;\n\t"
      "sub.cc.u32 t0, t0, y0;\n\tsubc.u32 t1, t1, y1;\n\t"
      "mov.b64 %0, {d0,d1};\n\tmov.b64 %1, {t0,t1};\n\t}"
      : "=l"(s), "=l"(T) : "l"(X), "l"(Y), "l"(p2), "l"(mp2), "r"(one));
  const uint64_t Q = __umul64hi(wp, T);
  Y = tail_plo1(Q, w * T, np1);
  X = s;
}

// C: like A but T's high word and the csub's subtraction on FMA (madc), select kept.
__device__ __forceinline__ void bfC(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t p2, uint32_t np1,
                                    uint32_t one, uint64_t mp2) {
  uint64_t s, T;
  asm("{\n\t.reg .u32 x0,x1,y0,y1,a0,a1,m0,m1,s0,s1,d0,d1,t0,t1;\n\t.reg .pred p;\n\t"
      "mov.b64 {x0,x1}, %2;\n\tmov.b64 {y0,y1}, %3;\n\tmov.b64 {a0,a1}, %4;\n\tmov.b64 {m0,m1}, %5;\n\t"
      "add.cc.u32 s0, x0, y0;\n\tmadc.lo.u32 s1, x1, %6, y1;\n\t"
      "add.cc.u32 d0, s0, m0;\n\tmadc.lo.u32 d1, s1, %6, m1;\n\t"
      "setp.lt.s32 p, d1, 0;\n\t"
      "selp.u32 s0, s0, d0, p;\n\tselp.u32 s1, s1, d1, p;\n\t"
      "add.cc.u32 t0, x0, a0;\n\tmadc.lo.u32 t1, x1, %6, a1;\n\t"
      "sub.cc.u32 t0, t0, y0;\n\tsubc.u32 t1, t1, y1;\n\t"
      "mov.b64 %0, {s0,s1};\n\tmov.b64 %1, {t0,t1};\n\t}"
      : "=l"(s), "=l"(T) : "l"(X), "l"(Y), "l"(p2), "l"(mp2), "r"(one));
  const uint64_t Q = __umul64hi(wp, T);
  Y = tail_plo1(Q, w * T, np1);
  X = s;
}

template <int V>
__global__ void __launch_bounds__(256) k(uint64_t* sink, const uint64_t* __restrict__ tw, uint64_t p, unsigned iters) {
  uint64_t x[8], y[8];
  const uint64_t p2 = 2 * p, mp2 = 0 - p2;
  const uint32_t np1 = 0u - (uint32_t)(p >> 32);
  const uint32_t one = (uint32_t)(p & 1);  // = 1 for odd p, opaque to ptxas
  for (int c = 0; c < 8; ++c) { x[c] = (threadIdx.x * 7ull + c) % p; y[c] = (threadIdx.x * 13ull + 3 * c) % p; }
#pragma unroll 1
  for (unsigned i = 0; i < iters; ++i) {
    const uint64_t w = tw[2 * (i & 63)], wp = tw[2 * (i & 63) + 1];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (V == 0) bfA(x[c], y[c], w, wp, p2, np1, one, mp2);
      if (V == 1) bfB(x[c], y[c], w, wp, p2, np1, one, mp2);
      if (V == 2) bfC(x[c], y[c], w, wp, p2, np1, one, mp2);
    }
  }
  uint64_t s = 0;
  for (int c = 0; c < 8; ++c) s ^= x[c] ^ y[c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  const uint64_t p = 4179340454199820289ull;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // twiddle table: (W, W') pairs, W = 3^(e*...) mod p by repeated multiplication
  uint64_t h[128];
  unsigned __int128 wv = 1;
  for (int e = 0; e < 64; ++e) {
    wv = wv * 3233568307201063014ull % p;
    h[2 * e] = (uint64_t)wv;
    h[2 * e + 1] = (uint64_t)(((unsigned __int128)(uint64_t)wv << 64) / p);
  }
  uint64_t *dtw, *sink;
  cudaMalloc(&dtw, sizeof h);
  cudaMemcpy(dtw, h, sizeof h, cudaMemcpyHostToDevice);
  const int grid = sms * 8, th = 256;
  cudaMalloc(&sink, (size_t)grid * th * 8);
  static uint64_t ref[148 * 8 * 256], got[148 * 8 * 256];
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const unsigned iters = 1024;
  const char* names[] = {"A library (SEL csub, IADD3 carries)", "B FMA-balanced (IMAD.X highs, IMAD sign add-back)",
                         "C FMA highs + SEL csub"};
  for (int v = 0; v < 3; ++v) {
    auto launch = [&] {
      if (v == 0) k<0><<<grid, th>>>(sink, dtw, p, iters);
      if (v == 1) k<1><<<grid, th>>>(sink, dtw, p, iters);
      if (v == 2) k<2><<<grid, th>>>(sink, dtw, p, iters);
    };
    launch();
    cudaMemcpy(v == 0 ? ref : got, sink, (size_t)grid * th * 8, cudaMemcpyDeviceToHost);
    bool same = true;
    if (v) for (int i = 0; i < grid * th; ++i) same &= got[i] == ref[i];
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bfly = 5.0 * grid * th * 8 * iters;
    printf("{\"variant\": \"%s\", \"Gbfly_s\": %.1f, \"same_as_A\": %s}\n", names[v], bfly / (ms * 1e-3) / 1e9,
           same ? "true" : "false");
  }
  return 0;
}
