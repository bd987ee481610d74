// Micro-benchmark of instruction formulations of the u64 Algorithm 3 butterfly
// on sm_100a: same arithmetic, different carry / select
// encodings, to see which keeps the fmaheavy (IMAD) pipe least loaded.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bfly_variants bfly_variants.cu
#include <cstdio>
#include <cstdint>
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

// V0: C++ adds/selects (current library code)
__device__ __forceinline__ void bf0(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t p2, uint32_t np1) {
  uint64_t s = X + Y; s = s >= p2 ? s - p2 : s;
  uint64_t T = X - Y + p2;
  uint64_t Q = __umul64hi(wp, T);
  Y = tail_plo1(Q, w * T, np1);
  X = s;
}
// V1: PTX carry chains; csub selects on the borrow of s - 2p
__device__ __forceinline__ void bf1(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t p2, uint32_t np1) {
  uint64_t s, T;
  asm("{\n\t.reg .u32 x0,x1,y0,y1,q0,q1,s0,s1,d0,d1,t0,t1,b;\n\t.reg .pred pb;\n\t"
      "mov.b64 {x0,x1}, %2;\n\tmov.b64 {y0,y1}, %3;\n\tmov.b64 {q0,q1}, %4;\n\t"
      "add.cc.u32 s0, x0, y0;\n\taddc.u32 s1, x1, y1;\n\t"
      "sub.cc.u32 d0, s0, q0;\n\tsubc.cc.u32 d1, s1, q1;\n\tsubc.u32 b, 0, 0;\n\t"
      "setp.ne.u32 pb, b, 0;\n\t"
      "selp.u32 s0, s0, d0, pb;\n\tselp.u32 s1, s1, d1, pb;\n\t"
      "sub.cc.u32 t0, x0, y0;\n\tsubc.u32 t1, x1, y1;\n\t"
      "add.cc.u32 t0, t0, q0;\n\taddc.u32 t1, t1, q1;\n\t"
      "mov.b64 %0, {s0,s1};\n\tmov.b64 %1, {t0,t1};\n\t}"
      : "=l"(s), "=l"(T) : "l"(X), "l"(Y), "l"(p2));
  uint64_t Q = __umul64hi(wp, T);
  Y = tail_plo1(Q, w * T, np1);
  X = s;
}
// V2: csub via the sign of s - 2p (s, 2p < 2^63 so s - 2p < 0 iff s < 2p)
__device__ __forceinline__ void bf2(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t p2, uint32_t np1) {
  uint64_t s = X + Y;
  int64_t d = (int64_t)(s - p2);
  s = d < 0 ? s : (uint64_t)d;
  uint64_t T = X - Y + p2;
  uint64_t Q = __umul64hi(wp, T);
  Y = tail_plo1(Q, w * T, np1);
  X = s;
}
// V3: hi64 with explicit 32-bit mul.wide + PTX carries (no zero-extension moves)
__device__ __forceinline__ uint64_t mulhi_ptx(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("{\n\t.reg .u32 a0,a1,b0,b1,l0,l1,m0,m1,n0,n1,h0,h1,c;\n\t.reg .u64 L,M,N,H;\n\t"
      "mov.b64 {a0,a1}, %1;\n\tmov.b64 {b0,b1}, %2;\n\t"
      "mul.wide.u32 L, a0, b0;\n\tmul.wide.u32 M, a0, b1;\n\tmul.wide.u32 N, a1, b0;\n\tmul.wide.u32 H, a1, b1;\n\t"
      "mov.b64 {l0,l1}, L;\n\tmov.b64 {m0,m1}, M;\n\tmov.b64 {n0,n1}, N;\n\tmov.b64 {h0,h1}, H;\n\t"
      "add.cc.u32 l1, l1, m0;\n\taddc.cc.u32 h0, h0, m1;\n\taddc.u32 h1, h1, 0;\n\t"
      "add.cc.u32 l1, l1, n0;\n\taddc.cc.u32 h0, h0, n1;\n\taddc.u32 h1, h1, 0;\n\t"
      "mov.b64 %0, {h0,h1};\n\t}"
      : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void bf3(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t p2, uint32_t np1) {
  uint64_t s = X + Y;
  int64_t d = (int64_t)(s - p2);
  s = d < 0 ? s : (uint64_t)d;
  uint64_t T = X - Y + p2;
  uint64_t Q = mulhi_ptx(wp, T);
  Y = tail_plo1(Q, w * T, np1);
  X = s;
}

template <int V>
__global__ void __launch_bounds__(256) k(uint64_t* sink, uint64_t p, uint64_t w, uint64_t wp, unsigned iters) {
  uint64_t x[8], y[8];
  const uint64_t p2 = 2 * p;
  const uint32_t np1 = 0u - (uint32_t)(p >> 32);
  for (int c = 0; c < 8; ++c) { x[c] = (threadIdx.x * 7ull + c) % p; y[c] = (threadIdx.x * 13ull + 3 * c) % p; }
  for (unsigned i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (V == 0) bf0(x[c], y[c], w, wp, p2, np1);
      if (V == 1) bf1(x[c], y[c], w, wp, p2, np1);
      if (V == 2) bf2(x[c], y[c], w, wp, p2, np1);
      if (V == 3) bf3(x[c], y[c], w, wp, p2, np1);
    }
  uint64_t s = 0;
  for (int c = 0; c < 8; ++c) s ^= x[c] ^ y[c];
  if (s == 0x1234) sink[0] = s;
}

// correctness against the plain formula
template <int V>
__global__ void check(uint64_t* out, const uint64_t* xs, const uint64_t* ys, uint64_t p, uint64_t w, uint64_t wp, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t X = xs[i], Y = ys[i];
  const uint64_t p2 = 2 * p;
  const uint32_t np1 = 0u - (uint32_t)(p >> 32);
  if (V == 0) bf0(X, Y, w, wp, p2, np1);
  if (V == 1) bf1(X, Y, w, wp, p2, np1);
  if (V == 2) bf2(X, Y, w, wp, p2, np1);
  if (V == 3) bf3(X, Y, w, wp, p2, np1);
  out[2 * i] = X;
  out[2 * i + 1] = Y;
}

int main() {
  const uint64_t p = 4179340454199820289ull, w = 3233568307201063014ull;
  const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* d;
  cudaMalloc(&d, 1 << 20);
  const int n = 4096;
  uint64_t hx[n], hy[n];
  for (int i = 0; i < n; ++i) { hx[i] = (i * 0x9E3779B97F4A7C15ull) % (2 * p); hy[i] = (i * 0xD1B54A32D192ED03ull) % (2 * p); }
  hx[0] = 2 * p - 1; hy[1] = 2 * p - 1;
  uint64_t *dx, *dy, *dout;
  cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8); cudaMalloc(&dout, 2 * n * 8);
  cudaMemcpy(dx, hx, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, hy, n * 8, cudaMemcpyHostToDevice);
  static uint64_t ref[2 * n], got[2 * n];
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto bench = [&](auto kern, auto chk, const char* name) {
    chk<<<n / 256, 256>>>(dout, dx, dy, p, w, wp, n);
    cudaMemcpy(got, dout, 2 * n * 8, cudaMemcpyDeviceToHost);
    bool same = true;
    for (int i = 0; i < 2 * n; ++i) same &= got[i] == ref[i];
    const int grid = sms * 8, iters = 2048;
    for (int r = 0; r < 3; ++r) kern<<<grid, 256>>>(d, p, w, wp, iters);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<grid, 256>>>(d, p, w, wp, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bfly = 5.0 * grid * 256 * 8 * iters;
    printf("{\"variant\": \"%s\", \"Gbfly_s\": %.1f, \"bitexact_vs_V0\": %s}\n", name, bfly / (ms * 1e-3) / 1e9,
           same ? "true" : "false");
  };
  check<0><<<n / 256, 256>>>(dout, dx, dy, p, w, wp, n);
  cudaMemcpy(ref, dout, 2 * n * 8, cudaMemcpyDeviceToHost);
  bench(k<0>, check<0>, "V0 C++ (library)");
  bench(k<1>, check<1>, "V1 PTX carries, borrow select");
  bench(k<2>, check<2>, "V2 sign-of-difference csub");
  bench(k<3>, check<3>, "V3 V2 + PTX mul.wide hi64");
  return 0;
}
