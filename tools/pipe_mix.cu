// Pipe-overlap microbenchmark (sm_100a): sustained warp-instruction rates of the ALU
// (LOP3/IADD3/SEL/ISETP) and FMA-heavy (IMAD, IMAD.WIDE, IMAD.HI) pipes alone and
// interleaved, to model the butterflies' issue limits.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix pipe_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8, ITERS = 2048;

#define XOR(v, k) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(k), "r"(v))  // (a & b) ^ c
#define ADD(v, k) asm volatile("add.u32 %0, %0, %1;" : "+r"(v) : "r"(k))
#define MADLO(v, k) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(v) : "r"(k))
#define MADHI(v, k) asm volatile("mad.hi.u32 %0, %0, %1, %1;" : "+r"(v) : "r"(k))
#define WIDE(v64, v, k) asm volatile("{.reg .u32 lo, hi; mov.b64 {lo, hi}, %0; mad.wide.u32 %0, lo, %1, %0;}" : "+l"(v64) : "r"(k))
#define WIDE2(lo, hi, v, k) asm volatile("{.reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t;}" : "=r"(lo), "=r"(hi) : "r"(v), "r"(k)); v ^= hi
#define ADDC(v, w, k) asm volatile("add.cc.u32 %0, %0, %2; addc.u32 %1, %1, %2;" : "+r"(v), "+r"(w) : "r"(k))
#define SELP(v, w, k) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; selp.u32 %0, %0, %2, p;}" : "+r"(v) : "r"(w), "r"(k))

template <int MODE>
__global__ void __launch_bounds__(256) kmix(uint32_t* out, uint32_t k1, uint32_t k2) {
  uint32_t a[CH], b[CH];
  uint64_t w[CH];
  uint32_t w0[CH], w1[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { a[c] = threadIdx.x + c; b[c] = threadIdx.x * 3 + c; w[c] = c; w0[c] = c * 7; w1[c] = c * 9; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MODE == 0) { XOR(a[c], k1); XOR(b[c], k2); }                 // 2 ALU
      if (MODE == 1) { MADLO(a[c], k1); MADLO(b[c], k2); }             // 2 IMAD
      if (MODE == 2) { WIDE(w[c], a[c], k1); WIDE(w[c], b[c], k2); }   // 2 IMAD.WIDE (data-dependent multiplier)
      if (MODE == 3) { MADHI(a[c], k1); MADHI(b[c], k2); }             // 2 IMAD.HI
      if (MODE == 4) { XOR(a[c], k1); MADLO(b[c], k2); }               // 1 ALU + 1 IMAD
      if (MODE == 5) { XOR(a[c], k1); XOR(b[c], k2); WIDE(w[c], b[c], k1); }  // 2 ALU + 1 WIDE
      if (MODE == 6) { ADDC(a[c], b[c], k1); }                          // IADD3 + IADD3.X carry pair
      if (MODE == 7) { SELP(a[c], b[c], k1); SELP(b[c], a[c], k2); }   // 2 x (ISETP + SEL)
      if (MODE == 8) { XOR(a[c], k1); XOR(b[c], k2); MADHI(a[c], k2); }  // 2 ALU + 1 IMAD.HI
      if (MODE == 9) { MADHI(a[c], k1); XOR(b[c], k2); }                 // 1 IMAD.HI + 1 ALU
      if (MODE == 10) { MADHI(a[c], k1); XOR(b[c], k2); XOR(w0[c], k1); XOR(w1[c], k2); XOR(b[c], k1); }  // HI + 4 ALU
      if (MODE == 11) { MADHI(a[c], k1); MADLO(b[c], k2); }              // HI + IMAD
      if (MODE == 12) { MADHI(a[c], k1); MADLO(b[c], k2); XOR(w0[c], k1); XOR(w1[c], k2); }  // HI + IMAD + 2 ALU
      if (MODE == 13) { WIDE2(w0[c], w1[c], a[c], k1); XOR(b[c], k2); } // 1 IMAD.WIDE + 1 ALU
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c] ^ b[c] ^ (uint32_t)w[c] ^ (uint32_t)(w[c] >> 32) ^ w0[c] ^ w1[c];
  if (s == 0x12345678u) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"2 LOP3 (ALU)", "2 IMAD", "2 IMAD.WIDE", "2 IMAD.HI", "LOP3 + IMAD", "2 LOP3 + IMAD.WIDE",
                         "add.cc + addc", "2 (ISETP + SEL)", "2 LOP3 + IMAD.HI", "HI + LOP3", "HI + 4 LOP3",
                         "HI + IMAD", "HI + IMAD + 2 LOP3", "WIDE + LOP3(+xor)"};
  const int instrs[] = {2, 2, 2, 2, 2, 3, 2, 4, 3, 2, 5, 2, 4, 3};
  for (int blocks_per_sm : {8, 2}) {
    for (int mode = 0; mode < 14; ++mode) {
      auto launch = [&] {
        const int g = sms * blocks_per_sm;
        switch (mode) {
          case 0: kmix<0><<<g, 256>>>(d, 3, 5); break;
          case 1: kmix<1><<<g, 256>>>(d, 3, 5); break;
          case 2: kmix<2><<<g, 256>>>(d, 3, 5); break;
          case 3: kmix<3><<<g, 256>>>(d, 3, 5); break;
          case 4: kmix<4><<<g, 256>>>(d, 3, 5); break;
          case 5: kmix<5><<<g, 256>>>(d, 3, 5); break;
          case 6: kmix<6><<<g, 256>>>(d, 3, 5); break;
          case 7: kmix<7><<<g, 256>>>(d, 3, 5); break;
          case 8: kmix<8><<<g, 256>>>(d, 3, 5); break;
          case 9: kmix<9><<<g, 256>>>(d, 3, 5); break;
          case 10: kmix<10><<<g, 256>>>(d, 3, 5); break;
          case 11: kmix<11><<<g, 256>>>(d, 3, 5); break;
          case 12: kmix<12><<<g, 256>>>(d, 3, 5); break;
          case 13: kmix<13><<<g, 256>>>(d, 3, 5); break;
        }
      };
      for (int w = 0; w < 2; ++w) launch();
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      const double warp_instr = (double)sms * blocks_per_sm * 8 * ITERS * CH * instrs[mode];
      const double cyc = ms * 1e-3 * 1965e6;  // at the max SM clock
      printf("{\"warps_per_smsp\": %d, \"mix\": \"%s\", \"warp_instr_per_clk_per_smsp\": %.3f, \"cycles_per_group\": %.2f}\n",
             blocks_per_sm * 2, names[mode], warp_instr / (sms * 4) / cyc, instrs[mode] / (warp_instr / (sms * 4) / cyc));
    }
  }
  return 0;
}
