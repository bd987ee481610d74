// modarith.cuh -- word arithmetic and the paper's butterflies on sm_100a.
//
// Word type W is uint32_t (beta = 2^32) or uint64_t (beta = 2^64).  Every
// function is branch-free: the conditional corrections compile to ISETP+SEL
// (P:93 prefers conditional moves to branches).  Citations P:n = PAPER.md line n.
#pragma once
#include <cstdint>

#ifdef NTT_RANGE_AUDIT
#include <cuda_runtime.h>

#include "internal.h"
#endif

namespace nttb {

// ---- range audit (debug build, -DNTT_RANGE_AUDIT) ----
// Every butterfly checks the intervals its theorem states -- Theorem 2: Alg. 3 inputs
// and outputs in [0,2p), T = X - Y + 2p in [0,4p); Theorem 3: Alg. 4 in [0,4p);
// Theorem 4: Alg. 5 outputs in [0,2p); Alg. 2 canonical -- and the column passes check
// the buffers they leave in HBM (< 2p forward, < 4p inverse) and every normalised output (< p).  A
// violation increments a per-translation-unit device counter, read through ntt_audit_counts().
// d_audit_mutate = 1 drops the "+2p" of Alg. 3 line 3 (SPEC's mutation control), which the T check
// must report.  The production build compiles all of this away.
#ifdef NTT_RANGE_AUDIT
namespace {
__device__ unsigned long long d_audit_count;
__device__ unsigned long long d_audit_checks;
__device__ int d_audit_mutate;
unsigned long long audit_read_tu() {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, d_audit_count, sizeof v);
  return v;
}
void audit_reset_tu() {
  const unsigned long long z = 0;
  cudaMemcpyToSymbol(d_audit_count, &z, sizeof z);
}
void audit_mutate_tu(int on) { cudaMemcpyToSymbol(d_audit_mutate, &on, sizeof on); }
struct AuditReg {
  AuditReg() { audit_register(AuditTU{audit_read_tu, audit_reset_tu, audit_mutate_tu}); }
} audit_reg_instance;
}  // namespace
// one predicated reduction, no C++ control flow (keeps the instrumented kernels quick to compile)
__device__ __forceinline__ void audit_lt(uint64_t x, uint64_t bound) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ge.u64 p, %0, %1;\n\t@p red.global.add.u64 [%2], 1;\n\t}"
               :: "l"(x), "l"(bound), "l"(&d_audit_count) : "memory");
}
// d_audit_mutate bit 0: the mutation control; bit 1: race stress -- every round starts (before it reads its
// inputs, and again before its butterflies) with a per-warp pseudo-random delay (up to ~4 us), so warps drift apart and a missing barrier between the rounds' shared-
// memory exchanges (or a TMA buffer reused too early) would surface as wrong results (compute-sanitizer's
// racecheck is not available on the pool)
__device__ __forceinline__ bool audit_mutated() { return (*(volatile int*)&d_audit_mutate & 1) != 0; }
__device__ __forceinline__ void audit_stress_point() {
  if (*(volatile int*)&d_audit_mutate & 2) {
    uint32_t h = (uint32_t)clock64() ^ (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    __nanosleep(h & 4095u);
  }
}
#define NTT_AUDIT(x, b) ::nttb::audit_lt((uint64_t)(x), (uint64_t)(b))
#define NTT_AUDIT_MUTATED() ::nttb::audit_mutated()
#define NTT_AUDIT_STRESS() ::nttb::audit_stress_point()
#else
#define NTT_AUDIT(x, b) ((void)0)
#define NTT_AUDIT_MUTATED() false
#define NTT_AUDIT_STRESS() ((void)0)
#endif

template <class W> struct TwPair;               // (W, W') twiddle pair, stored adjacently
template <> struct alignas(8) TwPair<uint32_t> { uint32_t w, wp; };
template <> struct alignas(16) TwPair<uint64_t> { uint64_t w, wp; };

__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }
__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }
// hi64(a b) as a 32-bit multiply-add carry chain (mad.lo.cc / madc.hi): fewer IMAD.X carry fix-ups
// than __umul64hi's expansion; measured 4% faster in the inverse (Algorithm 4) kernels, and with the
// carry-select csub 2-4% in the register-only forward loop (tools/bfly_hi64.cu), so it is shoup_mul's
// default (NTT_SHOUP_CHAIN_DEFAULT=false restores __umul64hi for A/B builds).
__device__ __forceinline__ uint64_t mulhi_chain(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("{\n\t.reg .u32 a0,a1,b0,b1,t,m1,h0,h1;\n\t"
      "mov.b64 {a0,a1}, %1;\n\tmov.b64 {b0,b1}, %2;\n\t"
      "mul.hi.u32 t, a0, b0;\n\t"
      "mad.lo.cc.u32 t, a0, b1, t;\n\t"
      "madc.hi.u32 m1, a0, b1, 0;\n\t"
      "mad.lo.cc.u32 t, a1, b0, t;\n\t"
      "madc.hi.cc.u32 m1, a1, b0, m1;\n\t"
      "addc.u32 h1, 0, 0;\n\t"
      "mad.lo.cc.u32 h0, a1, b1, m1;\n\t"
      "madc.hi.u32 h1, a1, b1, h1;\n\t"
      "mov.b64 %0, {h0,h1};\n\t}"
      : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Conditional subtraction x >= m ? x - m : x (every use: x < 2m, m in {p, 2p}, p < beta/4).
// u64 selects on the carry of x + (2^64 - m) (round 2; the sign test of x - m with NTT_CSUB_SIGN,
// round 1's form); u32 uses min(x, x - m) (one VIADDMNMX).
template <class W> __device__ __forceinline__ W csub(W x, W m);
template <> __device__ __forceinline__ uint64_t csub<uint64_t>(uint64_t x, uint64_t m) {
#ifndef NTT_CSUB_SIGN
  // x + (2^64 - m) carries out exactly when x >= m: the carry of the high word's add is the select
  // predicate (IADD3, IADD3.X with carry-out, 2 SEL), one instruction fewer than the sign test of
  // x - m (tools/bfly_hi64.cu); 2^64 - m is loop-invariant and hoisted
  uint64_t r;
  asm("{\n\t.reg .u32 x0,x1,n0,n1,d0,d1,c;\n\t.reg .pred q;\n\t"
      "mov.b64 {x0,x1}, %1;\n\tmov.b64 {n0,n1}, %2;\n\t"
      "add.cc.u32 d0, x0, n0;\n\taddc.cc.u32 d1, x1, n1;\n\taddc.u32 c, 0, 0;\n\t"
      "setp.ne.u32 q, c, 0;\n\tselp.u32 d0, d0, x0, q;\n\tselp.u32 d1, d1, x1, q;\n\t"
      "mov.b64 %0, {d0,d1};\n\t}" : "=l"(r) : "l"(x), "l"(0 - m));
  return r;
#else
  const int64_t d = (int64_t)(x - m);
  return d < 0 ? x : (uint64_t)d;
#endif
}
template <> __device__ __forceinline__ uint32_t csub<uint32_t>(uint32_t x, uint32_t m) { return umin(x, x - m); }

// Modulus context kept in registers: p, 2p and (for beta = 2^64 with
// p = 1 mod 2^32) np1 = -(p >> 32) mod 2^32, which turns lo64(Q p) into one IMAD.
template <class W> struct Mod {
  W p, p2;
  uint32_t np1;
  W J;  // p^{-1} mod beta (Algorithm 5 only)
};
template <class W> __device__ __forceinline__ Mod<W> make_mod(W p) {
  Mod<W> m;
  m.p = p;
  m.p2 = 2 * p;
  m.np1 = (uint32_t)(0u - (uint32_t)((uint64_t)p >> 32));
  W j = p;  // Newton: 3 correct bits for odd p, doubling each step
#pragma unroll
  for (int i = 0; i < 6; ++i) j *= (W)2 - p * j;
  m.J = j;
  return m;
}

// Shoup multiplication (Theorem 1 bound P:85): for any T < beta,
// returns WT - Qp in [0, 2p), congruent to W*T mod p, Q = floor(W'T/beta).
// PLO1 (beta = 2^64, p = 1 mod 2^32): Qp mod beta = Q + (q0 * p_hi) << 32, so the
// low product costs one 32-bit IMAD instead of a 64 x 64 -> 64 multiply.
#ifndef NTT_SHOUP_CHAIN_DEFAULT
#define NTT_SHOUP_CHAIN_DEFAULT true
#endif
template <class W, bool PLO1 = false, bool CHAIN = NTT_SHOUP_CHAIN_DEFAULT>
__device__ __forceinline__ W shoup_mul(W T, W w, W wp, const Mod<W>& m) {
  W Q;
  if constexpr (sizeof(W) == 8 && CHAIN) Q = mulhi_chain(wp, T);
  else Q = mulhi(wp, T);
  if constexpr (sizeof(W) == 8 && PLO1) {
    const uint64_t WT = (uint64_t)w * (uint64_t)T;
    uint64_t r;
    asm("{\n\t.reg .u32 q0,q1,r0,r1;\n\t"
        "mov.b64 {q0,q1}, %1;\n\tmov.b64 {r0,r1}, %2;\n\t"
        "sub.cc.u32 r0, r0, q0;\n\tsubc.u32 r1, r1, q1;\n\t"
        "mad.lo.u32 r1, q0, %3, r1;\n\t"
        "mov.b64 %0, {r0,r1};\n\t}"
        : "=l"(r) : "l"((uint64_t)Q), "l"(WT), "r"(m.np1));
    return (W)r;
  } else {
    return w * T - Q * m.p;  // mod beta
  }
}
// Plain-modulus overload (pointwise / debug paths).
template <class W> __device__ __forceinline__ W shoup_mul(W T, W w, W wp, W p) {
  W Q = mulhi(wp, T);
  return w * T - Q * p;
}

// Algorithm 3, the modified Shoup butterfly:
// X, Y in [0,2p) -> X' = X+Y, Y' = W(X-Y), both in [0,2p)  (Theorem 2).
template <class W, bool PLO1 = false>
__device__ __forceinline__ void bfly_alg3(W& X, W& Y, W w, W wp, const Mod<W>& m) {
  NTT_AUDIT(X, m.p2);
  NTT_AUDIT(Y, m.p2);
  W s = csub<W>(X + Y, m.p2);  // lines 1-2
  W T = X - Y + m.p2;          // line 3: T in [0,4p), no correction
  if (NTT_AUDIT_MUTATED()) T = X - Y;  // mutation control (audit build only)
  NTT_AUDIT(T, 2 * m.p2);
  Y = shoup_mul<W, PLO1>(T, w, wp, m);  // lines 4-5: [0,2p), no correction
  X = s;
  NTT_AUDIT(X, m.p2);
  NTT_AUDIT(Y, m.p2);
}
template <class W> __device__ __forceinline__ void bfly_alg3(W& X, W& Y, W w, W wp, W p, W p2) {
  bfly_alg3<W, false>(X, Y, w, wp, Mod<W>{p, p2, 0u, 0});
}

// W = 1 butterflies (O(L) butterflies have W = 1 and are cheaper):
// X' as in Alg. 3, Y' = T reduced once by 2p, so Y' in [0,2p), no multiply.
template <class W> __device__ __forceinline__ void bfly_alg3_w1(W& X, W& Y, W p2) {
  NTT_AUDIT(X, p2);
  NTT_AUDIT(Y, p2);
  W s = csub<W>(X + Y, p2);
  W T0 = X - Y + p2;
  if (NTT_AUDIT_MUTATED()) T0 = X - Y;
  NTT_AUDIT(T0, 2 * p2);
  W T = csub<W>(T0, p2);
  X = s;
  Y = T;
  NTT_AUDIT(X, p2);
  NTT_AUDIT(Y, p2);
}

// The W = 1 butterfly without its two corrections, outputs in [0,4p): X + Y and X - Y + 2p (congruent
// to X + Y and X - Y).  Only where a Shoup / Montgomery product follows on every output (dif_round
// LAZY_LAST), which accepts any T < beta and returns [0,2p).
template <class W> __device__ __forceinline__ void bfly_alg3_w1_lazy(W& X, W& Y, W p2) {
  NTT_AUDIT(X, p2);
  NTT_AUDIT(Y, p2);
  const W s = X + Y;
  W T = X - Y + p2;
  if (NTT_AUDIT_MUTATED()) T = X - Y;
  NTT_AUDIT(T, 2 * p2);
  X = s;
  Y = T;
}

// Algorithm 4, the modified inverse butterfly:
// X, Y in [0,4p) -> X' = X + WY, Y' = X - WY, both in [0,4p)  (Theorem 3).
template <class W, bool PLO1 = false>
__device__ __forceinline__ void bfly_alg4(W& X, W& Y, W w, W wp, const Mod<W>& m) {
  NTT_AUDIT(X, 2 * m.p2);
  NTT_AUDIT(Y, 2 * m.p2);
  W x = csub<W>(X, m.p2);                   // line 1
  W T = shoup_mul<W, PLO1, true>(Y, w, wp, m);  // lines 2-3: Y < 4p < beta is a legal Shoup input
  NTT_AUDIT(T, m.p2);
  X = x + T;
  Y = x - T + m.p2;
  NTT_AUDIT(X, 2 * m.p2);
  NTT_AUDIT(Y, 2 * m.p2);
}
template <class W> __device__ __forceinline__ void bfly_alg4(W& X, W& Y, W w, W wp, W p, W p2) {
  bfly_alg4<W, false>(X, Y, w, wp, Mod<W>{p, p2, 0u, 0});
}

// Algorithm 4 given the NEGATED twiddle (wn, wn') = (-W mod p, its Shoup W'), as read from the
// forward table (omega^{-e} = -omega^{N/2-e}, so no inverse table is stored):
// T~ = Shoup(wn, Y) = -WY mod p in [0,2p), and the two outputs of lines 4-5 swap their formulas:
// X' = X - T~ + 2p = X + WY, Y' = X + T~ = X - WY (mod p), both still in [0,4p) (Theorem 3's
// bounds, with T~ in place of T).
template <class W, bool PLO1 = false>
__device__ __forceinline__ void bfly_alg4n(W& X, W& Y, W wn, W wnp, const Mod<W>& m) {
  NTT_AUDIT(X, 2 * m.p2);
  NTT_AUDIT(Y, 2 * m.p2);
  W x = csub<W>(X, m.p2);                       // line 1
  W T = shoup_mul<W, PLO1, true>(Y, wn, wnp, m);  // lines 2-3 with -W
  NTT_AUDIT(T, m.p2);
  X = x - T + m.p2;
  Y = x + T;
  NTT_AUDIT(X, 2 * m.p2);
  NTT_AUDIT(Y, 2 * m.p2);
}

// W = 1 inverse butterfly: T = Y reduced once by 2p (Y < 4p -> T < 2p).
template <class W> __device__ __forceinline__ void bfly_alg4_w1(W& X, W& Y, W p2) {
  NTT_AUDIT(X, 2 * p2);
  NTT_AUDIT(Y, 2 * p2);
  W x = csub<W>(X, p2);
  W T = csub<W>(Y, p2);
  X = x + T;
  Y = x - T + p2;
  NTT_AUDIT(X, 2 * p2);
  NTT_AUDIT(Y, 2 * p2);
}

// Algorithm 2, NTL's butterfly, canonical [0,p) in and out (ablation F1).
// "if T < 0" is realised as X < Y.
template <class W> __device__ __forceinline__ void bfly_alg2(W& X, W& Y, W w, W wp, W p) {
  W s = csub<W>(X + Y, p);
  W T = (X < Y) ? X - Y + p : X - Y;
  W r = csub<W>(shoup_mul<W>(T, w, wp, p), p);
  X = s;
  Y = r;
}

// Algorithm 2 inside the transform kernels (ablation F1), same Shoup core as Alg. 3.
template <class W, bool PLO1>
__device__ __forceinline__ void bfly_alg2m(W& X, W& Y, W w, W wp, const Mod<W>& m) {
  NTT_AUDIT(X, m.p);
  NTT_AUDIT(Y, m.p);
  W s = csub<W>(X + Y, m.p);                        // lines 1-2
  W T = (X < Y) ? X - Y + m.p : X - Y;               // lines 3-4 (X < Y realises T < 0)
  Y = csub<W>(shoup_mul<W, PLO1>(T, w, wp, m), m.p);  // lines 5-7
  X = s;
  NTT_AUDIT(X, m.p);
  NTT_AUDIT(Y, m.p);
}
template <class W> __device__ __forceinline__ void bfly_alg2_w1(W& X, W& Y, W p) {
  NTT_AUDIT(X, p);
  NTT_AUDIT(Y, p);
  W s = csub<W>(X + Y, p);
  Y = (X < Y) ? X - Y + p : X - Y;
  X = s;
}

// Full product hi/lo for Algorithm 5.
__device__ __forceinline__ void mul_wide(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
  uint64_t r = (uint64_t)a * b;
  hi = (uint32_t)(r >> 32);
  lo = (uint32_t)r;
}
__device__ __forceinline__ void mul_wide(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  hi = __umul64hi(a, b);
  lo = a * b;
}

// Algorithm 5, the modified Montgomery butterfly; wm = beta W mod p,
// J = p^{-1} mod beta.  X, Y in [0,2p) -> [0,2p)  (Theorem 4).
template <class W> __device__ __forceinline__ void bfly_alg5(W& X, W& Y, W wm, W J, W p, W p2) {
  W s = csub<W>(X + Y, p2);
  W T = X - Y + p2;
  W R1, R0;
  mul_wide(wm, T, R1, R0);  // line 4
  W Q = R0 * J;             // line 5
  W H = mulhi(Q, p);        // line 6
  Y = R1 - H + p;           // line 7
  X = s;
}

template <class W> __device__ __forceinline__ void bfly_alg5m(W& X, W& Y, W wm, const Mod<W>& m) {
  NTT_AUDIT(X, m.p2);
  NTT_AUDIT(Y, m.p2);
  bfly_alg5<W>(X, Y, wm, m.J, m.p, m.p2);
  NTT_AUDIT(X, m.p2);
  NTT_AUDIT(Y, m.p2);
}

// Algorithm 5's multiply alone (lines 4-7): T * W mod p for wm = beta W mod p, any T < beta
// (R1 < p because wm < p), result in (0, 2p).  The four-step twiddle product of Alg. 5 plans.
template <class W> __device__ __forceinline__ W mont_mul(W T, W wm, const Mod<W>& m) {
  W R1, R0;
  mul_wide(wm, T, R1, R0);
  W Q = R0 * m.J;
  W H = mulhi(Q, m.p);
  return R1 - H + m.p;
}

// The forward butterfly of a plan (BF: 3 = Algorithm 3, the hot path; 2 = Algorithm 2 and 5 =
// Algorithm 5, the ablations F1 / F2 of SURVEY.md 8(f)).  (w, wp): the (W, W') pair; Alg. 5 uses w
// only, holding beta W mod p.
template <class W, bool PLO1, int BF>
__device__ __forceinline__ void bfly_fwd(W& X, W& Y, W w, W wp, const Mod<W>& m) {
  if constexpr (BF == 2) bfly_alg2m<W, PLO1>(X, Y, w, wp, m);
  else if constexpr (BF == 5) bfly_alg5m<W>(X, Y, w, m);
  else bfly_alg3<W, PLO1>(X, Y, w, wp, m);
}
// ... its W = 1 case
template <class W, int BF> __device__ __forceinline__ void bfly_fwd_w1(W& X, W& Y, const Mod<W>& m) {
  if constexpr (BF == 2) bfly_alg2_w1<W>(X, Y, m.p);
  else bfly_alg3_w1<W>(X, Y, m.p2);
}
// ... and its twiddle product T * W (four-step twiddle): Shoup (BF 2 keeps Algorithm 2's canonical
// operands), Montgomery for BF 5.
template <class W, bool PLO1, int BF>
__device__ __forceinline__ W twiddle_mul(W T, W w, W wp, const Mod<W>& m) {
  W r;
  if constexpr (BF == 5) r = mont_mul<W>(T, w, m);
  else if constexpr (BF == 2) r = csub<W>(shoup_mul<W, PLO1>(T, w, wp, m), m.p);
  else r = shoup_mul<W, PLO1>(T, w, wp, m);
  NTT_AUDIT(r, BF == 2 ? m.p : m.p2);
  return r;
}

// Final normalisation: [0,2p) -> [0,p) and [0,4p) -> [0,p).
template <class W> __device__ __forceinline__ W norm2(W x, W p) {
  NTT_AUDIT(x, 2 * p);
  const W y = csub<W>(x, p);
  NTT_AUDIT(y, p);
  return y;
}
template <class W> __device__ __forceinline__ W norm4(W x, W p, W p2) {
  NTT_AUDIT(x, 2 * p2);
  const W y = csub<W>(csub<W>(x, p2), p);
  NTT_AUDIT(y, p);
  return y;
}

// Pointwise product of two data values (no reusable W', so no Shoup; P:21 use):
// returns a*b*R^{-1}-style Montgomery REDC in the Alg. 5 pattern:
// for a, b < 2p: ab < 4p^2 < p beta, so R1 < p and the result lies in (0, 2p),
// congruent to a b beta^{-1} mod p.
template <class W> __device__ __forceinline__ W mont_redc_mul(W a, W b, W J, W p) {
  NTT_AUDIT(a, 2 * p);  // the REDC's precondition ab < 4p^2 < p beta
  NTT_AUDIT(b, 2 * p);
  W R1, R0;
  mul_wide(a, b, R1, R0);
  W Q = R0 * J;
  W H = mulhi(Q, p);
  return R1 - H + p;
}

}  // namespace nttb
