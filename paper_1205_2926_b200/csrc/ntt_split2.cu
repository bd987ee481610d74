// ntt_split2.cu -- transforms of length 2N, N = 2^LOGH the largest on-chip length,
// on a cluster of two CTAs (one SM each), without an HBM round trip between stages.
//
// Forward (Algorithm 1): stage 1 pairs x_k with x_{k+N} (m = L/2).  CTA r of
// the pair evaluates half r of that stage straight from HBM (r = 0: X+Y; r = 1:
// W (X-Y) with W = omega^k, Algorithm 3), after which its half is an independent
// N-point transform with root omega^2 (Alg. 1 stages 2..ell) -- the per-stage
// twiddle table of the full transform, offset by N, is exactly that transform's
// table.  A cluster barrier after the loads orders the partner's reads before the
// in-place stores.  Output half r = Alg. 1's bit-reversed positions [rN, (r+1)N).
//
// Inverse (Algorithm 1 run backwards): stages ell..2 are two independent
// N-point inverse transforms (one per CTA); stage 1 (Algorithm 4 on x_k, x_{k+N},
// W = omega^{-k}) reads the partner's half through distributed shared memory.
// With PW the pointwise product c = a b L^{-1} is computed while loading, so a
// cyclic convolution needs no separate pointwise pass.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "modarith.cuh"
#include "rounds.cuh"

namespace cg = cooperative_groups;

namespace nttb {

template <class W> __device__ __forceinline__ int sswz(int i) {  // element XOR swizzle (128-byte rows)
  constexpr int S = sizeof(W) == 8 ? 4 : 5;
  return i ^ ((i >> S) & ((1 << S) - 1));
}

template <int LOGH, int LE> struct SplitShape {
  static constexpr int N = 1 << LOGH, E = 1 << LE, T = N / E;
  using RC = Rounds<LOGH, LE>;
  static constexpr int R = RC::R;
};

struct PwArgs {
  const void* a;
  const void* b;
  uint64_t J, K, Kp;  // REDC constant and the Shoup constant restoring scale (beta L^{-1} mod p)
};

template <class W, int LOGH, int LE, bool INV, bool PLO1, bool PW, int r>
__device__ __forceinline__ void split_round(W* v, W* __restrict__ xb, W* sm, int t, int rank,
                                            const TwPair<W>* __restrict__ tw_full, const Mod<W>& m,
                                            const PwArgs& pw, size_t boff, cg::cluster_group& cluster) {
  using Sh = SplitShape<LOGH, LE>;
  using RC = typename Sh::RC;
  constexpr int N = Sh::N;
  constexpr int SR = RC::sr(r), LEVEL = RC::level(r);
  constexpr int S = 1 << SR, G = Sh::E >> SR;
  constexpr int D = N >> (LEVEL + SR), B = N >> LEVEL;
  const TwPair<W>* tw_sub = tw_full + N;  // stages 2..ell of the 2N-point per-stage table
  int c[G], blk[G];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = t + Sh::T * q;
    blk[q] = g / D;
    c[q] = g % D;
  }
  constexpr bool first = INV ? (r == Sh::R - 1) : (r == 0);
  constexpr bool last = INV ? (r == 0) : (r == Sh::R - 1);
  if constexpr (first) {
    if constexpr (!INV) {
      // global stage 1 from HBM: i = h*D + c, pairs (x_i, x_{i+N})
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int h = 0; h < S; ++h) {
          const int i = h * D + c[q];
          W X = xb[i], Y = xb[i + N];
          if (rank == 0) {
            v[q * S + h] = csub<W>(X + Y, m.p2);
          } else {
            W w, wp;
            ldtw<W>(tw_full, (uint32_t)i, w, wp);
            v[q * S + h] = shoup_mul<W, PLO1>(X - Y + m.p2, w, wp, m);
          }
        }
      cluster.sync();  // both CTAs have read x_b: in-place stores below are safe
    } else {
      // this CTA's half of the bit-reversed input (contiguous runs); PW: c = a b L^{-1}
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const size_t off = (size_t)rank * N + blk[q] * S;
        if constexpr (PW) {
          W av[S], bv[S];
          load_run<W, S>(reinterpret_cast<const W*>(pw.a) + boff + off, av);
          load_run<W, S>(reinterpret_cast<const W*>(pw.b) + boff + off, bv);
#pragma unroll
          for (int h = 0; h < S; ++h) {
            W prod = mont_redc_mul<W>(av[h], bv[h], (W)pw.J, m.p);
            v[q * S + h] = shoup_mul<W>(prod, (W)pw.K, (W)pw.Kp, m.p);
          }
        } else {
          load_run<W, S>(xb + off, v + q * S);
        }
      }
      // no cluster barrier needed: the cross-half stores of the epilogue come after
      // the epilogue's cluster barrier, long after both CTAs loaded their halves
    }
  } else {
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) v[q * S + h] = sm[sswz<W>(blk[q] * B + h * D + c[q])];
  }
  if constexpr (!INV) dif_round<W, LOGH, SR, LEVEL, G, PLO1>(v, c, tw_sub, m);
  else dit_round<W, LOGH, SR, LEVEL, G, PLO1>(v, c, tw_sub, m);
  if constexpr (last) {
    if constexpr (!INV) {
#pragma unroll
      for (int i = 0; i < Sh::E; ++i) v[i] = norm2<W>(v[i], m.p);
#pragma unroll
      for (int q = 0; q < G; ++q) store_run<W, S>(xb + (size_t)rank * N + blk[q] * S, v + q * S);
    } else {
      // global stage 1 (Algorithm 4, W = omega^{-k}) across the pair through DSMEM
      __syncthreads();
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int h = 0; h < S; ++h) sm[sswz<W>(h * D + c[q])] = v[q * S + h];
      cluster.sync();
      const W* x_half = cluster.map_shared_rank(sm, 0);  // values at k
      const W* y_half = cluster.map_shared_rank(sm, 1);  // values at k + N
      constexpr int PER_CTA = N / 2;
#pragma unroll 4
      for (int j = 0; j < PER_CTA / Sh::T; ++j) {
        const int k = rank * PER_CTA + t + Sh::T * j;
        W X = x_half[sswz<W>(k)], Y = y_half[sswz<W>(k)];
        W w, wp;
        ldtw<W>(tw_full, (uint32_t)k, w, wp);
        bfly_alg4<W, PLO1>(X, Y, w, wp, m);
        xb[k] = norm4<W>(X, m.p, m.p2);
        xb[k + N] = norm4<W>(Y, m.p, m.p2);
      }
      cluster.sync();  // the partner is done reading this CTA's shared memory
    }
  } else {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) sm[sswz<W>(blk[q] * B + h * D + c[q])] = v[q * S + h];
    __syncthreads();
    constexpr int nr = INV ? r - 1 : r + 1;
    split_round<W, LOGH, LE, INV, PLO1, PW, nr>(v, xb, sm, t, rank, tw_full, m, pw, boff, cluster);
  }
}

template <class W, int LOGH, int LE, bool INV, bool PLO1, bool PW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SplitShape<LOGH, LE>::T, 1)
    k_split2(W* __restrict__ x, size_t batch, const TwPair<W>* __restrict__ tw_full, W p, PwArgs pw) {
  using Sh = SplitShape<LOGH, LE>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int t = threadIdx.x;
  const Mod<W> m = make_mod<W>(p);
  W v[Sh::E];
  const size_t pairs = gridDim.x / 2;
  for (size_t b = blockIdx.x / 2; b < batch; b += pairs) {
    const size_t boff = b * 2 * (size_t)Sh::N;
    constexpr int r0 = INV ? Sh::R - 1 : 0;
    split_round<W, LOGH, LE, INV, PLO1, PW, r0>(v, x + boff, sm, t, rank, tw_full, m, pw, boff, cluster);
    __syncthreads();
  }
}

template <class W> struct SplitLE { static constexpr int value = 5; };

template <class W, int LOGH, bool INV, bool PLO1, bool PW>
static cudaError_t run_split(void* x, size_t batch, const void* tw, uint64_t p, const PwArgs& pw, cudaStream_t s) {
  constexpr int LE = SplitLE<W>::value;
  using Sh = SplitShape<LOGH, LE>;
  const size_t smem = (size_t)Sh::N * sizeof(W);
  auto kern = k_split2<W, LOGH, LE, INV, PLO1, PW>;
  static bool init = false;
  static int sms = 148;
  if (!init) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    init = true;
  }
  size_t grid = 2 * batch;
  const size_t cap = (size_t)(sms / 2) * 2;  // one CTA per SM, pairs
  if (grid > cap) grid = cap;
  if (!grid) return cudaSuccess;
  kern<<<(unsigned)grid, Sh::T, smem, s>>>(reinterpret_cast<W*>(x), batch, reinterpret_cast<const TwPair<W>*>(tw),
                                           (W)p, pw);
  return cudaGetLastError();
}

bool split2_supported(int wbytes, int logn) {
  return logn == (wbytes == 8 ? kContigMaxLog64 : kContigMaxLog32) + 1;
}

cudaError_t launch_split2(int wbytes, int logn, bool inverse, void* x, size_t batch, const void* tw, uint64_t p,
                          const void* pw_a, const void* pw_b, uint64_t J, uint64_t K, uint64_t Kp, cudaStream_t s) {
  PwArgs pw{pw_a, pw_b, J, K, Kp};
  const bool fused = pw_a != nullptr;
  if (wbytes == 8) {
    if (logn != kContigMaxLog64 + 1) return cudaErrorInvalidValue;
    constexpr int H = kContigMaxLog64;
    const bool plo1 = (p & 0xffffffffull) == 1;
    if (!inverse) return plo1 ? run_split<uint64_t, H, false, true, false>(x, batch, tw, p, pw, s)
                              : run_split<uint64_t, H, false, false, false>(x, batch, tw, p, pw, s);
    if (fused) return plo1 ? run_split<uint64_t, H, true, true, true>(x, batch, tw, p, pw, s)
                           : run_split<uint64_t, H, true, false, true>(x, batch, tw, p, pw, s);
    return plo1 ? run_split<uint64_t, H, true, true, false>(x, batch, tw, p, pw, s)
                : run_split<uint64_t, H, true, false, false>(x, batch, tw, p, pw, s);
  }
  if (logn != kContigMaxLog32 + 1) return cudaErrorInvalidValue;
  constexpr int H = kContigMaxLog32;
  if (!inverse) return run_split<uint32_t, H, false, false, false>(x, batch, tw, p, pw, s);
  if (fused) return run_split<uint32_t, H, true, false, true>(x, batch, tw, p, pw, s);
  return run_split<uint32_t, H, true, false, false>(x, batch, tw, p, pw, s);
}

}  // namespace nttb
