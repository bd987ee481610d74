// ntt_split2.cu -- transforms of length L = K*Q on a cluster of K CTAs (K = 2 or 4),
// Q = 2^LOGQ words per CTA, without an HBM round trip between stages.
//
// Forward (Algorithm 1): after the first s = log2 K stages, the block of
// positions [rQ, (r+1)Q) is an independent Q-point transform with root omega^K
// (stages s+1..ell), whose per-stage twiddle table is the full table's suffix from
// offset L - Q.  CTA r evaluates only its path through stages 1..s straight from HBM:
// for each j < Q it loads x_{j + tQ} (t < K) and, at stage i, keeps the sum
// (Algorithm 3 lines 1-2) or the twiddled difference (lines 3-5, W = zeta_i^{j + tQ})
// as bit (s - i) of r says.  (Stage 1 is evaluated by two CTAs when K = 4: +1/ell
// work, no data exchange.)  A cluster barrier after the loads orders every CTA's
// reads before the in-place stores; output block r = Alg. 1's positions [rQ, (r+1)Q).
//
// Inverse (Algorithm 1 run backwards): stages ell..s+1 are K independent
// Q-point inverses (one per CTA); stages s..1 (Algorithm 4, W = zeta_i^{-k}) act on
// the K values at positions j + tQ, read from the K CTAs' shared memory through
// distributed shared memory; CTA r finishes j in [rQ/K, (r+1)Q/K).  With PW the
// pointwise product c = a b L^{-1} is formed while loading, so a cyclic
// convolution needs no separate pointwise pass.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"
#include "modarith.cuh"
#include "rounds.cuh"

namespace cg = cooperative_groups;

namespace nttb {

template <class W> __device__ __forceinline__ int sswz(int i) {  // element XOR swizzle (128-byte rows)
  constexpr int S = sizeof(W) == 8 ? 4 : 5;
  return i ^ ((i >> S) & ((1 << S) - 1));
}

template <int LOGQ, int LE, int K, int WB = 8> struct SplitShape {
  static constexpr int Q = 1 << LOGQ, E = 1 << LE, T = Q / E;
  static constexpr int S_SPLIT = K == 4 ? 2 : 1;  // log2 K
  static constexpr int LOGL = LOGQ + S_SPLIT;
  // two CTAs per SM when the Q-word block fits twice in shared memory
  static constexpr int MINB = (T <= 512 && Q * WB <= 64 * 1024) ? 2 : 1;
  using RC = Rounds<LOGQ, LE>;
  static constexpr int R = RC::R;
};

struct PwArgs {
  const void* a;
  const void* b;
  uint64_t J, K, Kp;  // REDC constant and the Shoup constant restoring scale (beta L^{-1} mod p)
};

template <class W, int LOGQ, int LE, int K, bool INV, bool PLO1, bool PW, int r>
__device__ __forceinline__ void split_round(W* v, W* __restrict__ xb, W* sm, int t, int rank,
                                            const TwPair<W>* __restrict__ tw_full, const Mod<W>& m,
                                            const PwArgs& pw, size_t boff, cg::cluster_group& cluster) {
  using Sh = SplitShape<LOGQ, LE, K, (int)sizeof(W)>;
  using RC = typename Sh::RC;
  constexpr int Q = Sh::Q, SS = Sh::S_SPLIT, LOGL = Sh::LOGL;
  constexpr int SR = RC::sr(r), LEVEL = RC::level(r);
  constexpr int S = 1 << SR, G = Sh::E >> SR;
  constexpr int D = Q >> (LEVEL + SR), B = Q >> LEVEL;
  const TwPair<W>* tw_sub = tw_full + ((1 << LOGL) - Q);  // stages s+1..ell of the full per-stage table
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
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int h = 0; h < S; ++h) {
          const int j = h * D + c[q];
          W u[K];
#pragma unroll
          for (int tt = 0; tt < K; ++tt) u[tt] = xb[j + tt * Q];
          // this CTA's path through stages 1..s
#pragma unroll
          for (int i = 1; i <= SS; ++i) {
            const int cnt = K >> (i - 1);
            const bool upper = (rank >> (SS - i)) & 1;
            const int off = stage_off(LOGL, i);
#pragma unroll
            for (int tt = 0; tt < cnt / 2; ++tt) {
              const W X = u[tt], Y = u[tt + cnt / 2];
              if (!upper) {
                u[tt] = csub<W>(X + Y, m.p2);
              } else {
                W w, wp;
                ldtw<W>(tw_full, (uint32_t)(off + j + tt * Q), w, wp);
                u[tt] = shoup_mul<W, PLO1>(X - Y + m.p2, w, wp, m);
              }
            }
          }
          v[q * S + h] = u[0];
        }
      cluster.sync();  // every CTA has read x_b: in-place stores below are safe
    } else {
      // this CTA's block of the bit-reversed input (contiguous runs); PW: c = a b L^{-1}
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const size_t off = (size_t)rank * Q + blk[q] * S;
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
      // no barrier needed here: the cross-CTA stores of the epilogue follow the
      // epilogue's cluster barrier, after every CTA has loaded its block
    }
  } else {
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) v[q * S + h] = sm[sswz<W>(blk[q] * B + h * D + c[q])];
  }
  if constexpr (!INV) dif_round<W, LOGQ, SR, LEVEL, G, PLO1>(v, c, tw_sub, m);
  else dit_round<W, LOGQ, SR, LEVEL, G, PLO1>(v, c, tw_sub, m);
  if constexpr (last) {
    if constexpr (!INV) {
#pragma unroll
      for (int i = 0; i < Sh::E; ++i) v[i] = norm2<W>(v[i], m.p);
#pragma unroll
      for (int q = 0; q < G; ++q) store_run<W, S>(xb + (size_t)rank * Q + blk[q] * S, v + q * S);
    } else {
      // stages s..1 across the cluster through DSMEM (Algorithm 4)
      __syncthreads();
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int h = 0; h < S; ++h) sm[sswz<W>(h * D + c[q])] = v[q * S + h];
      cluster.sync();
      const W* part[K];
#pragma unroll
      for (int tt = 0; tt < K; ++tt) part[tt] = cluster.map_shared_rank(sm, tt);  // values at j + tt*Q
      constexpr int PER_CTA = Q / K;
#pragma unroll 2
      for (int jj = 0; jj < PER_CTA / Sh::T; ++jj) {
        const int j = rank * PER_CTA + t + Sh::T * jj;
        W u[K];
#pragma unroll
        for (int tt = 0; tt < K; ++tt) u[tt] = part[tt][sswz<W>(j)];
#pragma unroll
        for (int i = SS; i >= 1; --i) {
          const int half = K >> i;  // pairs (tt, tt + half) inside blocks of 2*half
          const int off = stage_off(LOGL, i);
#pragma unroll
          for (int bb = 0; bb < K; bb += 2 * half)
#pragma unroll
            for (int tt = 0; tt < half; ++tt) {
              W w, wp;
              ldtw<W>(tw_full, (uint32_t)(off + j + tt * Q), w, wp);
              bfly_alg4<W, PLO1>(u[bb + tt], u[bb + tt + half], w, wp, m);
            }
        }
#pragma unroll
        for (int tt = 0; tt < K; ++tt) xb[j + tt * Q] = norm4<W>(u[tt], m.p, m.p2);
      }
      cluster.sync();  // the other CTAs are done reading this CTA's shared memory
    }
  } else {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) sm[sswz<W>(blk[q] * B + h * D + c[q])] = v[q * S + h];
    __syncthreads();
    constexpr int nr = INV ? r - 1 : r + 1;
    split_round<W, LOGQ, LE, K, INV, PLO1, PW, nr>(v, xb, sm, t, rank, tw_full, m, pw, boff, cluster);
  }
}

template <class W, int LOGQ, int LE, int K, bool INV, bool PLO1, bool PW>
__global__ void __launch_bounds__(SplitShape<LOGQ, LE, K, (int)sizeof(W)>::T,
                                  SplitShape<LOGQ, LE, K, (int)sizeof(W)>::MINB)
    k_splitk(W* __restrict__ x, size_t batch, const TwPair<W>* __restrict__ tw_full, W p, PwArgs pw) {
  using Sh = SplitShape<LOGQ, LE, K, (int)sizeof(W)>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int t = threadIdx.x;
  const Mod<W> m = make_mod<W>(p);
  W v[Sh::E];
  const size_t groups = gridDim.x / K;
  for (size_t b = blockIdx.x / K; b < batch; b += groups) {
    const size_t boff = b * (size_t)K * Sh::Q;
    constexpr int r0 = INV ? Sh::R - 1 : 0;
    split_round<W, LOGQ, LE, K, INV, PLO1, PW, r0>(v, x + boff, sm, t, rank, tw_full, m, pw, boff, cluster);
    __syncthreads();
  }
}

template <class W, int K> struct SplitLE { static constexpr int value = 5; };

template <class W, int LOGL, int K, bool INV, bool PLO1, bool PW>
static cudaError_t run_split(void* x, size_t batch, const void* tw, uint64_t p, const PwArgs& pw, cudaStream_t s) {
  constexpr int LOGQ = LOGL - (K == 4 ? 2 : 1);
  constexpr int LE = SplitLE<W, K>::value;
  using Sh = SplitShape<LOGQ, LE, K, (int)sizeof(W)>;
  const size_t smem = (size_t)Sh::Q * sizeof(W);
  auto kern = k_splitk<W, LOGQ, LE, K, INV, PLO1, PW>;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  static int max_clusters = 0;
  if (!max_clusters) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(K * 1024);
    q.blockDim = dim3(Sh::T);
    q.dynamicSmemBytes = smem;
    q.attrs = attr;
    q.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &q) != cudaSuccess || max_clusters <= 0) {
      cudaGetLastError();
      max_clusters = 148 / K;
    }
  }
  const size_t groups = batch < (size_t)max_clusters ? batch : (size_t)max_clusters;
  if (!groups) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(groups * K));
  cfg.blockDim = dim3(Sh::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, reinterpret_cast<W*>(x), batch, reinterpret_cast<const TwPair<W>*>(tw),
                            (W)p, pw);
}

// K = 2 is the default: measured faster than K = 4 (C3 1.44e12 vs 1.06e12 bfly/s, C4
// 5.7e11 vs 4.5e11), whose redundant stage-1 work and four strided loads per word cost
// more than its second CTA per SM gains.  NTT_SPLIT_K=4 selects the 4-CTA variant.
static int split_k() {
  static int k = 0;
  if (!k) {
    const char* e = getenv("NTT_SPLIT_K");
    k = (e && e[0] == '4') ? 4 : 2;
  }
  return k;
}

bool split2_supported(int wbytes, int logn) {
  return logn == (wbytes == 8 ? kContigMaxLog64 : kContigMaxLog32) + 1;
}

template <class W, int LOGL, bool INV, bool PLO1, bool PW>
static cudaError_t run_split_k(void* x, size_t batch, const void* tw, uint64_t p, const PwArgs& pw, cudaStream_t s) {
  if (split_k() == 2) return run_split<W, LOGL, 2, INV, PLO1, PW>(x, batch, tw, p, pw, s);
  return run_split<W, LOGL, 4, INV, PLO1, PW>(x, batch, tw, p, pw, s);
}

cudaError_t launch_split2(int wbytes, int logn, bool inverse, void* x, size_t batch, const void* tw, uint64_t p,
                          const void* pw_a, const void* pw_b, uint64_t J, uint64_t K, uint64_t Kp, cudaStream_t s) {
  PwArgs pw{pw_a, pw_b, J, K, Kp};
  const bool fused = pw_a != nullptr;
  if (wbytes == 8) {
    if (logn != kContigMaxLog64 + 1) return cudaErrorInvalidValue;
    constexpr int L = kContigMaxLog64 + 1;
    const bool plo1 = (p & 0xffffffffull) == 1;
    if (!inverse) return plo1 ? run_split_k<uint64_t, L, false, true, false>(x, batch, tw, p, pw, s)
                              : run_split_k<uint64_t, L, false, false, false>(x, batch, tw, p, pw, s);
    if (fused) return plo1 ? run_split_k<uint64_t, L, true, true, true>(x, batch, tw, p, pw, s)
                           : run_split_k<uint64_t, L, true, false, true>(x, batch, tw, p, pw, s);
    return plo1 ? run_split_k<uint64_t, L, true, true, false>(x, batch, tw, p, pw, s)
                : run_split_k<uint64_t, L, true, false, false>(x, batch, tw, p, pw, s);
  }
  if (logn != kContigMaxLog32 + 1) return cudaErrorInvalidValue;
  constexpr int L = kContigMaxLog32 + 1;
  if (!inverse) return run_split_k<uint32_t, L, false, false, false>(x, batch, tw, p, pw, s);
  if (fused) return run_split_k<uint32_t, L, true, false, true>(x, batch, tw, p, pw, s);
  return run_split_k<uint32_t, L, true, false, false>(x, batch, tw, p, pw, s);
}

}  // namespace nttb
