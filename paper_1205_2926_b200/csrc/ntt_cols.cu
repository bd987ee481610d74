// ntt_cols.cu -- the register-direct four-step column pass (k_cols): the fallback of the TMA-staged
// k_cols_tma (ntt_cols_tma.cu) for tiles it does not take (NTT_DISABLE_TMA=1, unaligned views, and
// the distributed entry points' shard layouts it cannot map).  Split from ntt_kernels.cu so the two
// translation units compile in parallel.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"
#include "modarith.cuh"
#include "rounds.cuh"
#include "fourstep.cuh"

namespace nttb {

// ----------------------------------------------------------------- four-step column pass
// Tile = N rows x C columns (C*sizeof(W) = 128 bytes), threads (t, cc) with cc
// fastest, so every global access is a full 128-byte row segment and every smem
// access of a (half-)warp hits one 128-byte smem row: conflict-free, no swizzle.
template <class W> struct ColsC { static constexpr int C = 128 / sizeof(W); };

template <class W, int LOGN, int LE> struct ColsShape {
  static constexpr int N = 1 << LOGN, E = 1 << LE, T = N / E, C = ColsC<W>::C, THREADS = T * C;
  static constexpr int MINB = THREADS >= 512 ? 1 : 512 / THREADS;
  using RC = Rounds<LOGN, LE>;
  static constexpr int R = RC::R;
};

template <class W, int LOGN, int LE, bool INV, bool PLO1, int r>
__device__ __forceinline__ void cols_round(W* v, W* __restrict__ xb, W* sm, int t, int cc, uint32_t cglob,
                                           const ColsParams& prm, const TwPair<W>* __restrict__ tw,
                                           const TwPair<W>* __restrict__ fa, const TwPair<W>* __restrict__ fb,
                                           const Mod<W>& m) {
  NTT_AUDIT_STRESS();  // audit build only: per-warp random delay before the round reads its inputs
  const W p = m.p, p2 = m.p2;
  using Sh = ColsShape<W, LOGN, LE>;
  using RC = typename Sh::RC;
  constexpr int SR = RC::sr(r), LEVEL = RC::level(r);
  constexpr int S = 1 << SR, G = Sh::E >> SR;
  constexpr int D = Sh::N >> (LEVEL + SR), B = Sh::N >> LEVEL;
  constexpr int C = Sh::C;
  const uint32_t logS = prm.log_S;
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
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) {
        const int row = blk[q] * B + h * D + c[q];
        W val = xb[((size_t)row << logS) + cc];
        if constexpr (INV) {  // four-step twiddle omega^{-c rev(r)} before the inverse column NTT
          if (prm.twiddle) {
            const uint32_t rv = __brev((uint32_t)row) >> (32 - LOGN);
            const uint32_t e = ((cglob * rv) << prm.log_tw_mul);
            const uint32_t einv = (uint32_t)((((uint64_t)1 << prm.ell) - e) & (((uint64_t)1 << prm.ell) - 1));
            val = fourstep_twiddle<W, PLO1>(val, einv, prm, fa, fb, m);
          }
        }
        v[q * S + h] = val;
      }
  } else {
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) v[q * S + h] = sm[(blk[q] * B + h * D + c[q]) * C + cc];
  }
  if constexpr (!INV) dif_round<W, LOGN, SR, LEVEL, G, PLO1>(v, c, tw, m);
  else dit_round<W, LOGN, SR, LEVEL, G, PLO1>(v, c, tw, m);
  if constexpr (last) {
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) {
        const int row = blk[q] * B + h * D + c[q];
        W val = v[q * S + h];
        if constexpr (!INV) {  // four-step twiddle omega^{c rev(r)} after the forward column NTT
          if (prm.twiddle) {
            const uint32_t rv = __brev((uint32_t)row) >> (32 - LOGN);
            val = fourstep_twiddle<W, PLO1>(val, (cglob * rv) << prm.log_tw_mul, prm, fa, fb, m);
          }
          if (prm.normalize) val = norm2<W>(val, p);
        } else {
          if (prm.normalize) val = norm4<W>(val, p, p2);
        }
        NTT_AUDIT(val, prm.normalize ? p : (INV ? 2 * p2 : p2));  // the buffer left for the next pass
        xb[((size_t)row << logS) + cc] = val;
      }
  } else {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) sm[(blk[q] * B + h * D + c[q]) * C + cc] = v[q * S + h];
    __syncthreads();
    constexpr int nr = INV ? r - 1 : r + 1;
    cols_round<W, LOGN, LE, INV, PLO1, nr>(v, xb, sm, t, cc, cglob, prm, tw, fa, fb, m);
  }
}

template <class W, int LOGN, int LE, bool INV, bool PLO1>
__global__ void __launch_bounds__(ColsShape<W, LOGN, LE>::THREADS, ColsShape<W, LOGN, LE>::MINB)
    k_cols(W* __restrict__ x, ColsParams prm, const TwPair<W>* __restrict__ tw, const TwPair<W>* __restrict__ fa,
           const TwPair<W>* __restrict__ fb, W p) {
  using Sh = ColsShape<W, LOGN, LE>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);
  const int cc = threadIdx.x % Sh::C, t = threadIdx.x / Sh::C;
  const Mod<W> m = make_mod<W>(p);
  W v[Sh::E];
  const uint64_t cg_mask = ((uint64_t)1 << prm.log_colgroups) - 1;
  for (uint64_t tile = blockIdx.x; tile < prm.n_tiles; tile += gridDim.x) {
    const uint64_t bq = tile >> prm.log_colgroups, cg = tile & cg_mask;
    // block bq spans N*S words; this tile covers columns [cg*C, cg*C + C)
    W* xb = x + (bq << (LOGN + prm.log_S)) + cg * Sh::C;
    uint32_t cloc = (uint32_t)(cg * Sh::C + cc);
    uint32_t cglob = cloc;
    if (prm.shard) {  // local flat column -> global column of the N1 x N2 matrix
      const uint32_t rb = cloc >> prm.log_local_w, cl = cloc & ((1u << prm.log_local_w) - 1);
      cglob = (rb << prm.log_n2) | (prm.col0 + cl);
    }
    constexpr int r0 = INV ? Sh::R - 1 : 0;
    cols_round<W, LOGN, LE, INV, PLO1, r0>(v, xb, sm, t, cc, cglob, prm, tw, fa, fb, m);
  }
}


static int num_sms() {
  static PerDevice cache;
  return cache.get([] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  });
}

template <class KernelT> static int occupancy(KernelT k, int threads, size_t smem) {
  int blocks = 0;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, threads, smem);
  return blocks > 0 ? blocks : 1;
}

template <class W, int LOGN> struct ColsLE {
  static constexpr int value = sizeof(W) == 8 ? 4 : (LOGN < 5 ? LOGN : 5);
};

template <class W, int LOGN, bool INV, bool PLO1>
static cudaError_t run_cols(void* x, const ColsParams& prm, const DevTables& t, uint64_t p, cudaStream_t s) {
  constexpr int LE = ColsLE<W, LOGN>::value;
  using Sh = ColsShape<W, LOGN, LE>;
  const size_t smem = (size_t)Sh::N * Sh::C * sizeof(W);
  auto kern = k_cols<W, LOGN, LE, INV, PLO1>;
  static PerDevice occ_cache;
  const int occ = occ_cache.get([&] { return occupancy(kern, Sh::THREADS, smem); });
  const uint64_t maxg = (uint64_t)occ * num_sms();
  const unsigned grid = (unsigned)(prm.n_tiles < maxg ? prm.n_tiles : maxg);
  if (!grid) return cudaSuccess;
  kern<<<grid, Sh::THREADS, smem, s>>>(reinterpret_cast<W*>(x), prm,
                                       reinterpret_cast<const TwPair<W>*>(INV ? t.sub_inv : t.sub_fwd),
                                       reinterpret_cast<const TwPair<W>*>(t.fa),
                                       reinterpret_cast<const TwPair<W>*>(t.fb), (W)p);
  return cudaGetLastError();
}

// compile-time dispatch over LOGN
template <class W, bool INV, int LO, int HI>
static cudaError_t cols_dispatch(int logn, void* x, const ColsParams& prm, const DevTables& t, uint64_t p,
                                 cudaStream_t s) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (logn == LO) {
      if constexpr (sizeof(W) == 8) {
        if ((p & 0xffffffffull) == 1) return run_cols<W, LO, INV, true>(x, prm, t, p, s);
      }
      return run_cols<W, LO, INV, false>(x, prm, t, p, s);
    }
    return cols_dispatch<W, INV, LO + 1, HI>(logn, x, prm, t, p, s);
  }
}

cudaError_t launch_cols(int wbytes, int logn, bool inverse, void* x, const ColsParams& prm, const DevTables& t,
                        uint64_t p, cudaStream_t s) {
  if (wbytes == 8)
    return inverse ? cols_dispatch<uint64_t, true, kColsMinLog, kColsMaxLog64>(logn, x, prm, t, p, s)
                   : cols_dispatch<uint64_t, false, kColsMinLog, kColsMaxLog64>(logn, x, prm, t, p, s);
  return inverse ? cols_dispatch<uint32_t, true, kColsMinLog, kColsMaxLog32>(logn, x, prm, t, p, s)
                 : cols_dispatch<uint32_t, false, kColsMinLog, kColsMaxLog32>(logn, x, prm, t, p, s);
}

unsigned elementwise_grid(size_t n, int threads) {
  size_t g = (n + threads - 1) / threads;
  size_t cap = (size_t)num_sms() * 16;
  return (unsigned)(g < cap ? (g ? g : 1) : cap);
}

}  // namespace nttb
