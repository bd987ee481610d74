// ntt_cols_tma.cu -- the four-step column pass with TMA staging.
//
// Same work as k_cols (ntt_kernels.cu): a tile is N rows x one 128-byte row segment
// (C = 128 / sizeof(W) columns) of a block of the nested four-step view; the pass
// runs length-N NTTs (Algorithm 1, Algorithm 3 / 4 butterflies) down the
// C columns and applies the four-step twiddle omega^{c rev(r)} (forward: after,
// inverse: omega^{-c rev(r)} before).  Here the tile comes in through one 3-D TMA
// load (cp.async.bulk.tensor.3d; plain 128-byte rows, see NTT_COLS_SWZ) into one
// of two shared-memory buffers while the CTA computes the other, and leaves through
// a TMA bulk tensor store, so HBM latency is off the critical path of the strided
// (2^9-2^19-word stride) column accesses.  Every round of a warp touches whole
// 128-byte smem rows, so the plain row layout is bank-conflict free.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "fourstep.cuh"
#include "internal.h"
#include "modarith.cuh"
#include "rounds.cuh"
#include "tma.cuh"

namespace nttb {

// Tile layout: plain 128-byte rows (NTT_COLS_SWZ 0, default) or the TMA 128-byte swizzle (1, round 2's
// form).  Every shared-memory access of this kernel is one warp (u32) or one half-warp (u64) reading or
// writing one whole 128-byte row, so the plain layout is conflict-free too, and its addresses are a
// per-thread base plus compile-time row offsets (no XOR per access).
#ifndef NTT_COLS_SWZ
#define NTT_COLS_SWZ 0
#endif
#ifndef NTT_COLS_MIDBAR  // 1: a CTA barrier between a round's butterflies and its write-back (round 2's form)
#define NTT_COLS_MIDBAR 0
#endif
template <class W> __device__ __forceinline__ int cswz(int i) {
  if constexpr (NTT_COLS_SWZ) return tswz<W>(i);
  else return i;
}

// NTT_COLS_NC2: C4's u64 2^9 column pass gives each thread two adjacent columns (NC = 2: 16-byte shared-memory
// accesses, and every stage twiddle it loads serves both columns' butterflies), 512 threads per tile
#ifndef NTT_COLS_NC2
#define NTT_COLS_NC2 1
#endif
template <class W, int LOGN, int LE> struct ColsNC {
  static constexpr int value = (NTT_COLS_NC2 && !NTT_COLS_SWZ && sizeof(W) == 8 && LOGN == 9 && LE == 3) ? 2 : 1;
};
template <class W, int LOGN, int LE> struct ColsTmaShape {
  static constexpr int NC = ColsNC<W, LOGN, LE>::value;  // adjacent columns per thread
  static constexpr int N = 1 << LOGN, E = 1 << LE, T = N / E, C = 128 / (int)sizeof(W), THREADS = T * C / NC;
  static constexpr int TILE_BYTES = N * 128;
  static constexpr int BOX_ROWS = N < 256 ? N : 256;
  static constexpr int BOXES = N / BOX_ROWS;
  static constexpr size_t SMEM = 2 * (size_t)TILE_BYTES + 64 + NTT_SMEM_ALIGN_SLACK;
  static constexpr int MINB = THREADS >= 512 ? 1 : 512 / THREADS;
  using RC = Rounds<LOGN, LE>;
  static constexpr int R = RC::R;
  static_assert(TILE_BYTES % 1024 == 0, "tiles must keep the 1024-byte swizzle period");
};

template <class W, int LOGN, int LE, bool BM>
__device__ __forceinline__ void cols_tma_issue(const CUtensorMap* map, uint64_t tile, const ColsParams& prm,
                                               uint32_t buf, uint32_t bar) {
  using Sh = ColsTmaShape<W, LOGN, LE>;
  uint64_t b64;
  uint32_t cg;
  cols_tile_coords<BM>(tile, prm, b64, cg);
  const int bq = (int)b64, c0 = (int)cg * Sh::C;
  mbar_expect_tx(bar, Sh::TILE_BYTES);
#pragma unroll
  for (int bx = 0; bx < Sh::BOXES; ++bx) tma_load_3d(buf + bx * Sh::BOX_ROWS * 128, map, c0, bx * Sh::BOX_ROWS, bq, bar);
}

template <class W, int LOGN, int LE, bool INV, bool PLO1, int TWM, int BF, int r>
__device__ __forceinline__ void cols_tma_round(W* v, W* sm, int t, int cc, const uint32_t (&cgl)[2], const ColsParams& prm,
                                               const TwPair<W>* __restrict__ tw, const TwPair<W>* __restrict__ fa,
                                               const TwPair<W>* __restrict__ fb, const TwPair<W>* __restrict__ fm,
                                               const Mod<W>& m, const CUtensorMap* map, uint64_t next_tile,
                                               uint32_t next_buf,
                                               uint32_t next_bar, bool prefetch) {
  NTT_AUDIT_STRESS();  // audit build only: per-warp random delay before the round reads its inputs
  using Sh = ColsTmaShape<W, LOGN, LE>;
  using RC = typename Sh::RC;
  constexpr int SR = RC::sr(r), LEVEL = RC::level(r);
  constexpr int S = 1 << SR, G = Sh::E >> SR;
  constexpr int D = Sh::N >> (LEVEL + SR), B = Sh::N >> LEVEL;
  constexpr int C = Sh::C, NC = Sh::NC, E = Sh::E;
  int c[G], blk[G];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = t + Sh::T * q;
    blk[q] = g / D;
    c[q] = g % D;
  }
  // column k < NC of this thread (cc + k) keeps its words at v[k E + q S + h]
  constexpr bool first = INV ? (r == Sh::R - 1) : (r == 0);
  constexpr bool last = INV ? (r == 0) : (r == Sh::R - 1);
#pragma unroll
  for (int q = 0; q < G; ++q)
#pragma unroll
    for (int h = 0; h < S; ++h) {
      const int row = blk[q] * B + h * D + c[q];
      if constexpr (NC == 2) {
        const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(sm + row * C + cc);
        v[q * S + h] = (W)u.x;
        v[E + q * S + h] = (W)u.y;
      } else {
        v[q * S + h] = sm[cswz<W>(row * C + cc)];
      }
    }
  if constexpr (INV && first) {  // four-step twiddle omega^{-c rev(r)} before the inverse column NTT
    if (prm.twiddle) {
      const uint32_t emask = (uint32_t)((((uint64_t)1 << prm.ell)) - 1);
#pragma unroll
      for (int k = 0; k < NC; ++k)
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int h = 0; h < S; ++h) {
          const int row = blk[q] * B + h * D + c[q];
          const uint32_t rv = __brev((uint32_t)row) >> (32 - LOGN);
          const uint32_t e = (cgl[k] * rv) << prm.log_tw_mul;
          v[k * E + q * S + h] =
              fourstep_twiddle_ct<W, PLO1, TWM != 0>(v[k * E + q * S + h], (0u - e) & emask, prm.H, fa, fb, m);
        }
    }
  }
  // forward column passes multiply every output by the four-step twiddle next: the last stage's W = 1
  // butterflies skip their corrections (LAZY_LAST); prm.twiddle is 1 for every forward column pass
  if constexpr (!INV) dif_round<W, LOGN, SR, LEVEL, G, PLO1, BF, last, NC>(v, c, tw, m);
  else dit_round<W, LOGN, SR, LEVEL, G, PLO1, NC>(v, c, tw, m);
  if constexpr (!last) {
    // (no CTA barrier here: a round writes back exactly the positions each thread read, and the other
    // buffer is free since the previous tile's closing barrier; only thread 0's own store group matters)
    if constexpr (NTT_COLS_MIDBAR) __syncthreads();
    if (prefetch && threadIdx.x == 0) {  // the other buffer's store has been issued: reuse it once read
      bulk_wait_read0();
      cols_tma_issue<W, LOGN, LE, TWM == 2>(map, next_tile, prm, next_buf, next_bar);
    }
  }
  if constexpr (last) {
    if constexpr (!INV) {  // four-step twiddle omega^{c rev(r)} after the forward column NTT (every forward
      {                    // column pass has one; the lazy last stage above relies on it)
#pragma unroll
        for (int k = 0; k < NC; ++k)
#pragma unroll
        for (int q = 0; q < G; ++q)
#pragma unroll
          for (int h = 0; h < S; ++h) {
            const int row = blk[q] * B + h * D + c[q];
            W& x = v[k * E + q * S + h];
            if constexpr (TWM == 2) {  // twiddle matrix: M[row][c] = omega_B^{c rev(row)}, one product
              W w, wp;
              ldtw_bf<W, BF>(fm, ((uint32_t)row << prm.log_S) + cgl[k], w, wp);
              x = twiddle_mul<W, PLO1, BF>(x, w, wp, m);
            } else {
              const uint32_t rv = __brev((uint32_t)row) >> (32 - LOGN);
              x = fourstep_twiddle_bf<W, PLO1, TWM == 1, BF>(x, (cgl[k] * rv) << prm.log_tw_mul, prm.H, fa, fb, m);
            }
          }
      }
      if (prm.normalize) {
#pragma unroll
        for (int i = 0; i < NC * E; ++i) v[i] = norm2<W>(v[i], m.p);
      }
    } else {
      if (prm.normalize) {
#pragma unroll
        for (int i = 0; i < NC * E; ++i) v[i] = norm4<W>(v[i], m.p, m.p2);
      }
    }
  }
#ifdef NTT_RANGE_AUDIT
  if constexpr (last) {  // the buffer this pass leaves for the next one (or the final output)
#pragma unroll
    for (int i = 0; i < NC * E; ++i) NTT_AUDIT(v[i], prm.normalize ? m.p : (INV ? 2 * m.p2 : m.p2));
  }
#endif
#pragma unroll
  for (int q = 0; q < G; ++q)
#pragma unroll
    for (int h = 0; h < S; ++h) {
      const int row = blk[q] * B + h * D + c[q];
      if constexpr (NC == 2) {  // each thread rewrites exactly the positions it read
        *reinterpret_cast<ulonglong2*>(sm + row * C + cc) =
            make_ulonglong2((unsigned long long)v[q * S + h], (unsigned long long)v[E + q * S + h]);
      } else {
        sm[cswz<W>(row * C + cc)] = v[q * S + h];  // each thread rewrites exactly the positions it read
      }
    }
  if constexpr (!last) {
    __syncthreads();
    constexpr int nr = INV ? r - 1 : r + 1;
    cols_tma_round<W, LOGN, LE, INV, PLO1, TWM, BF, nr>(v, sm, t, cc, cgl, prm, tw, fa, fb, fm, m, map, next_tile,
                                                    next_buf, next_bar, false);
  }
}

template <class W, int LOGN, int LE, bool INV, bool PLO1, bool P2P, int TWM, int BF>
__global__ void __launch_bounds__(ColsTmaShape<W, LOGN, LE>::THREADS, ColsTmaShape<W, LOGN, LE>::MINB)
    k_cols_tma(const __grid_constant__ CUtensorMap tmap, ColsParams prm, const TwPair<W>* __restrict__ tw,
               const TwPair<W>* __restrict__ fa, const TwPair<W>* __restrict__ fb, const TwPair<W>* __restrict__ fm,
               W p) {
  using Sh = ColsTmaShape<W, LOGN, LE>;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t s0 = smem_u32(smem_raw);
  unsigned char* base = smem_raw + (((s0 + 1023u) & ~1023u) - s0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + 2 * (size_t)Sh::TILE_BYTES);
  // buffer / mbarrier of slot i by arithmetic, not a per-thread array (a dynamically indexed
  // array would live on the stack)
  const uint32_t buf0 = smem_u32(base), bar0 = smem_u32(&bars[0]);
  auto buf_of = [&](int i) { return buf0 + (uint32_t)i * (uint32_t)Sh::TILE_BYTES; };
  auto bar_of = [&](int i) { return bar0 + (uint32_t)i * 8u; };
  const int cc = (threadIdx.x % (Sh::C / Sh::NC)) * Sh::NC, t = threadIdx.x / (Sh::C / Sh::NC);
  const Mod<W> m = make_mod<W>(p);
  if (threadIdx.x == 0) {
    mbar_init(bar_of(0), 1);
    mbar_init(bar_of(1), 1);
    fence_mbar_init();
  }
  __syncthreads();
  // tiles: grid-stride, or (twiddle-matrix passes with bmajor == 2) one contiguous range per CTA, so a
  // CTA walks one column group through every block before the next and its matrix rows stay on chip
  uint64_t tile = blockIdx.x, tend = prm.n_tiles, tstep = gridDim.x;
  if constexpr (TWM == 2) {
    if (prm.bmajor == 2) {
      tile = prm.n_tiles * blockIdx.x / gridDim.x;
      tend = prm.n_tiles * (blockIdx.x + 1) / gridDim.x;
      tstep = 1;
    }
  }
  if (threadIdx.x == 0 && tile < tend) cols_tma_issue<W, LOGN, LE, TWM == 2>(&tmap, tile, prm, buf_of(0), bar_of(0));
  W v[Sh::E * Sh::NC];
  for (uint32_t it = 0; tile < tend; ++it, tile += tstep) {
    const int cur = it & 1;
    const uint64_t next = tile + tstep;
    if constexpr (Sh::R == 1) {  // no exchange to hide the prefetch behind: issue it now
      if (threadIdx.x == 0 && next < tend) {
        bulk_wait_read0();
        cols_tma_issue<W, LOGN, LE, TWM == 2>(&tmap, next, prm, buf_of(cur ^ 1), bar_of(cur ^ 1));
      }
    }
    mbar_wait(bar_of(cur), (it >> 1) & 1);
    uint64_t bq;
    uint32_t cg;
    cols_tile_coords<TWM == 2>(tile, prm, bq, cg);
    uint32_t cgl[2];
    cgl[0] = cols_global_column(cg * Sh::C + cc, prm);
    cgl[1] = Sh::NC == 2 ? cols_global_column(cg * Sh::C + cc + 1, prm) : cgl[0];
    W* sm = reinterpret_cast<W*>(base + (size_t)cur * Sh::TILE_BYTES);
    constexpr int r0 = INV ? Sh::R - 1 : 0;
    cols_tma_round<W, LOGN, LE, INV, PLO1, TWM, BF, r0>(v, sm, t, cc, cgl, prm, tw, fa, fb, fm, m, &tmap, next,
                                                    buf_of(cur ^ 1), bar_of(cur ^ 1), Sh::R > 1 && next < tend);
    fence_proxy_async_smem();  // generic smem writes -> visible to the async (TMA) proxy
    __syncthreads();
    if constexpr (P2P) {
      // fused all-to-all: every 16-byte chunk of the tile goes straight to the receive buffer of
      // the rank that owns its row (peer memory over NVLink; the caller's cross-rank barrier
      // orders these stores before the row pass reads them)
      const uint32_t c0 = cg * Sh::C, rmask = (1u << prm.log_rows_rank) - 1;
      constexpr int PER = 16 / (int)sizeof(W);
      for (int i = threadIdx.x; i < Sh::N * 8; i += Sh::THREADS) {
        const int row = i >> 3, k = i & 7;
        const uint4 val = lds128(reinterpret_cast<const unsigned char*>(sm) + row * 128 +
                                 ((NTT_COLS_SWZ ? (k ^ (row & 7)) : k) << 4));
        const uint64_t r = bq * Sh::N + (uint64_t)row;  // global row (the last pass's blocks are N rows x N2/G)
        W* dst = reinterpret_cast<W*>(select_peer(prm.peer, (uint32_t)(r >> prm.log_rows_rank))) +
                 ((uint64_t)prm.src_rank << (prm.log_rows_rank + prm.log_local_w)) +
                 ((uint64_t)(r & rmask) << prm.log_local_w) + c0 + (uint32_t)k * PER;
        *reinterpret_cast<uint4*>(dst) = val;
      }
      fence_proxy_async_smem();  // these generic reads precede the buffer's next TMA load
      // the next iteration's prefetch into this buffer (at the top of the loop when R == 1, else in the
      // next tile's first round, which has no CTA barrier before it): every warp must have finished
      // reading it first
      if constexpr (Sh::R == 1 || !NTT_COLS_MIDBAR) __syncthreads();
    } else if (threadIdx.x == 0) {
      const int c0 = (int)cg * Sh::C;
#pragma unroll
      for (int bx = 0; bx < Sh::BOXES; ++bx)
        tma_store_3d(&tmap, c0, bx * Sh::BOX_ROWS, (int)bq, buf_of(cur) + bx * Sh::BOX_ROWS * 128);
      bulk_commit();
    }
  }
  // the last bulk store must have read shared memory before the CTA exits (its global writes
  // complete with the grid, as CUTLASS's TMA epilogues rely on)
  if (threadIdx.x == 0) bulk_wait_read0();
}

// ----------------------------------------------------------------- host side
#ifndef NTT_COLS_LE64_9
#define NTT_COLS_LE64_9 3
#endif
// u64 2^9 columns (C4's column pass): 8 words per thread, 1024 threads per tile, three rounds of one
// group each (measured C4 -0.4% against 16 words per thread; 2^8 columns keep 16: C5 +13% with 8)
template <class W, int LOGN> struct ColsTmaLE {
  static constexpr int value =
      sizeof(W) == 8 ? (LOGN == 9 ? NTT_COLS_LE64_9 : (LOGN < 4 ? LOGN : 4)) : (LOGN < 5 ? LOGN : 5);
};

// L2 promotion of the tile loads (A/B hook NTT_COLS_L2PROMO = 0 / 128 / 256, default 256: a tile's
// 128-byte row segments pull their neighbour column group's half of each 256-byte line into L2)
static CUtensorMapL2promotion cols_l2_promotion() {
  static const int v = [] {
    const char* e = getenv("NTT_COLS_L2PROMO");
    return e ? atoi(e) : 256;
  }();
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                : (v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
}

template <class W, int LOGN, bool INV, bool PLO1, bool P2P, int TWM, int BF = 3>
static cudaError_t run_cols_tma_k(void* x, const ColsParams& prm, const DevTables& tb, uint64_t p, cudaStream_t s) {
  constexpr int LE = ColsTmaLE<W, LOGN>::value;
  using Sh = ColsTmaShape<W, LOGN, LE>;
  auto enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const uint64_t S = 1ull << prm.log_S, blocks = prm.n_tiles >> prm.log_colgroups;
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)S, (cuuint64_t)Sh::N, (cuuint64_t)blocks};
  cuuint64_t strides[2] = {(cuuint64_t)(S * sizeof(W)), (cuuint64_t)(S * Sh::N * sizeof(W))};
  cuuint32_t box[3] = {(cuuint32_t)Sh::C, (cuuint32_t)Sh::BOX_ROWS, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(&map, sizeof(W) == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, x, dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    NTT_COLS_SWZ ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    cols_l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  auto kern = k_cols_tma<W, LOGN, LE, INV, PLO1, P2P, TWM, BF>;
  static PerDevice occ_cache;
  const int occ = occ_cache.get([&] {
    int o = 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, Sh::THREADS, Sh::SMEM);
    return o > 0 ? o : 1;
  });
  const uint64_t maxg = (uint64_t)occ * sm_count();
  const unsigned grid = (unsigned)(prm.n_tiles < maxg ? prm.n_tiles : maxg);
  if (!grid) return cudaSuccess;
  kern<<<grid, Sh::THREADS, Sh::SMEM, s>>>(map, prm, reinterpret_cast<const TwPair<W>*>(INV ? tb.sub_inv : tb.sub_fwd),
                                           reinterpret_cast<const TwPair<W>*>(tb.fa),
                                           reinterpret_cast<const TwPair<W>*>(tb.fb),
                                           reinterpret_cast<const TwPair<W>*>(tb.fm), (W)p);
  return cudaGetLastError();
}

template <class W, int LOGN, bool INV, bool PLO1, bool P2P>
static cudaError_t run_cols_tma(void* x, const ColsParams& prm, const DevTables& tb, uint64_t p, cudaStream_t s) {
  if constexpr (!INV && !P2P) {
    // ablations F1 / F2 (forward column passes of Algorithm 2 / 5 plans): factored tables or the matrix
    if (prm.bf == 2 || prm.bf == 5) {
      if (!prm.matrix && !prm.H) return cudaErrorNotSupported;  // ablation plans never use direct tables
      if constexpr (sizeof(W) == 8) {
        if (prm.bf == 5) {
          if constexpr (PLO1) return cudaErrorNotSupported;  // Algorithm 5 has no p-specific product
          else return prm.matrix ? run_cols_tma_k<W, LOGN, INV, false, P2P, 2, 5>(x, prm, tb, p, s)
                                 : run_cols_tma_k<W, LOGN, INV, false, P2P, 1, 5>(x, prm, tb, p, s);
        }
        return prm.matrix ? run_cols_tma_k<W, LOGN, INV, PLO1, P2P, 2, 2>(x, prm, tb, p, s)
                          : run_cols_tma_k<W, LOGN, INV, PLO1, P2P, 1, 2>(x, prm, tb, p, s);
      } else {
        return cudaErrorNotSupported;  // beta = 2^32 multi-pass ablations: not built
      }
    }
    if (prm.matrix && tb.fm) return run_cols_tma_k<W, LOGN, INV, PLO1, P2P, 2>(x, prm, tb, p, s);
  }
  if (prm.H) return run_cols_tma_k<W, LOGN, INV, PLO1, P2P, 1>(x, prm, tb, p, s);
  return run_cols_tma_k<W, LOGN, INV, PLO1, P2P, 0>(x, prm, tb, p, s);
}

template <class W, bool INV, int LO, int HI>
static cudaError_t cols_tma_dispatch(int logn, void* x, const ColsParams& prm, const DevTables& tb, uint64_t p,
                                     cudaStream_t s) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (logn == LO) {
      // the fused all-to-all (p2p) epilogue is a separate instantiation, forward only
      if constexpr (sizeof(W) == 8) {
        if ((p & 0xffffffffull) == 1 && prm.bf != 5) {
          if constexpr (!INV) {
            if (prm.p2p) return run_cols_tma<W, LO, INV, true, true>(x, prm, tb, p, s);
          }
          return run_cols_tma<W, LO, INV, true, false>(x, prm, tb, p, s);
        }
      }
      if constexpr (!INV) {
        if (prm.p2p) return run_cols_tma<W, LO, INV, false, true>(x, prm, tb, p, s);
      }
      return run_cols_tma<W, LO, INV, false, false>(x, prm, tb, p, s);
    }
    return cols_tma_dispatch<W, INV, LO + 1, HI>(logn, x, prm, tb, p, s);
  }
}

bool cols_tma_supported(int wbytes, int logn, const ColsParams& prm, const void* x) {
  // tiles of <= 64 KiB (two buffers per CTA); TMA needs a 16-byte aligned base and row stride
  return logn >= kColsMinLog && logn <= kColsTmaMaxLog && ((uintptr_t)x & 15) == 0 &&
         (((uint64_t)wbytes << prm.log_S) % 16) == 0 && (prm.n_tiles >> prm.log_colgroups) < (1ull << 31);
}

cudaError_t launch_cols_tma(int wbytes, int logn, bool inverse, void* x, const ColsParams& prm, const DevTables& t,
                            uint64_t p, cudaStream_t s) {
  if (wbytes == 8)
    return inverse ? cols_tma_dispatch<uint64_t, true, kColsMinLog, kColsTmaMaxLog>(logn, x, prm, t, p, s)
                   : cols_tma_dispatch<uint64_t, false, kColsMinLog, kColsTmaMaxLog>(logn, x, prm, t, p, s);
  return inverse ? cols_tma_dispatch<uint32_t, true, kColsMinLog, kColsTmaMaxLog>(logn, x, prm, t, p, s)
                 : cols_tma_dispatch<uint32_t, false, kColsMinLog, kColsTmaMaxLog>(logn, x, prm, t, p, s);
}

}  // namespace nttb
