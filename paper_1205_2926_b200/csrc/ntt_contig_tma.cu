// ntt_contig_tma.cu -- the on-chip (single-pass) transform with TMA staging.
//
// Each persistent CTA walks tiles of K consecutive transforms.  A tile is
// brought into shared memory by the Tensor Memory Accelerator
// (cp.async.bulk.tensor.2d, SWIZZLE_128B) while the CTA computes the previous
// tile (two buffers, one mbarrier each), so HBM latency is off the critical
// path and no registers are spent on loads.  The rounds of rounds.cuh then run
// out of the swizzled buffer: the TMA 128-byte swizzle (16-byte chunk index
// XOR row mod 8) keeps every round's access pattern bank-conflict free when
// contiguous runs are read as 16-byte vectors (tools/bank_sim.py).  The last
// round writes its results back into the tile, which leaves through one TMA bulk
// tensor store (cp.async.bulk.tensor.2d.global.shared::cta), so both the
// bit-reversed forward output and the natural-order inverse output are written
// as full 128-byte rows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "internal.h"
#include "modarith.cuh"
#include "rounds.cuh"
#include "tma.cuh"

namespace nttb {

// ----------------------------------------------------------------- shape
template <class W, int LOGN, int LE> struct TmaShape {
  static constexpr int N = 1 << LOGN, E = 1 << LE, T = N / E;
  static constexpr int K = T >= 256 ? 1 : 256 / T;   // transforms per tile
  static constexpr int THREADS = K * T;
#ifndef NTT_TMA_MINB_THREADS
#define NTT_TMA_MINB_THREADS 512
#endif
  static constexpr int MINB = THREADS >= NTT_TMA_MINB_THREADS ? 1 : NTT_TMA_MINB_THREADS / THREADS;
  static constexpr int TILE_WORDS = K * N;
  static constexpr int TILE_BYTES = TILE_WORDS * (int)sizeof(W);
  static constexpr int ROW_WORDS = 128 / (int)sizeof(W);
  static constexpr int TILE_ROWS = TILE_WORDS / ROW_WORDS;
  static constexpr int BOX_ROWS = TILE_ROWS < 256 ? TILE_ROWS : 256;
  static constexpr int BOXES = TILE_ROWS / BOX_ROWS;
  static constexpr int BOX_BYTES = BOX_ROWS * 128;
  static constexpr size_t SMEM = 2 * (size_t)TILE_BYTES + 64 + NTT_SMEM_ALIGN_SLACK;
  using RC = Rounds<LOGN, LE>;
  static constexpr int R = RC::R;
  static_assert(R >= 2, "TMA kernel needs at least one exchange");
  static_assert(N * sizeof(W) % 1024 == 0, "slot buffers must keep the 1024-byte swizzle period");
};

template <class W, int LOGN, int LE, bool INV, bool PLO1, int BF, int r>
__device__ __forceinline__ void tma_round(W* v, W* __restrict__ xb, W* sb, int t, bool active,
                                          const TwPair<W>* __restrict__ tw, const Mod<W>& m, bool norm,
                                          bool first_exchange, const CUtensorMap* map, size_t next_tile,
                                          size_t ntiles, uint32_t next_buf, uint32_t next_bar) {
  NTT_AUDIT_STRESS();  // audit build only: per-warp random delay before the round reads its inputs
  using Sh = TmaShape<W, LOGN, LE>;
  using RC = typename Sh::RC;
  constexpr int SR = RC::sr(r), LEVEL = RC::level(r);
  constexpr int S = 1 << SR, G = Sh::E >> SR;
  constexpr int D = Sh::N >> (LEVEL + SR), B = Sh::N >> LEVEL;
  constexpr int PER = 16 / (int)sizeof(W);
  constexpr bool VEC = (D == 1) && (S >= PER);
  int c[G], blk[G];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = t + Sh::T * q;
    blk[q] = g / D;
    c[q] = g % D;
  }
  constexpr bool last = INV ? (r == 0) : (r == Sh::R - 1);
  // ---- load from the swizzled tile buffer
#pragma unroll
  for (int q = 0; q < G; ++q) {
    if constexpr (VEC) {
#pragma unroll
      for (int h = 0; h < S; h += PER)
        unpack16<W>(lds128(sb + tswz<W>(blk[q] * B + h)), v + q * S + h);
    } else {
#pragma unroll
      for (int h = 0; h < S; ++h) v[q * S + h] = sb[tswz<W>(blk[q] * B + h * D + c[q])];
    }
  }
  // ---- compute
  if constexpr (!INV) dif_round<W, LOGN, SR, LEVEL, G, PLO1, BF>(v, c, tw, m);
  else dit_round<W, LOGN, SR, LEVEL, G, PLO1>(v, c, tw, m);
  if constexpr (last) {
    if (norm) {
#pragma unroll
      for (int i = 0; i < Sh::E; ++i) v[i] = INV ? norm4<W>(v[i], m.p, m.p2) : norm2<W>(v[i], m.p);
    }
    // each thread writes back exactly the positions it read (no cross-thread hazard),
    // then the tile leaves through one TMA bulk tensor store (see k_contig_tma)
#pragma unroll
    for (int q = 0; q < G; ++q) {
      if constexpr (VEC) {
#pragma unroll
        for (int h = 0; h < S; h += PER)
          sts128(sb + tswz<W>(blk[q] * B + h), pack16<W>(v + q * S + h));
      } else {
#pragma unroll
        for (int h = 0; h < S; ++h) sb[tswz<W>(blk[q] * B + h * D + c[q])] = v[q * S + h];
      }
    }
    (void)xb;
    (void)active;
  } else {
    // The exchange between the contiguous-run round and its neighbour is warp-local when that
    // round's blocks fit a warp (rounds.cuh): warps then skew freely instead of meeting twice per
    // tile.  The next tile's prefetch needs a CTA-wide barrier, so it rides on the forward's first
    // exchange and on the inverse's last one.
    constexpr int nr = INV ? r - 1 : r + 1;
    constexpr bool PREFETCH = INV ? (nr == 0) : (r == 0);
    constexpr bool WL = !PREFETCH && warp_local_exchange<LOGN, LE, r, nr>();
    (void)first_exchange;
    if constexpr (WL) __syncwarp();
    else __syncthreads();
    if (PREFETCH && threadIdx.x == 0 && next_tile < ntiles) {
      // every thread has finished the previous tile (the other buffer): once its TMA
      // store has read the buffer, prefetch the next tile into it
      bulk_wait_read0();
      mbar_expect_tx(next_bar, Sh::TILE_BYTES);
      const int row0 = (int)(next_tile * Sh::TILE_ROWS);
#pragma unroll
      for (int bx = 0; bx < Sh::BOXES; ++bx)
        tma_load_2d(next_buf + bx * Sh::BOX_BYTES, map, 0, row0 + bx * Sh::BOX_ROWS, next_bar);
    }
    // ---- exchange (same positions as this round's load)
#pragma unroll
    for (int q = 0; q < G; ++q) {
      if constexpr (VEC) {
#pragma unroll
        for (int h = 0; h < S; h += PER)
          sts128(sb + tswz<W>(blk[q] * B + h), pack16<W>(v + q * S + h));
      } else {
#pragma unroll
        for (int h = 0; h < S; ++h) sb[tswz<W>(blk[q] * B + h * D + c[q])] = v[q * S + h];
      }
    }
    if constexpr (WL) __syncwarp();
    else __syncthreads();
    tma_round<W, LOGN, LE, INV, PLO1, BF, nr>(v, xb, sb, t, active, tw, m, norm, false, map, next_tile, ntiles,
                                              next_buf, next_bar);
  }
}

template <class W, int LOGN, int LE, bool INV, bool PLO1, int BF>
__global__ void __launch_bounds__(TmaShape<W, LOGN, LE>::THREADS, TmaShape<W, LOGN, LE>::MINB)
    k_contig_tma(const __grid_constant__ CUtensorMap tmap, W* __restrict__ x, size_t batch,
                 const TwPair<W>* __restrict__ tw, W p, int norm) {
  using Sh = TmaShape<W, LOGN, LE>;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the swizzle period, by pointer arithmetic on the shared
  // array itself so that every access below stays an LDS/STS (not a generic LD/ST)
  const uint32_t s0 = smem_u32(smem_raw);
  unsigned char* base = smem_raw + (((s0 + 1023u) & ~1023u) - s0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + 2 * (size_t)Sh::TILE_BYTES);
  // buffer / mbarrier of slot i by arithmetic, not a per-thread array (a dynamically indexed
  // array would live on the stack)
  const uint32_t buf0 = smem_u32(base), bar0 = smem_u32(&bars[0]);
  auto buf_of = [&](int i) { return buf0 + (uint32_t)i * (uint32_t)Sh::TILE_BYTES; };
  auto bar_of = [&](int i) { return bar0 + (uint32_t)i * 8u; };
  const int slot = threadIdx.x / Sh::T, t = threadIdx.x % Sh::T;
  const Mod<W> m = make_mod<W>(p);
  const size_t ntiles = (batch + Sh::K - 1) / Sh::K;
  if (threadIdx.x == 0) {
    mbar_init(bar_of(0), 1);
    mbar_init(bar_of(1), 1);
    fence_mbar_init();
  }
  __syncthreads();
  size_t tile = blockIdx.x;
  if (threadIdx.x == 0 && tile < ntiles) {
    mbar_expect_tx(bar_of(0), Sh::TILE_BYTES);
#pragma unroll
    for (int bx = 0; bx < Sh::BOXES; ++bx)
      tma_load_2d(buf_of(0) + bx * Sh::BOX_BYTES, &tmap, 0, (int)(tile * Sh::TILE_ROWS) + bx * Sh::BOX_ROWS,
                  bar_of(0));
  }
  W v[Sh::E];
  for (uint32_t it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int cur = it & 1;
    mbar_wait(bar_of(cur), (it >> 1) & 1);
    const size_t b = tile * Sh::K + slot;
    const bool active = b < batch;
    constexpr int r0 = INV ? Sh::R - 1 : 0;
    W* sb = reinterpret_cast<W*>(base + (size_t)cur * Sh::TILE_BYTES) + slot * Sh::N;  // stays in shared space
    tma_round<W, LOGN, LE, INV, PLO1, BF, r0>(v, x + b * Sh::N, sb, t, active, tw, m, norm != 0, true, &tmap,
                                              tile + gridDim.x, ntiles, buf_of(cur ^ 1), bar_of(cur ^ 1));
    fence_proxy_async_smem();  // generic smem writes -> visible to the async (TMA) proxy
    __syncthreads();
    if (threadIdx.x == 0) {  // rows past the tensor end (partial last tile) are clipped by TMA
#pragma unroll
      for (int bx = 0; bx < Sh::BOXES; ++bx)
        tma_store_2d(&tmap, 0, (int)(tile * Sh::TILE_ROWS) + bx * Sh::BOX_ROWS, buf_of(cur) + bx * Sh::BOX_BYTES);
      bulk_commit();
    }
  }
  // the last bulk store must have read shared memory before the CTA exits (its global writes
  // complete with the grid, as CUTLASS's TMA epilogues rely on)
  if (threadIdx.x == 0) bulk_wait_read0();
}

// ----------------------------------------------------------------- host side
#ifndef NTT_TMA_LE64
#define NTT_TMA_LE64 4
#endif
#ifndef NTT_TMA_LE32
#define NTT_TMA_LE32 5
#endif
template <class W> struct TmaLE {
  static constexpr int value = sizeof(W) == 8 ? NTT_TMA_LE64 : NTT_TMA_LE32;
};

// Latency variant for batches that do not fill the GPU (config C1: one 2^10 transform): 8 words per
// thread, so a transform spreads over 4x more threads and each round's dependent chain is short
// (measured C1 10.2 -> 8.2 us after an L2 flush).
constexpr int kTmaLatencyLE = 3;
constexpr int kTmaLatencyMaxLog = 12;

template <class W, int LOGN, bool INV, bool PLO1, int BF, int LE = TmaLE<W>::value>
static cudaError_t run_tma(void* x, size_t batch, const void* tw, uint64_t p, bool norm, cudaStream_t s) {
  if constexpr (LE == TmaLE<W>::value && BF == 3 && LOGN <= kTmaLatencyMaxLog && kTmaLatencyLE < LE) {
    using Std = TmaShape<W, LOGN, LE>;
    if ((batch + Std::K - 1) / Std::K < (size_t)sm_count())
      return run_tma<W, LOGN, INV, PLO1, BF, kTmaLatencyLE>(x, batch, tw, p, norm, s);
  }
  using Sh = TmaShape<W, LOGN, LE>;
  const uint64_t rows = (uint64_t)batch * Sh::N / Sh::ROW_WORDS;
  // The tensor map depends only on (x, rows) for this instantiation: the last one is reused, so a
  // latency-bound caller (config C1, one transform per call) skips the host-side encode.
  struct MapCache { const void* x = nullptr; uint64_t rows = 0; int dev = -1; CUtensorMap map; };
  static thread_local MapCache mc;
  int dev = 0;
  cudaGetDevice(&dev);
  if (mc.x != x || mc.rows != rows || mc.dev != dev) {
    auto enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {(cuuint64_t)Sh::ROW_WORDS, (cuuint64_t)rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {(cuuint32_t)Sh::ROW_WORDS, (cuuint32_t)Sh::BOX_ROWS};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&mc.map, sizeof(W) == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, x,
                      dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
      mc.x = nullptr;
      return cudaErrorInvalidValue;
    }
    mc.x = x;
    mc.rows = rows;
    mc.dev = dev;
  }
  const CUtensorMap& map = mc.map;
  auto kern = k_contig_tma<W, LOGN, LE, INV, PLO1, BF>;
  static PerDevice occ_cache;
  const int occ = occ_cache.get([&] {
    int o = 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, Sh::THREADS, Sh::SMEM);
    return o > 0 ? o : 1;
  });
  const size_t ntiles = (batch + Sh::K - 1) / Sh::K;
  const size_t maxg = (size_t)occ * sm_count();
  const unsigned grid = (unsigned)(ntiles < maxg ? ntiles : maxg);
  if (!grid) return cudaSuccess;
  kern<<<grid, Sh::THREADS, Sh::SMEM, s>>>(map, reinterpret_cast<W*>(x), batch,
                                           reinterpret_cast<const TwPair<W>*>(tw), (W)p, norm ? 1 : 0);
  return cudaGetLastError();
}

template <class W, bool INV, int BF, int LO, int HI>
static cudaError_t tma_dispatch(int logn, void* x, size_t batch, const void* tw, uint64_t p, bool norm,
                                cudaStream_t s) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (logn == LO) {
      if constexpr (sizeof(W) == 8 && BF != 5) {
        if ((p & 0xffffffffull) == 1) return run_tma<W, LO, INV, true, BF>(x, batch, tw, p, norm, s);
      }
      return run_tma<W, LO, INV, false, BF>(x, batch, tw, p, norm, s);
    }
    return tma_dispatch<W, INV, BF, LO + 1, HI>(logn, x, batch, tw, p, norm, s);
  }
}

bool tma_supported(int wbytes, int logn) {
  return wbytes == 8 ? (logn >= kTmaMinLog && logn <= kTmaMaxLog64) : (logn >= kTmaMinLog && logn <= kTmaMaxLog32);
}

cudaError_t launch_contig_tma(int wbytes, int logn, bool inverse, bool normalize, void* x, size_t batch,
                              const void* tw, uint64_t p, cudaStream_t s, int bf) {
  if (inverse) {
    if (wbytes == 8) return tma_dispatch<uint64_t, true, 3, kTmaMinLog, kTmaMaxLog64>(logn, x, batch, tw, p, normalize, s);
    return tma_dispatch<uint32_t, true, 3, kTmaMinLog, kTmaMaxLog32>(logn, x, batch, tw, p, normalize, s);
  }
  if (wbytes == 8) {
    if (bf == 2) return tma_dispatch<uint64_t, false, 2, kTmaMinLog, kTmaMaxLog64>(logn, x, batch, tw, p, normalize, s);
    if (bf == 5) return tma_dispatch<uint64_t, false, 5, kTmaMinLog, kTmaMaxLog64>(logn, x, batch, tw, p, normalize, s);
    return tma_dispatch<uint64_t, false, 3, kTmaMinLog, kTmaMaxLog64>(logn, x, batch, tw, p, normalize, s);
  }
  if (bf == 2) return tma_dispatch<uint32_t, false, 2, kTmaMinLog, kTmaMaxLog32>(logn, x, batch, tw, p, normalize, s);
  if (bf == 5) return tma_dispatch<uint32_t, false, 5, kTmaMinLog, kTmaMaxLog32>(logn, x, batch, tw, p, normalize, s);
  return tma_dispatch<uint32_t, false, 3, kTmaMinLog, kTmaMaxLog32>(logn, x, batch, tw, p, normalize, s);
}

}  // namespace nttb
