// fourstep.cuh -- the four-step twiddle of a column pass and the
// global-column mapping of a distributed shard, shared by k_cols and k_cols_tma.
#pragma once
#include <cstdint>

#include "internal.h"
#include "modarith.cuh"
#include "rounds.cuh"

namespace nttb {

// omega_L^e by the direct table (H == 0) or the factored tables
// omega^{(e >> H) << H} * omega^{e & (2^H - 1)} (two Shoup multiplies).
template <class W, bool PLO1>
__device__ __forceinline__ W fourstep_twiddle(W val, uint32_t e, const ColsParams& prm, const TwPair<W>* __restrict__ fa,
                                              const TwPair<W>* __restrict__ fb, const Mod<W>& m) {
  W w, wp;
  if (prm.H == 0) {
    ldtw<W>(fa, e, w, wp);
    return shoup_mul<W, PLO1>(val, w, wp, m);
  }
  ldtw<W>(fb, e & ((1u << prm.H) - 1), w, wp);
  val = shoup_mul<W, PLO1>(val, w, wp, m);
  ldtw<W>(fa, e >> prm.H, w, wp);
  return shoup_mul<W, PLO1>(val, w, wp, m);
}

// The same with the table form fixed at compile time (FACT: factored, two Shoup multiplies), so
// a kernel's per-element twiddle code has no branch and its loads can be scheduled early.
template <class W, bool PLO1, bool FACT>
__device__ __forceinline__ W fourstep_twiddle_ct(W val, uint32_t e, uint32_t H, const TwPair<W>* __restrict__ fa,
                                                 const TwPair<W>* __restrict__ fb, const Mod<W>& m) {
  W w, wp;
  if constexpr (!FACT) {
    ldtw<W>(fa, e, w, wp);
    return shoup_mul<W, PLO1>(val, w, wp, m);
  } else {
    W w2, wp2;
    ldtw<W>(fb, e & ((1u << H) - 1), w, wp);
    ldtw<W>(fa, e >> H, w2, wp2);
    val = shoup_mul<W, PLO1>(val, w, wp, m);
    return shoup_mul<W, PLO1>(val, w2, wp2, m);
  }
}

// The same for the ablation butterflies (BF 2: Shoup pairs, canonical result; BF 5: one-word
// Montgomery tables, Algorithm 5's multiply), factored (FACT) or direct tables.
template <class W, bool PLO1, bool FACT, int BF>
__device__ __forceinline__ W fourstep_twiddle_bf(W val, uint32_t e, uint32_t H, const TwPair<W>* __restrict__ fa,
                                                 const TwPair<W>* __restrict__ fb, const Mod<W>& m) {
  if constexpr (BF == 3) {
    return fourstep_twiddle_ct<W, PLO1, FACT>(val, e, H, fa, fb, m);
  } else if constexpr (!FACT) {
    W w, wp;
    ldtw_bf<W, BF>(fa, e, w, wp);
    return twiddle_mul<W, PLO1, BF>(val, w, wp, m);
  } else {
    W w, wp, w2, wp2;
    ldtw_bf<W, BF>(fb, e & ((1u << H) - 1), w, wp);
    ldtw_bf<W, BF>(fa, e >> H, w2, wp2);
    val = twiddle_mul<W, PLO1, BF>(val, w, wp, m);
    return twiddle_mul<W, PLO1, BF>(val, w2, wp2, m);
  }
}

#ifndef NTT_COLS_POW2  // tile coordinates by shifts when the block count is a power of two
#define NTT_COLS_POW2 1
#endif
// Block index and column group of a column-pass tile (ColsParams::bmajor: DESIGN.md §5).
// BM: the kernel supports the block-major order (only the twiddle-matrix instantiations do).
template <bool BM = true>
__device__ __forceinline__ void cols_tile_coords(uint64_t tile, const ColsParams& prm, uint64_t& bq, uint32_t& cg) {
  if (!BM || !prm.bmajor) {
    bq = tile >> prm.log_colgroups;
    cg = (uint32_t)(tile & ((1ull << prm.log_colgroups) - 1));
  } else {
    const uint64_t nblk = prm.n_tiles >> prm.log_colgroups, rest = tile >> prm.log_cgi;
    uint64_t qt;
    if (NTT_COLS_POW2 && (nblk & (nblk - 1)) == 0) {  // a power-of-two count of blocks (C4, C5): no division
      bq = rest & (nblk - 1);
      qt = rest >> (__ffsll((long long)nblk) - 1);
    } else {
      bq = rest % nblk;
      qt = rest / nblk;
    }
    cg = ((uint32_t)qt << prm.log_cgi) | (uint32_t)(tile & ((1u << prm.log_cgi) - 1));
  }
}

// Global column of local column `cloc` (ColsParams.shard: config C5 column shard).
__device__ __forceinline__ uint32_t cols_global_column(uint32_t cloc, const ColsParams& prm) {
  if (!prm.shard) return cloc;
  const uint32_t rb = cloc >> prm.log_local_w, cl = cloc & ((1u << prm.log_local_w) - 1);
  return (rb << prm.log_n2) | (prm.col0 + cl);
}

// peer[h] without dynamic indexing of a kernel-parameter array (which would copy the whole
// parameter struct to the stack): an unrolled select over the <= 8 entries.
__device__ __forceinline__ uint64_t select_peer(const uint64_t (&peer)[8], uint32_t h) {
  uint64_t d = peer[0];
#pragma unroll
  for (uint32_t i = 1; i < 8; ++i) d = (h == i) ? peer[i] : d;
  return d;
}

}  // namespace nttb
