// rounds.cuh -- the register "round" engine shared by every transform kernel.
//
// Algorithm 1 on an N = 2^LOGN point transform is cut into rounds of
// SR <= LE consecutive stages.  In a round a thread holds G = E/2^SR groups of
// 2^SR words; group (blk, c) holds positions blk*B + h*D + c (h < 2^SR) with
// B = N >> LEVEL and D = N >> (LEVEL + SR), so all butterflies of the round's
// stages pair words held by the same thread.
//
// Twiddles use the per-stage table layout: stage i (1-based) stores
// zeta_i^k = omega^{2^{i-1} k} for k < m_i = N >> i at offset
// N - (N >> (i-1)).  In every round the index k = hh*D + c is consecutive across
// lanes (c) or uniform (D = 1), so table reads are coalesced / broadcast.
#pragma once
#include <cstdint>

#include "modarith.cuh"

namespace nttb {

template <class W> __device__ __forceinline__ void ldtw(const TwPair<W>* tw, uint32_t e, W& w, W& wp);
template <> __device__ __forceinline__ void ldtw<uint64_t>(const TwPair<uint64_t>* tw, uint32_t e, uint64_t& w,
                                                           uint64_t& wp) {
  ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(tw) + e);
  w = t.x;
  wp = t.y;
}
template <> __device__ __forceinline__ void ldtw<uint32_t>(const TwPair<uint32_t>* tw, uint32_t e, uint32_t& w,
                                                           uint32_t& wp) {
  uint2 t = __ldg(reinterpret_cast<const uint2*>(tw) + e);
  w = t.x;
  wp = t.y;
}

// Twiddle load for forward butterfly BF: (W, W') pairs, or for Algorithm 5 the single word
// beta W mod p ("only a single value W' must be stored") -- its tables hold one word per entry.
template <class W, int BF>
__device__ __forceinline__ void ldtw_bf(const TwPair<W>* tw, uint32_t e, W& w, W& wp) {
  if constexpr (BF == 5) {
    w = __ldg(reinterpret_cast<const W*>(tw) + e);
    wp = 0;
  } else {
    ldtw<W>(tw, e, w, wp);
  }
}

// Offset of stage i's table inside the per-stage layout of an N-point transform: stage i holds
// zeta_i^k for k <= m_i = N >> i (m_i + 1 entries; the last one is zeta_i^{m_i} = omega^{N/2} = -1).
__host__ __device__ constexpr int stage_off(int logn, int i) {
  return (1 << logn) - ((1 << logn) >> (i - 1)) + (i - 1);
}

// The inverse reads the same table (no second table).  zeta_i^{-k} = -zeta_i^{m_i - k}
// (zeta_i^{m_i} = omega^{N/2} = -1), so entry m_i - k holds (W~, W~') with W~ = -zeta_i^{-k} mod p,
// and the inverse butterfly bfly_alg4n takes the negated twiddle.  Index of that entry:
__host__ __device__ constexpr int inv_index(int logn, int i, int k) {
  return stage_off(logn, i) + ((1 << logn) >> i) - k;
}

// Round structure: R rounds of balanced stage counts sr(r) <= LE.
template <int LOGN, int LE> struct Rounds {
  static constexpr int R = (LOGN + LE - 1) / LE;
  __host__ __device__ static constexpr int sr(int r) { return LOGN / R + (r < LOGN % R ? 1 : 0); }
  __host__ __device__ static constexpr int level(int r) {
    int s = 0;
    for (int i = 0; i < r; ++i) s += sr(i);
    return s;
  }
};

// True when the exchange between rounds ra and rb of an N = 2^LOGN transform with T = N/2^LE
// threads stays inside each warp: one round holds contiguous runs (D = 1), the other one group
// (G = 1) of the same run length S per thread with D <= 32 dividing 32, so warp w holds the
// elements [32 S w, 32 S (w+1)) in both.  Such an exchange needs __syncwarp, not __syncthreads.
template <int LOGN, int LE, int ra, int rb> __host__ __device__ constexpr bool warp_local_exchange() {
  using RC = Rounds<LOGN, LE>;
  constexpr int N = 1 << LOGN, T = N >> LE;
  constexpr int Sa = 1 << RC::sr(ra), Sb = 1 << RC::sr(rb);
  constexpr int Da = N >> (RC::level(ra) + RC::sr(ra)), Db = N >> (RC::level(rb) + RC::sr(rb));
  constexpr bool G1 = (Sa == (1 << LE)) && (Sb == (1 << LE));
  constexpr bool runs = (Da == 1 && Db <= 32 && 32 % Db == 0) || (Db == 1 && Da <= 32 && 32 % Da == 0);
  return T % 32 == 0 && G1 && runs;
}

// Forward round: stages LEVEL+1 .. LEVEL+SR with the Algorithm 3 butterfly.
// Butterflies known at compile time to have W = 1 (the whole last stage, m = 1, and
// every k = 0 butterfly of a round with D = 1) take the multiply-free path.
// BF selects the butterfly: 3 = Algorithm 3 (the product path), 2 = Algorithm 2 and
// 5 = Algorithm 5 (ablations F1/F2 of SURVEY.md §8(f); Alg. 5 reads W' = beta W mod p
// from a one-word-per-entry table, ldtw_bf).
// LAZY_LAST: the transform's last stage (m = 1, W = 1) leaves X + Y and X - Y + 2p unreduced, in [0,4p):
// only for callers that multiply every output by a twiddle next (the four-step column pass), since a
// Shoup product takes any T < beta and returns [0,2p) -- the two corrections of P:226's W = 1
// butterfly are then redundant.
// NC: the thread holds NC copies of its G groups (v[k G S + q S + h], k < NC) at the same positions
// of NC different transforms (the column pass's adjacent columns), so each twiddle load serves NC
// butterflies.
template <class W, int LOGN, int SR, int LEVEL, int G, bool PLO1, int BF = 3, bool LAZY_LAST = false, int NC = 1>
__device__ __forceinline__ void dif_round(W* v, const int* c, const TwPair<W>* __restrict__ tw, const Mod<W>& m) {
  NTT_AUDIT_STRESS();  // audit build only: per-warp random delay (race stress)
  constexpr int S = 1 << SR;
  constexpr int D = (1 << LOGN) >> (LEVEL + SR);
#pragma unroll
  for (int j = 0; j < SR; ++j) {
    const int half = S >> (j + 1);
    const bool w1 = (LEVEL + j + 1 == LOGN);
    const int off = stage_off(LOGN, LEVEL + j + 1);
#pragma unroll
    for (int q = 0; q < G; ++q) {
#pragma unroll
      for (int hh = 0; hh < half; ++hh) {
        // k = hh*D + c; when D == 1 (c == 0) the hh == 0 butterflies have k = 0, i.e. W = 1
        const bool unit = w1 || (D == 1 && hh == 0);
        W w = 1, wp = 0;
        if (!unit) ldtw_bf<W, BF>(tw, (uint32_t)(off + hh * D + c[q]), w, wp);
#pragma unroll
        for (int k = 0; k < NC; ++k)
#pragma unroll
        for (int b = 0; b < (1 << j); ++b) {
          const int h = b * 2 * half + hh;
          W* u = v + k * G * S + q * S;
          if (LAZY_LAST && BF != 2 && w1) bfly_alg3_w1_lazy<W>(u[h], u[h + half], m.p2);
          else if (unit) bfly_fwd_w1<W, BF>(u[h], u[h + half], m);
          else bfly_fwd<W, PLO1, BF>(u[h], u[h + half], w, wp, m);
        }
      }
    }
  }
}

// Inverse round: the same stages run backwards, Algorithm 4 with the twiddles
// zeta_i^{-k}, read as their negations from the forward table (inv_index, bfly_alg4n).
template <class W, int LOGN, int SR, int LEVEL, int G, bool PLO1, int NC = 1>
__device__ __forceinline__ void dit_round(W* v, const int* c, const TwPair<W>* __restrict__ twi, const Mod<W>& m) {
  NTT_AUDIT_STRESS();
  constexpr int S = 1 << SR;
  constexpr int D = (1 << LOGN) >> (LEVEL + SR);
  // one base pointer per group, twi - c[q]: every entry m - k = (m - hh D) - c[q] of the round is then a
  // compile-time offset from it (a per-load runtime index would cost an IMAD.WIDE address each)
  const TwPair<W>* tq[G];
#pragma unroll
  for (int q = 0; q < G; ++q) tq[q] = twi - c[q];
#pragma unroll
  for (int j = SR - 1; j >= 0; --j) {
    const int half = S >> (j + 1);
    const bool w1 = (LEVEL + j + 1 == LOGN);
    const int off = stage_off(LOGN, LEVEL + j + 1);
#pragma unroll
    for (int q = 0; q < G; ++q) {
#pragma unroll
      for (int hh = 0; hh < half; ++hh) {
        const bool unit = w1 || (D == 1 && hh == 0);  // k = 0: W = 1
        W w = 1, wp = 0;
        // negated twiddle -zeta^{-k} = zeta^{m - k} from the forward table (inv_index)
        if (!unit) ldtw<W>(tq[q], (uint32_t)(off + ((1 << LOGN) >> (LEVEL + j + 1)) - hh * D), w, wp);
#pragma unroll
        for (int k = 0; k < NC; ++k)
#pragma unroll
        for (int b = 0; b < (1 << j); ++b) {
          const int h = b * 2 * half + hh;
          W* u = v + k * G * S + q * S;
          if (unit) bfly_alg4_w1<W>(u[h], u[h + half], m.p2);
          else bfly_alg4n<W, PLO1>(u[h], u[h + half], w, wp, m);
        }
      }
    }
  }
}

// 16-byte vector helpers (two u64 or four u32 words).
template <class W> __device__ __forceinline__ void unpack16(const uint4& u, W* v) {
  if constexpr (sizeof(W) == 8) {
    v[0] = ((uint64_t)u.y << 32) | u.x;
    v[1] = ((uint64_t)u.w << 32) | u.z;
  } else {
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  }
}
template <class W> __device__ __forceinline__ uint4 pack16(const W* v) {
  uint4 u;
  if constexpr (sizeof(W) == 8) {
    u.x = (uint32_t)v[0]; u.y = (uint32_t)(v[0] >> 32);
    u.z = (uint32_t)v[1]; u.w = (uint32_t)(v[1] >> 32);
  } else {
    u.x = v[0]; u.y = v[1]; u.z = v[2]; u.w = v[3];
  }
  return u;
}

// Contiguous run of S words: widest aligned vector accesses (global or shared).
template <class W, int S> __device__ __forceinline__ void load_run(const W* src, W* v) {
  if constexpr (S * sizeof(W) >= 16) {
    constexpr int PER = 16 / sizeof(W);
#pragma unroll
    for (int i = 0; i < S / PER; ++i) unpack16<W>(*reinterpret_cast<const uint4*>(src + i * PER), v + i * PER);
  } else {
#pragma unroll
    for (int i = 0; i < S; ++i) v[i] = src[i];
  }
}
template <class W, int S> __device__ __forceinline__ void store_run(W* dst, const W* v) {
  if constexpr (S * sizeof(W) >= 16) {
    constexpr int PER = 16 / sizeof(W);
#pragma unroll
    for (int i = 0; i < S / PER; ++i) *reinterpret_cast<uint4*>(dst + i * PER) = pack16<W>(v + i * PER);
  } else {
#pragma unroll
    for (int i = 0; i < S; ++i) dst[i] = v[i];
  }
}

}  // namespace nttb
