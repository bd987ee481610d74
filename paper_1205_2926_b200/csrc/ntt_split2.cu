// ntt_split2.cu -- transforms of length L = K*Q on a cluster of K CTAs (K = 2 or 4),
// Q = 2^LOGQ words per CTA, without an HBM round trip between stages.
//
// Forward (Algorithm 1): after the first s = log2 K stages, the block of
// positions [rQ, (r+1)Q) is an independent Q-point transform with root omega^K
// (stages s+1..ell), whose per-stage twiddle table is the full table's suffix from
// offset L - Q.  CTA r evaluates only its path through stages 1..s: for each j < Q it
// reads x_{j + tQ} (t < K) and, at stage i, keeps the sum (Algorithm 3 lines 1-2) or the
// twiddled difference (lines 3-5, W = zeta_i^{j + tQ}) as bit (s - i) of r says.  (Stage 1
// is evaluated by two CTAs when K = 4: +1/ell work, no data exchange.)  K = 2 brings both
// blocks in by TMA, in chunks through shared memory, the first ones while the previous
// transform computes (SplitFwd); K = 4 loads them from global memory.  A cluster barrier
// orders every CTA's reads before the in-place stores (K = 2: arrive after stage 1, wait
// before the last round's store); output block r = Alg. 1's positions [rQ, (r+1)Q).
//
// Inverse (Algorithm 1 run backwards): stages ell..s+1 are K independent
// Q-point inverses (one per CTA); stages s..1 (Algorithm 4, W = zeta_i^{-k}) act on
// the K values at positions j + tQ through distributed shared memory (K = 2: each CTA pushes the
// half it does not finish into the other's shared memory; K = 4: reads from the K CTAs); CTA r
// finishes j in [rQ/K, (r+1)Q/K).  With PW the
// pointwise product c = a b L^{-1} is formed while loading, so a cyclic
// convolution needs no separate pointwise pass.
//
// Forward with PW (cyclic convolution): the last round multiplies b-hat (registers) by this
// CTA's block of a-hat, staged by TMA into the Q-word buffer while the round computes, and the
// product c-hat = a-hat b-hat L^{-1} leaves over a-hat; b is only read, so no cluster barrier.
//
// Staging (inverse): each CTA's own block of the next transform (x, or a when PW) is
// brought into shared memory by TMA (2-D tensor map of 128-byte rows, SWIZZLE_128B) once
// the cluster's DSMEM epilogue no longer reads the buffer; the first round then reads it
// from shared memory and only b (PW) comes from global memory.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"
#include "modarith.cuh"
#include "rounds.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;


namespace nttb {

template <class W> __device__ __forceinline__ int sswz(int i) {  // element XOR swizzle (128-byte rows)
  constexpr int S = sizeof(W) == 8 ? 4 : 5;
  return i ^ ((i >> S) & ((1 << S) - 1));
}

// Forward's last round with G > 1 groups of contiguous runs (u64 2^15: rounds 5,5,4): groups assigned
// g = t G + q instead of g = t + T q give each thread E consecutive words, so a warp holds the same
// 32 E words as in the previous round (G = 1, D <= 32) and their exchange is warp-local.  Its layout
// then swaps 16-byte chunks by (row / 2) mod 8 (xswz) -- conflict-free for both sides, where the
// element swizzle of the other exchanges is not.
#ifndef NTT_SPLIT_REMAP
#define NTT_SPLIT_REMAP 1
#endif
template <int LOGQ, int LE, int r> __host__ __device__ constexpr bool split_remap_last() {
  using RC = Rounds<LOGQ, LE>;
  constexpr int Q = 1 << LOGQ, E = 1 << LE, T = Q >> LE;
  if constexpr (!NTT_SPLIT_REMAP || r != RC::R - 1 || r == 0) {
    return false;
  } else {
    constexpr int S = 1 << RC::sr(r), D = Q >> (RC::level(r) + RC::sr(r));
    constexpr int Sp = 1 << RC::sr(r - 1), Dp = Q >> (RC::level(r - 1) + RC::sr(r - 1));
    return S < E && D == 1 && Sp == E && Dp <= 32 && 32 % Dp == 0 && T % 32 == 0;
  }
}
// An exchange between rounds ra and rb whose groups both have D >= one 128-byte row of words (32 u32 /
// 16 u64) is conflict-free in the plain layout: every (half-)warp access covers one whole row on both
// sides.  It then skips the element swizzle, whose per-access XOR (D-strided reads: c ^ h) costs an
// instruction per word (NTT_SPLIT_PLAINX = 0 keeps the swizzle everywhere).
#ifndef NTT_SPLIT_PLAINX
#define NTT_SPLIT_PLAINX 1
#endif
template <int LOGQ, int LE, int WB, int ra, int rb> __host__ __device__ constexpr bool plain_exchange() {
  using RC = Rounds<LOGQ, LE>;
  constexpr int Q = 1 << LOGQ, T = Q >> LE, ROWW = 128 / WB;
  constexpr int Da = Q >> (RC::level(ra) + RC::sr(ra)), Db = Q >> (RC::level(rb) + RC::sr(rb));
  // (u64 only: measured u64 2^15 inverse -6.3 %, forward -0.1 %; for u32 the plain exchange made C3 +2.8 %)
  return NTT_SPLIT_PLAINX && WB == 8 && T % 32 == 0 && Da >= ROWW && Db >= ROWW;
}
// NTT_SPLIT_REMAP2 (default): lane l of warp w takes the remapped round's groups 32 G w + 32 q + l (one
// 128-byte row each for u64) instead of G consecutive ones, still inside the warp's 32 E words; the
// exchange then uses the TMA swizzle itself (chunk ^= row mod 8), so the round's 16-byte reads and the
// epilogue's 16-byte stores into the TMA-swizzled buffer cover 8 chunk positions per 8 lanes: no 2-way
// conflict on the epilogue's STS.128 (with G consecutive rows per thread, row mod 8 took 4 values).
#ifndef NTT_SPLIT_REMAP2
#define NTT_SPLIT_REMAP2 1
#endif
// u32 forward (NTT_SPLIT_RUNV): the exchange into the last round, whose groups are one 32-word run per
// thread (G = 1, D = 1) written by a round with D >= 32, uses the TMA chunk swizzle (16-byte chunk ^=
// row mod 8) instead of the element swizzle, so the last round reads its run with 8 16-byte loads
// instead of 32 4-byte ones (conflict-free on both sides: a warp writes one whole row per store, and the
// 8 lanes of a quarter-warp read 8 distinct chunk positions).
#ifndef NTT_SPLIT_RUNV
#define NTT_SPLIT_RUNV 1
#endif
template <int LOGQ, int LE, int WB, int r> __host__ __device__ constexpr bool runv_round() {
  using RC = Rounds<LOGQ, LE>;
  constexpr int Q = 1 << LOGQ, E = 1 << LE, T = Q >> LE;
  if constexpr (!NTT_SPLIT_RUNV || WB != 4 || r != RC::R - 1 || r == 0) {
    return false;
  } else {
    constexpr int S = 1 << RC::sr(r), D = Q >> (RC::level(r) + RC::sr(r));
    constexpr int Dp = Q >> (RC::level(r - 1) + RC::sr(r - 1));
    return S == E && D == 1 && Dp >= 32 && T % 32 == 0;
  }
}
template <class W> __device__ __forceinline__ int xswz(int i) {  // 16-byte chunk ^= (row / 2) mod 8
  constexpr int CS = sizeof(W) == 8 ? 1 : 2;  // log2 words per chunk
  constexpr int RS = sizeof(W) == 8 ? 4 : 5;  // log2 words per 128-byte row
  if constexpr (NTT_SPLIT_REMAP2) return i ^ (((i >> RS) & 7) << CS);
  else return i ^ ((((i >> RS) >> 1) & 7) << CS);
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

// Cluster barrier for write-after-read hazards only: every value the caller loaded before it
// has already been consumed (in-order issue), so a relaxed arrive suffices and the
// MEMBAR.ALL.GPU that cluster.sync() emits for its release is skipped.
__device__ __forceinline__ void cluster_sync_war() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

struct PwArgs {
  const void* a;
  const void* b;
  uint64_t J, K, Kp;  // REDC constant and the Shoup constant restoring scale (beta L^{-1} mod p)
  const void* tw1s;   // forward with PW: stage-1 table scaled by K (zeta_1^j K, its W')
};

// Shared-memory staging of a transform (inverse only): this CTA's block of Q words in NCH chunks
// of one TMA box (256 rows of 128 bytes).  K = 2: the first NX = 3 chunks go to spare slots after
// the Q-word buffer and are loaded for the next transform as soon as this one's first round has
// read them; the rest land in the buffer once the DSMEM epilogue no longer reads it.  One mbarrier
// per chunk after the slots.  (K = 4 runs two CTAs per SM: no spare slots, NX = 0.)  Measured
// (u32 2^16 / u64 2^15 inverse): -3% / -5% against staging the whole block after the epilogue.
template <class W, int LOGQ, int LE, int K, bool INV, bool PW> struct SplitStaging {
  static constexpr bool ON = INV;
  static constexpr int Q = 1 << LOGQ;
  static constexpr uint32_t BYTES = (uint32_t)(Q * sizeof(W));
  static constexpr int ROWS = (int)(BYTES / 128), BOX = ROWS < 256 ? ROWS : 256, NCH = ROWS / BOX;
  static constexpr uint32_t CH = BOX * 128;
  static constexpr int CW = (int)(CH / sizeof(W));  // words per chunk
  // (PW keeps the L1 large: its b operand streams through it with LDG.128, and spare slots that
  // shrink the L1 carveout made the fused convolution slower: 3 slots +20%, 2 +6%, 1 +2%)
  static constexpr int NX = (K == 2 && NCH == 4 && !PW) ? 3 : 0;
  static constexpr uint32_t X_OFF = BYTES, BAR_OFF = X_OFF + NX * CH;
  static constexpr size_t SMEM = BAR_OFF + 8 * NCH + 8;  // + the K = 2 push mbarrier (st.async epilogue)
  __device__ static constexpr uint32_t slot(int k) { return k < NX ? X_OFF + k * CH : k * CH; }
  __device__ static uint32_t bar(uint32_t sbase, int k) { return sbase + BAR_OFF + 8 * k; }
  __device__ static uint32_t push_bar(uint32_t sbase) { return sbase + BAR_OFF + 8 * NCH; }
  // chunks [k0, k1) of this CTA's block of transform b
  __device__ static void issue(const CUtensorMap* map, size_t b, int rank, int k0, int k1, uint32_t sbase) {
    const int row0 = (int)((b * K + (size_t)rank) * (size_t)ROWS);
    for (int k = k0; k < k1; ++k) {
      mbar_expect_tx(bar(sbase, k), CH);
      tma_load_2d(sbase + slot(k), map, 0, row0 + k * BOX, bar(sbase, k));
    }
  }
};

// Staging state of the current transform: the 2-D map (128-byte rows) over x (forward,
// plain inverse) or a (PW), the mbarrier parity to wait for, and the cluster's next
// transform (next_b >= batch: none).  The tile sits at the start of shared memory and its
// mbarrier right after it (k_splitk).
struct SplitStage {
  const CUtensorMap* map;
  uint32_t phase;
  size_t b, next_b, batch;
  const CUtensorMap* map_a;  // forward with PW: 128-byte rows of a (a-hat in, c-hat out)
};

#ifndef NTT_SPLIT_DRAIN  // plain K = 2 forward: buffer chunks issued per drained store group, after the
#define NTT_SPLIT_DRAIN 1  // stage-1 X barrier (0: all at the transform's start after the whole store read)
#endif
#ifndef NTT_SPLIT_STASYNC  // K = 2 inverse: the cross-CTA push by st.async + mbarrier (0: remote stores +
#define NTT_SPLIT_STASYNC 1  // cluster.sync, round 2's form)
#endif
// Timing-only experiment hooks (results wrong; DESIGN.md §7 removal bounds): NTT_XP_NOEXCH drops the
// exchanges' shared-memory traffic, NTT_XP_NOWAIT the stage-1 data waits of the K = 2 forward.
#ifndef NTT_SPLIT_NX  // spare staging slots of the K = 2 forward (A/B on one box, round 2: 2 slots
#define NTT_SPLIT_NX 2    // beat 3 -- C4 row pass 10.68 -> 10.61 ms, C3 2.537 -> 2.523 ms -- the smaller
#endif                    // shared-memory footprint leaves more L1 to the twiddle loads)

// Forward staging (K = 2): the first round's inputs x_{hD + t} and x_{Q + hD + t} (h < 32) come in
// NCH chunks of HC h-rows of both blocks (2 x HC x D words; one TMA box of 128-byte rows per
// block).  NX chunk slots sit after the Q-word buffer and are filled with the next transform's
// first chunks while this one computes; the next 4 chunks land in the Q-word buffer itself once
// the previous transform's bulk store has read it, the rest in the X slots once consumed.
template <class W, int LOGQ, int LE> struct SplitFwd {
  static constexpr int Q = 1 << LOGQ, S = 1 << Rounds<LOGQ, LE>::sr(0), D = Q / S;
  static constexpr int NCH = 8, HC = S / NCH, NX = NTT_SPLIT_NX, NB = 4;
  static constexpr uint32_t HALF = (uint32_t)(HC * D * sizeof(W)), CH = 2 * HALF;
  static constexpr int BOXR = (int)(HALF / 128);  // rows of one block's part of a chunk
  static constexpr uint32_t X_OFF = (uint32_t)(Q * sizeof(W)), BAR_OFF = X_OFF + NX * CH;
  static constexpr size_t SMEM = BAR_OFF + NCH * 8;
  static_assert(NB * CH == (uint32_t)(Q * sizeof(W)), "4 chunks fill the Q-word buffer");
  static_assert(NX + NB < NCH && NCH - NX - NB <= NX, "late chunks reuse X slots");
  static_assert(HALF % 1024 == 0 && BOXR <= 256, "swizzle period / TMA box");
  __device__ static constexpr uint32_t slot(int k) {
    return k < NX ? X_OFF + k * CH : (k < NX + NB ? (k - NX) * CH : X_OFF + (k - NX - NB) * CH);
  }
  // chunk k of transform b: two boxes (block 0 rows, block 1 rows) into its slot
  __device__ static void issue(const CUtensorMap* map, size_t b, int k, uint32_t sbase) {
    const uint32_t bar = sbase + BAR_OFF + 8 * k, dst = sbase + slot(k);
    constexpr int ROWS_BLK = (int)(Q * sizeof(W) / 128);
    mbar_expect_tx(bar, CH);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
      tma_load_2d(dst + hf * HALF, map, 0, (int)((b * 2 + hf) * (size_t)ROWS_BLK) + k * BOXR, bar);
  }
};

// Chunk NX + i of transform b into buffer slot i once the previous transform's bulk store group i has
// read it (NTT_SPLIT_DRAIN; the store commits one group per chunk slot).
template <class W, int LOGQ, int LE, int I = 0>
__device__ __forceinline__ void split_issue_drained(const CUtensorMap* map, size_t b, uint32_t sbase) {
  using F = SplitFwd<W, LOGQ, LE>;
  if constexpr (I < F::NB) {
    bulk_wait_read<F::NB - 1 - I>();
    F::issue(map, b, F::NX + I, sbase);
    split_issue_drained<W, LOGQ, LE, I + 1>(map, b, sbase);
  }
}

// Stage 1 of the forward from the staged chunks: CTA 0 keeps sums, CTA 1 twiddled differences.
// SCALE (forward with the pointwise product): stage 1 also multiplies by K = beta L^{-1} -- CTA 0's
// sums by one Shoup product (work CTA 1 already spends on its twiddles), CTA 1's differences through
// the pre-scaled table -- so the final product needs one REDC instead of REDC + Shoup.
template <class W, int LOGQ, int LE, int LOGL, bool PLO1, bool UPPER, bool SCALE = false, int BF = 3>
__device__ __forceinline__ void split_fwd_stage1(W* v, const W* sm, int t, const TwPair<W>* __restrict__ tw_full,
                                                 const Mod<W>& m, const SplitStage& st, const PwArgs& pw) {
  using F = SplitFwd<W, LOGQ, LE>;
  const unsigned char* base = reinterpret_cast<const unsigned char*>(sm);
  const uint32_t sbase = smem_u32(sm);
  const int tsw = tswz<W>(t);  // (h - h0) D is a multiple of the swizzle period
  const int off = stage_off(LOGL, 1);
  NTT_AUDIT_STRESS();
#pragma unroll
  for (int k = 0; k < F::NCH; ++k) {
#ifndef NTT_XP_NOWAIT
    mbar_wait(sbase + F::BAR_OFF + 8 * k, st.phase);
#endif
    const W* lo = reinterpret_cast<const W*>(base + F::slot(k));
    const W* hi = reinterpret_cast<const W*>(base + F::slot(k) + F::HALF);
#pragma unroll
    for (int hh = 0; hh < F::HC; ++hh) {
      const int h = k * F::HC + hh, j = h * F::D + t;
      const W a = lo[hh * F::D + tsw], b = hi[hh * F::D + tsw];
      NTT_AUDIT(a, BF == 2 ? m.p : m.p2);  // Alg. 3 / 5 input range (Alg. 2: canonical)
      NTT_AUDIT(b, BF == 2 ? m.p : m.p2);
      if constexpr (!UPPER && SCALE) {
        v[h] = shoup_mul<W, PLO1>(a + b, (W)pw.K, (W)pw.Kp, m);  // a + b < 4p < beta: a Shoup input
      } else if constexpr (!UPPER) {
        v[h] = csub<W>(a + b, BF == 2 ? m.p : m.p2);  // Alg. 3/5 lines 1-2 (Alg. 2: canonical)
      } else {
        W w, wp;
        if constexpr (SCALE) ldtw<W>(reinterpret_cast<const TwPair<W>*>(pw.tw1s), (uint32_t)j, w, wp);
        else ldtw_bf<W, BF>(tw_full, (uint32_t)(off + j), w, wp);
        if constexpr (BF == 2) v[h] = twiddle_mul<W, PLO1, 2>(a < b ? a - b + m.p : a - b, w, wp, m);  // Alg. 2
        else if constexpr (BF == 5) v[h] = mont_mul<W>(a - b + m.p2, w, m);                           // Alg. 5
        else {
          W T = a - b + m.p2;
          if (NTT_AUDIT_MUTATED()) T = a - b;
          NTT_AUDIT(T, 2 * m.p2);  // Theorem 2: T in [0,4p)
          v[h] = shoup_mul<W, PLO1>(T, w, wp, m);
        }
      }
      NTT_AUDIT(v[h], BF == 2 ? m.p : m.p2);
    }
    if (k == F::NX - 1) {  // X slots consumed: the late chunks reuse them
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        if constexpr (NTT_SPLIT_DRAIN) {
          // the buffer chunks NX..NX+NB-1, each as soon as the previous transform's store (one bulk
          // group per chunk slot, committed in slot order) has read that slot; the other warps go on
          // to wait for chunk NX's data instead of for this thread
          split_issue_drained<W, LOGQ, LE>(st.map, st.b, sbase);
        }
#pragma unroll
        for (int kk = F::NX + F::NB; kk < F::NCH; ++kk) F::issue(st.map, st.b, kk, sbase);
      }
    }
  }
  // (the X slots take the next transform's first chunks at the first round's exchange barrier)
}


template <class W, int LOGQ, int LE, int K, bool INV, bool PLO1, bool PW, int BF, int r>
__device__ __forceinline__ void split_round(W* v, W* __restrict__ xb, W* sm, int t, int rank,
                                            const TwPair<W>* __restrict__ tw_full, const Mod<W>& m,
                                            const PwArgs& pw, size_t boff, cg::cluster_group& cluster,
                                            const SplitStage& st) {
  NTT_AUDIT_STRESS();  // audit build only: per-warp random delay before the round reads its inputs
  using Sh = SplitShape<LOGQ, LE, K, (int)sizeof(W)>;
  using RC = typename Sh::RC;
  constexpr int Q = Sh::Q, SS = Sh::S_SPLIT, LOGL = Sh::LOGL;
  constexpr int SR = RC::sr(r), LEVEL = RC::level(r);
  constexpr int S = 1 << SR, G = Sh::E >> SR;
  constexpr int D = Q >> (LEVEL + SR), B = Q >> LEVEL;
  // stages s+1..ell of the full per-stage table (Alg. 5 tables: one word per entry)
  const TwPair<W>* tw_sub =
      BF == 5 ? reinterpret_cast<const TwPair<W>*>(reinterpret_cast<const W*>(tw_full) + stage_off(LOGL, SS + 1))
              : tw_full + stage_off(LOGL, SS + 1);
  constexpr bool REMAP = !INV && split_remap_last<LOGQ, LE, r>();  // this round: remapped groups
  constexpr bool RUNV = !INV && runv_round<LOGQ, LE, (int)sizeof(W), r>();  // this round: 16-byte run reads
  int c[G], blk[G];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = REMAP ? (NTT_SPLIT_REMAP2 ? (t >> 5) * (32 * G) + 32 * q + (t & 31) : t * G + q) : t + Sh::T * q;
    blk[q] = g / D;
    c[q] = g % D;
  }
  constexpr bool first = INV ? (r == Sh::R - 1) : (r == 0);
  constexpr bool last = INV ? (r == 0) : (r == Sh::R - 1);
  if constexpr (first) {
    if constexpr (!INV && K == 2) {
      // stage 1 (m = L/2) on x_j and x_{j+Q}: CTA 0 keeps the sums (Algorithm 3 lines 1-2), CTA 1
      // the twiddled differences (lines 3-5, W = zeta_1^j).  The CTA-uniform choice is made outside
      // the element loops so the loads (data and twiddles) are scheduled ahead of their use.
      static_assert(G == 1 && S == SplitFwd<W, LOGQ, LE>::S, "first round: one column per thread");
      if (rank == 0) split_fwd_stage1<W, LOGQ, LE, LOGL, PLO1, false, PW, BF>(v, sm, t, tw_full, m, st, pw);
      else split_fwd_stage1<W, LOGQ, LE, LOGL, PLO1, true, PW, BF>(v, sm, t, tw_full, m, st, pw);
      // every CTA has read x_b (the loaded values are consumed, so a relaxed arrive orders them):
      // arrive here, wait only before the last round's in-place store.  Measured against a full
      // cluster.sync() at this point: u32 2^16 -7%, u64 2^15 -3% (the wait no longer stalls the
      // early CTA, and cluster.sync's MEMBAR.GPU + L1 invalidate are gone).
      if constexpr (!PW) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    } else if constexpr (!INV) {
      static_assert(BF == 3, "the K = 4 forward runs Algorithm 3 only");
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
      // every CTA has read x_b: in-place stores below are safe (K = 4 keeps one full barrier here;
      // K = 2 splits it into an arrive after stage 1 and a wait before the store)
      cluster.sync();
    } else {
      // this CTA's block of the bit-reversed input (contiguous runs, from shared memory);
      // PW: c = a b L^{-1} with b read from global memory 16 bytes at a time
      constexpr int PER = 16 / (int)sizeof(W);
      using St = SplitStaging<W, LOGQ, LE, K, INV, PW>;
      if constexpr (PW) {  // the whole block staged first (measured: 1.5% faster than overlapping the waits)
#pragma unroll
        for (int k = 0; k < St::NCH; ++k) mbar_wait(St::bar(smem_u32(sm), k), st.phase);
      }
      if constexpr (PW) {  // every b load in flight first (into v itself), then combine with a
#pragma unroll
        for (int q = 0; q < G; ++q)
#pragma unroll
          for (int h = 0; h < S; h += PER) {
            const size_t off = (size_t)rank * Q + blk[q] * S + h;
            unpack16<W>(__ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const W*>(pw.b) + boff + off)),
                        v + q * S + h);
          }
      }
      // this CTA's block of the transform has been staged in shared memory (without PW each group
      // waits for the chunk its run lies in)
      static_assert(St::CW % S == 0, "runs do not straddle chunks");
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const int e0 = blk[q] * S, k = e0 / St::CW;
        if constexpr (!PW) mbar_wait(St::bar(smem_u32(sm), k), st.phase);
        const W* src = reinterpret_cast<const W*>(reinterpret_cast<const unsigned char*>(sm) + St::slot(k)) - k * St::CW;
#pragma unroll
        for (int h = 0; h < S; h += PER) {
          W av[PER];
          unpack16<W>(lds128(src + tswz<W>(e0 + h)), av);
          if constexpr (PW) {
#pragma unroll
            for (int e = 0; e < PER; ++e) {
              W prod = mont_redc_mul<W>(av[e], v[q * S + h + e], (W)pw.J, m.p);
              v[q * S + h + e] = shoup_mul<W>(prod, (W)pw.K, (W)pw.Kp, m.p);
            }
          } else {
#pragma unroll
            for (int e = 0; e < PER; ++e) v[q * S + h + e] = av[e];
          }
        }
      }
      // no barrier needed here: the epilogue's cross-CTA accesses follow its own cluster barrier,
      // after every CTA has consumed its block
    }
  } else {
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) {
        if constexpr (REMAP || RUNV) {
          constexpr int PER = 16 / (int)sizeof(W);
#ifndef NTT_XP_NOEXCH
          if (h % PER == 0)
            unpack16<W>(lds128(sm + (RUNV ? tswz<W>(blk[q] * B + h) : xswz<W>(blk[q] * B + h))), v + q * S + h);
#else
          v[q * S + h] += (W)(blk[q] * B + h);
#endif
        } else {
#ifndef NTT_XP_NOEXCH
          constexpr int pr = INV ? r + 1 : r - 1;  // the round that wrote this exchange
          constexpr bool PLAIN = plain_exchange<LOGQ, LE, (int)sizeof(W), pr, r>();
          const int i = blk[q] * B + h * D + c[q];
          v[q * S + h] = sm[PLAIN ? i : sswz<W>(i)];
#else
          v[q * S + h] += (W)(blk[q] * B + h * D + c[q]);
#endif
        }
      }
  }
  if constexpr (PW && !INV && last) {
    // forward with the pointwise product: every thread has its last-round inputs, so the buffer
    // takes this CTA's block of a-hat (TMA) while the round computes
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      using F = SplitFwd<W, LOGQ, LE>;
      constexpr int ROWS = Q * (int)sizeof(W) / 128;
      const uint32_t abar = smem_u32(sm) + (uint32_t)F::SMEM;
      const int row0 = (int)((st.b * K + (size_t)rank) * (size_t)ROWS);
      mbar_expect_tx(abar, (uint32_t)(Q * sizeof(W)));
#pragma unroll
      for (int bx = 0; bx < ROWS / F::BOXR; ++bx)
        tma_load_2d(smem_u32(sm) + bx * F::BOXR * 128, st.map_a, 0, row0 + bx * F::BOXR, abar);
    }
  }
  if constexpr (!INV) dif_round<W, LOGQ, SR, LEVEL, G, PLO1, BF>(v, c, tw_sub, m);
  else dit_round<W, LOGQ, SR, LEVEL, G, PLO1>(v, c, tw_sub, m);
  if constexpr (last) {
    if constexpr (!INV) {
      if constexpr (PW) {
        // c-hat = a-hat b-hat L^{-1} with b-hat (already scaled by beta L^{-1} in stage 1, in
        // [0,2p)) straight from the registers: one REDC; c-hat in (0,2p) is a valid inverse input
        mbar_wait(smem_u32(sm) + (uint32_t)SplitFwd<W, LOGQ, LE>::SMEM, st.phase);
        constexpr int PER = 16 / (int)sizeof(W);
#pragma unroll
        for (int q = 0; q < G; ++q)
#pragma unroll
          for (int h = 0; h < S; h += PER) {
            W av[PER];
            unpack16<W>(lds128(sm + tswz<W>(blk[q] * S + h)), av);
#pragma unroll
            for (int e = 0; e < PER; ++e) v[q * S + h + e] = mont_redc_mul<W>(av[e], v[q * S + h + e], (W)pw.J, m.p);
          }
      } else {
#pragma unroll
        for (int i = 0; i < Sh::E; ++i) v[i] = norm2<W>(v[i], m.p);
      }
      // out through shared memory in the TMA 128-byte-swizzled layout and one bulk tensor store
      // of the block: per-thread strided 16-byte global stores congested the LSU (lg_throttle, and
      // long-scoreboard waits on the stores' source registers)
      static_assert(D == 1, "the forward's last round holds contiguous runs");
      constexpr int PER = 16 / (int)sizeof(W);
      // every thread has read its last-round inputs from sm (only its own warp's region when the
      // exchange into this round was warp-local and no a-hat was staged over the buffer)
      if constexpr (!PW && (REMAP || warp_local_exchange<LOGQ, LE, r - 1, r>())) __syncwarp();
      else __syncthreads();
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int h = 0; h < S; h += PER) sts128(sm + tswz<W>(blk[q] * S + h), pack16<W>(v + q * S + h));
      fence_proxy_async_smem();
      __syncthreads();
      // partner read x_b (PW: x is only read; c-hat goes to a's block, read only by this CTA)
      if constexpr (K == 2 && !PW) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
      if (threadIdx.x == 0) {
        constexpr int ROWS = Q * (int)sizeof(W) / 128;
        constexpr int BOX = (K == 2) ? SplitFwd<W, LOGQ, LE>::BOXR : (ROWS < 256 ? ROWS : 256);
        const int row0 = (int)((st.b * K + (size_t)rank) * (size_t)ROWS);
        const CUtensorMap* omap = PW ? st.map_a : st.map;
        // K = 2 with NTT_SPLIT_DRAIN: one bulk group per staging-chunk slot of the buffer, in slot order,
        // so the next transform's chunks can follow the store's reads slot by slot
        constexpr int PERG = (K == 2 && NTT_SPLIT_DRAIN) ? (int)(SplitFwd<W, LOGQ, LE>::CH / (BOX * 128)) : ROWS / BOX;
#pragma unroll
        for (int bx = 0; bx < ROWS / BOX; ++bx) {
          tma_store_2d(omap, 0, row0 + bx * BOX, smem_u32(sm) + bx * BOX * 128);
          if ((bx + 1) % PERG == 0) bulk_commit();
        }
      }
    } else {
      // stages s..1 across the cluster through DSMEM (Algorithm 4)
      constexpr int PER_CTA = Q / K;
      if constexpr (K == 2) {
        // Stage 1 across the pair, push model: thread t of either CTA holds positions j = hD + t of its
        // block (D = T here), so the two values of butterfly j sit in the same thread of the two CTAs.
        // Each CTA stores the half it does not finish straight from registers into the other's shared
        // memory (16-byte-free remote stores: no DSMEM load latency), keeps the other half in
        // registers, and after one cluster barrier finishes its half (CTA 0: h < S/2) with local loads.
        static_assert(G == 1 && D == Sh::T, "one column of the block per thread");
        constexpr int H2 = S / 2;
        // the other CTA has consumed its round inputs (relaxed: this CTA's inputs are consumed too,
        // the round's arithmetic used them) before this CTA's stores overwrite its buffer
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        if constexpr (NTT_SPLIT_STASYNC) {
          // asynchronous remote stores that count their bytes on the receiver's push mbarrier (armed
          // for H2 D words once per transform by its thread 0): the receiver waits on its own mbarrier,
          // with no cluster barrier and none of cluster.sync()'s release / acquire fences
          using St = SplitStaging<W, LOGQ, LE, K, INV, PW>;
          const uint32_t pbar = St::push_bar(smem_u32(sm));
          if (threadIdx.x == 0) mbar_expect_tx(pbar, (uint32_t)(H2 * D * sizeof(W)));
          const uint32_t rbase = mapa_u32(smem_u32(sm + t), (uint32_t)(rank ^ 1));
          const uint32_t rbar = mapa_u32(pbar, (uint32_t)(rank ^ 1));
#pragma unroll
          for (int h = 0; h < H2; ++h)
            st_async(rbase + (uint32_t)(h * D * sizeof(W)), rank == 0 ? v[H2 + h] : v[h], rbar);
          mbar_wait(pbar, st.phase);  // the other CTA's half has landed
        } else {
          W* other = cluster.map_shared_rank(sm, rank ^ 1);
          if (rank == 0) {
#pragma unroll
            for (int h = 0; h < H2; ++h) other[h * D + t] = v[H2 + h];
          } else {
#pragma unroll
            for (int h = 0; h < H2; ++h) other[h * D + t] = v[h];
          }
          cluster.sync();  // the pushed halves are visible
        }
        const int off = stage_off(LOGL, 1);
        constexpr int U = sizeof(W) == 4 ? 8 : 4;
        static_assert(H2 % U == 0, "whole groups");
        auto finish = [&](const W* mine_v, bool r0) {
          // -zeta_1^{-j} at entry Q - j of stage 1 (inv_index); the per-thread base is made opaque here
          // so its address arithmetic is not hoisted above the rounds (register pressure)
          uint32_t jr = (uint32_t)(off + Q - (r0 ? 0 : PER_CTA) - t);
          asm volatile("" : "+r"(jr));
#pragma unroll
          for (int h0 = 0; h0 < H2; h0 += U) {
            W u0[U], u1[U], w[U], wp[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const W theirs = sm[(h0 + u) * D + t];
              u0[u] = r0 ? mine_v[h0 + u] : theirs;  // x_j sits in CTA 0, x_{j+Q} in CTA 1
              u1[u] = r0 ? theirs : mine_v[h0 + u];
              ldtw<W>(tw_full, jr - (uint32_t)((h0 + u) * D), w[u], wp[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int j = (r0 ? 0 : PER_CTA) + (h0 + u) * D + t;
              bfly_alg4n<W, PLO1>(u0[u], u1[u], w[u], wp[u], m);
              xb[j] = norm4<W>(u0[u], m.p, m.p2);
              xb[j + Q] = norm4<W>(u1[u], m.p, m.p2);
            }
          }
        };
        if (rank == 0) finish(v, true);
        else finish(v + H2, false);
        // no trailing cluster barrier: the other CTA's next stores into this buffer come after the
        // next transform's pre-store barrier, which this CTA reaches only after these loads
      } else {
      __syncthreads();
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int h = 0; h < S; ++h) sm[sswz<W>(h * D + c[q])] = v[q * S + h];
      cluster.sync();
      {
        const W* part[K];
#pragma unroll
        for (int tt = 0; tt < K; ++tt) part[tt] = cluster.map_shared_rank(sm, tt);  // values at j + tt*Q
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
                ldtw<W>(tw_full, (uint32_t)(off + ((1 << LOGL) >> i) - (j + tt * Q)), w, wp);  // inv_index
                bfly_alg4n<W, PLO1>(u[bb + tt], u[bb + tt + half], w, wp, m);
              }
          }
#pragma unroll
          for (int tt = 0; tt < K; ++tt) xb[j + tt * Q] = norm4<W>(u[tt], m.p, m.p2);
        }
        cluster_sync_war();  // the other CTAs are done reading this CTA's shared memory
      }
      }
    }
  } else {
    // forward: the previous transform's bulk store must have read the buffer before it is reused
    if constexpr (!INV) {
      if (threadIdx.x == 0) bulk_wait_read0();
    }
    // The exchange next to the contiguous-run round is warp-local when its blocks fit a warp
    // (rounds.cuh).  The inverse's spare-slot refill needs every thread past its first round (a CTA
    // barrier): it rides on the first exchange, or on the second when the first is warp-local.
    constexpr int nr_ = INV ? r - 1 : r + 1;
    constexpr bool NEXT_REMAP = !INV && split_remap_last<LOGQ, LE, nr_>();  // writes into the remapped round
    constexpr bool NEXT_RUNV = !INV && runv_round<LOGQ, LE, (int)sizeof(W), nr_>();
    constexpr bool WL = (warp_local_exchange<LOGQ, LE, r, nr_>() || NEXT_REMAP) && !(INV && Sh::R < 3);
    constexpr bool FIRST_WL = INV && Sh::R >= 3 && warp_local_exchange<LOGQ, LE, Sh::R - 1, Sh::R - 2>();
    using St = SplitStaging<W, LOGQ, LE, K, INV, PW>;
    constexpr bool REFILL = INV && St::NX > 0 && (FIRST_WL ? r == Sh::R - 2 : first);
    // forward (K = 2): the first round's exchange barrier also tells that stage 1 has consumed every
    // staged chunk, so the spare slots take the next transform's first chunks there
    constexpr bool FWD_REFILL = !INV && K == 2 && first;
    if constexpr (REFILL || FWD_REFILL) fence_proxy_async_smem();
    if constexpr (WL) __syncwarp();
    else __syncthreads();
    if constexpr (FWD_REFILL) {
      using F = SplitFwd<W, LOGQ, LE>;
      if (threadIdx.x == 0 && st.next_b < st.batch)
#pragma unroll
        for (int kk = 0; kk < F::NX; ++kk) F::issue(st.map, st.next_b, kk, smem_u32(sm));
    }
    if constexpr (REFILL) {  // the spare slots take the next transform's chunks
      if (threadIdx.x == 0 && st.next_b < st.batch) St::issue(st.map, st.next_b, rank, 0, St::NX, smem_u32(sm));
    }
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) {
        const int i = blk[q] * B + h * D + c[q];
#ifndef NTT_XP_NOEXCH
        constexpr bool PLAIN = plain_exchange<LOGQ, LE, (int)sizeof(W), r, nr_>();
        sm[NEXT_REMAP ? xswz<W>(i) : (NEXT_RUNV ? tswz<W>(i) : (PLAIN ? i : sswz<W>(i)))] = v[q * S + h];
#else
        if (i == 0) sm[0] = v[q * S + h];
#endif
      }
    if constexpr (WL) __syncwarp();
    else __syncthreads();
    constexpr int nr = INV ? r - 1 : r + 1;
    split_round<W, LOGQ, LE, K, INV, PLO1, PW, BF, nr>(v, xb, sm, t, rank, tw_full, m, pw, boff, cluster, st);
  }
}

template <class W, int LOGQ, int LE, int K, bool INV, bool PLO1, bool PW, int BF>
__global__ void __launch_bounds__(SplitShape<LOGQ, LE, K, (int)sizeof(W)>::T,
                                  SplitShape<LOGQ, LE, K, (int)sizeof(W)>::MINB)
    k_splitk(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_a, W* __restrict__ x,
             size_t batch,
             const TwPair<W>* __restrict__ tw_full, W p, PwArgs pw) {
  using Sh = SplitShape<LOGQ, LE, K, (int)sizeof(W)>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // dynamic shared memory starts 1024-byte aligned (tma.cuh), as the TMA swizzle period needs
  W* sm = reinterpret_cast<W*>(smem_raw);
  using St = SplitStaging<W, LOGQ, LE, K, INV, PW>;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int t = threadIdx.x;
  const Mod<W> m = make_mod<W>(p);
  SplitStage st{&tmap, 0u, 0, 0, batch, &tmap_a};
  if constexpr (St::ON) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < St::NCH; ++k) mbar_init(St::bar(smem_u32(sm), k), 1);
      if constexpr (K == 2 && NTT_SPLIT_STASYNC) mbar_init(St::push_bar(smem_u32(sm)), 1);
      fence_mbar_init();
    }
    // the partner's st.async pushes signal this CTA's push mbarrier: its initialisation must be
    // visible cluster-wide first (the epilogue's own cluster barrier is a relaxed one)
    if constexpr (K == 2 && NTT_SPLIT_STASYNC) cluster.sync();
    else __syncthreads();
  }
  constexpr bool FWD_TMA = !INV && K == 2;
  using F = SplitFwd<W, LOGQ, LE>;
  W v[Sh::E];
  const size_t groups = gridDim.x / K;
  size_t b = blockIdx.x / K;
  if constexpr (FWD_TMA) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < F::NCH; ++k) mbar_init(smem_u32(sm) + F::BAR_OFF + 8 * k, 1);
      if constexpr (PW) mbar_init(smem_u32(sm) + (uint32_t)F::SMEM, 1);  // a-hat staging
      fence_mbar_init();
      if (b < batch)
#pragma unroll
        for (int k = 0; k < F::NX; ++k) F::issue(&tmap, b, k, smem_u32(sm));
    }
    __syncthreads();
  }
  if (St::ON && threadIdx.x == 0 && b < batch) St::issue(st.map, b, rank, 0, St::NCH, smem_u32(sm));
  for (uint32_t it = 0; b < batch; b += groups, ++it) {
    const size_t boff = b * (size_t)K * Sh::Q;
    st.phase = it & 1;
    st.b = b;
    st.next_b = b + groups;
    if constexpr (FWD_TMA && !NTT_SPLIT_DRAIN) {
      // the Q-word buffer takes chunks NX..NX+3 once the previous transform's store has read it
      if (threadIdx.x == 0) {
        bulk_wait_read0();
#pragma unroll
        for (int k = F::NX; k < F::NX + F::NB; ++k) F::issue(&tmap, b, k, smem_u32(sm));
      }
    }
    constexpr int r0 = INV ? Sh::R - 1 : 0;
    split_round<W, LOGQ, LE, K, INV, PLO1, PW, BF, r0>(v, x + boff, sm, t, rank, tw_full, m, pw, boff, cluster, st);
    if constexpr (INV) {
      // after the epilogue's cluster barrier no CTA reads this buffer any more
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0 && st.next_b < batch) St::issue(st.map, st.next_b, rank, St::NX, St::NCH, smem_u32(sm));
    }
    __syncthreads();
  }
  if constexpr (!INV) {
    if (threadIdx.x == 0) bulk_wait_read0();  // the last bulk store has read shared memory
  }
}

template <class W, int K> struct SplitLE { static constexpr int value = 5; };

template <class W, int LOGL, int K, bool INV, bool PLO1, bool PW, int BF = 3>
static cudaError_t run_split(void* x, size_t batch, const void* tw, uint64_t p, const PwArgs& pw, cudaStream_t s) {
  constexpr int LOGQ = LOGL - (K == 4 ? 2 : 1);
  constexpr int LE = SplitLE<W, K>::value;
  using Sh = SplitShape<LOGQ, LE, K, (int)sizeof(W)>;
  constexpr bool FWD_TMA = !INV && K == 2;
  const size_t smem = FWD_TMA ? SplitFwd<W, LOGQ, LE>::SMEM + (PW ? 8 : 0)
                              : (SplitStaging<W, LOGQ, LE, K, INV, PW>::ON ? SplitStaging<W, LOGQ, LE, K, INV, PW>::SMEM
                                                                       : (size_t)Sh::Q * sizeof(W));
  auto enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  // 2-D tensor maps of 128-byte rows: map over the array the first round reads (x; a for the
  // inverse with PW), map_a over a for the forward with PW (a-hat in, c-hat out)
  constexpr int ROW_WORDS = 128 / (int)sizeof(W);
  constexpr int ROWS = Sh::Q / ROW_WORDS;
  CUtensorMap maps[2];
  void* srcs[2] = {(INV && PW) ? const_cast<void*>(pw.a) : x, PW ? const_cast<void*>(pw.a) : x};
  for (int i = 0; i < 2; ++i) {
    cuuint64_t dims[2] = {(cuuint64_t)ROW_WORDS, (cuuint64_t)(batch * K * (size_t)Sh::Q / ROW_WORDS)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {(cuuint32_t)ROW_WORDS,
                         (cuuint32_t)(FWD_TMA ? SplitFwd<W, LOGQ, LE>::BOXR : (ROWS < 256 ? ROWS : 256))};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&maps[i], sizeof(W) == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
                      srcs[i], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  auto kern = k_splitk<W, LOGQ, LE, K, INV, PLO1, PW, BF>;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  static PerDevice mc_cache;
  const int max_clusters = mc_cache.get([&] {
    int mc = 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(K * 1024);
    q.blockDim = dim3(Sh::T);
    q.dynamicSmemBytes = smem;
    q.attrs = attr;
    q.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &q) != cudaSuccess || mc <= 0) {
      cudaGetLastError();
      mc = sm_count() / K;
    }
    return mc;
  });
  const size_t groups = batch < (size_t)max_clusters ? batch : (size_t)max_clusters;
  if (!groups) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(groups * K));
  cfg.blockDim = dim3(Sh::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], reinterpret_cast<W*>(x), batch,
                            reinterpret_cast<const TwPair<W>*>(tw), (W)p, pw);
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
                          const void* pw_a, const void* pw_b, uint64_t J, uint64_t K, uint64_t Kp, cudaStream_t s,
                          const void* tw1s, int bf) {
  PwArgs pw{pw_a, pw_b, J, K, Kp, tw1s};
  if (bf != 3) {  // ablations F1 / F2: the plain forward on 2-CTA clusters (J for Algorithm 5)
    if (inverse || pw_a || split_k() != 2 || (bf != 2 && bf != 5)) return cudaErrorNotSupported;
    if (wbytes == 8) {
      if (logn != kContigMaxLog64 + 1) return cudaErrorInvalidValue;
      constexpr int L = kContigMaxLog64 + 1;
      const bool plo1 = (p & 0xffffffffull) == 1;
      if (bf == 5) return run_split<uint64_t, L, 2, false, false, false, 5>(x, batch, tw, p, pw, s);
      return plo1 ? run_split<uint64_t, L, 2, false, true, false, 2>(x, batch, tw, p, pw, s)
                  : run_split<uint64_t, L, 2, false, false, false, 2>(x, batch, tw, p, pw, s);
    }
    if (logn != kContigMaxLog32 + 1) return cudaErrorInvalidValue;
    constexpr int L = kContigMaxLog32 + 1;
    if (bf == 5) return run_split<uint32_t, L, 2, false, false, false, 5>(x, batch, tw, p, pw, s);
    return run_split<uint32_t, L, 2, false, false, false, 2>(x, batch, tw, p, pw, s);
  }
  // fused (pw_a set): inverse -- a <- InvNTT(a * b L^{-1}); forward -- a <- NTT(x) * a L^{-1}, x only
  // read (K = 2 only)
  const bool fused = pw_a != nullptr;
  if (fused && !inverse && (split_k() != 2 || !tw1s)) return cudaErrorNotSupported;
  if (wbytes == 8) {
    if (logn != kContigMaxLog64 + 1) return cudaErrorInvalidValue;
    constexpr int L = kContigMaxLog64 + 1;
    const bool plo1 = (p & 0xffffffffull) == 1;
    if (!inverse && fused) return plo1 ? run_split<uint64_t, L, 2, false, true, true>(x, batch, tw, p, pw, s)
                                       : run_split<uint64_t, L, 2, false, false, true>(x, batch, tw, p, pw, s);
    if (!inverse) return plo1 ? run_split_k<uint64_t, L, false, true, false>(x, batch, tw, p, pw, s)
                              : run_split_k<uint64_t, L, false, false, false>(x, batch, tw, p, pw, s);
    if (fused) return plo1 ? run_split_k<uint64_t, L, true, true, true>(x, batch, tw, p, pw, s)
                           : run_split_k<uint64_t, L, true, false, true>(x, batch, tw, p, pw, s);
    return plo1 ? run_split_k<uint64_t, L, true, true, false>(x, batch, tw, p, pw, s)
                : run_split_k<uint64_t, L, true, false, false>(x, batch, tw, p, pw, s);
  }
  if (logn != kContigMaxLog32 + 1) return cudaErrorInvalidValue;
  constexpr int L = kContigMaxLog32 + 1;
  if (!inverse && fused) return run_split<uint32_t, L, 2, false, false, true>(x, batch, tw, p, pw, s);
  if (!inverse) return run_split_k<uint32_t, L, false, false, false>(x, batch, tw, p, pw, s);
  if (fused) return run_split_k<uint32_t, L, true, false, true>(x, batch, tw, p, pw, s);
  return run_split_k<uint32_t, L, true, false, false>(x, batch, tw, p, pw, s);
}

}  // namespace nttb
