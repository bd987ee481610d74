// ntt_kernels.cu -- sm_100a kernels of the batched NTT engine.
//
// Algorithm 1 is executed as "rounds": a thread holds
// E = 2^LE words in registers and runs up to LE consecutive radix-2 stages on
// them (the lazy butterflies of modarith.cuh); between rounds the CTA exchanges
// data through an XOR-swizzled shared-memory tile.  The first round reads HBM
// directly into registers (coalesced across lanes) and the last round writes
// back (vectorised), so a transform that fits on chip costs one HBM read and one
// HBM write.  Longer transforms use the nested four-step schedule of DESIGN.md
// (column passes with the fused twiddle, then a contiguous row pass).
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"
#include "modarith.cuh"
#include "rounds.cuh"
#include "fourstep.cuh"

namespace nttb {

// ----------------------------------------------------------------- helpers
// XOR swizzle of the word index inside a 128-byte smem row (v1 kernel), so that
// the strided exchange patterns of every round hit distinct banks.
template <class W> __device__ __forceinline__ int swz(int i) {
  constexpr int S = sizeof(W) == 8 ? 4 : 5;
  return i ^ ((i >> S) & ((1 << S) - 1));
}

// ----------------------------------------------------------------- contiguous single-pass kernel
// K transforms of N = 2^LOGN words per CTA iteration; T = N / 2^LE threads each.
// GATHER (config C5 row pass): the input row is the concatenation of 2^log_world
// column blocks of the all-to-all receive buffer (see ntt_fourstep_rows).
template <int LOGN, int LE> struct ContigShape {
  static constexpr int N = 1 << LOGN;
  static constexpr int E = 1 << LE;
  static constexpr int T = N / E;
  static constexpr int K = T >= 256 ? 1 : 256 / T;
  static constexpr int THREADS = K * T;
  static constexpr int MINB = THREADS >= 512 ? 1 : 512 / THREADS;
  using RC = Rounds<LOGN, LE>;
  static constexpr int R = RC::R;
};

// GATHER: forward (config C5 row pass) reads its row from the all-to-all receive blocks;
// inverse (distributed inverse, F4) writes its natural-order row into the send blocks.
struct GatherArgs {
  void* ext;                  // receive buffer (forward) / send buffer (inverse), or nullptr
  uint32_t log_w;             // log2(N2/G): width of one block
  uint32_t log_rows_local;    // log2(N1/G): rows per block
  // inverse with the all-to-all fused (ntt_fourstep_rows_inv_p2p): block hb of row `row` goes to
  // block src_rank of rank hb's receive buffer peer[hb] (peer memory over NVLink)
  uint32_t p2p, src_rank;
  uint64_t peer[8];
};

template <class W, int LOGN, int LE, bool INV, bool GATHER, bool PLO1, int r>
__device__ __forceinline__ void contig_round(W* v, W* __restrict__ xb, const W* __restrict__ gin, size_t row,
                                             const GatherArgs& ga, W* sb, int t, bool active,
                                             const TwPair<W>* __restrict__ tw, const Mod<W>& m, bool norm) {
  NTT_AUDIT_STRESS();  // audit build only: per-warp random delay before the round reads its inputs
  const W p = m.p, p2 = m.p2;
  using Sh = ContigShape<LOGN, LE>;
  using RC = typename Sh::RC;
  constexpr int SR = RC::sr(r), LEVEL = RC::level(r);
  constexpr int S = 1 << SR, G = Sh::E >> SR;
  constexpr int D = Sh::N >> (LEVEL + SR), B = Sh::N >> LEVEL;
  int c[G], blk[G];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = t + Sh::T * q;
    blk[q] = g / D;
    c[q] = g % D;
  }
  constexpr bool first = INV ? (r == Sh::R - 1) : (r == 0);
  constexpr bool last = INV ? (r == 0) : (r == Sh::R - 1);
  // ---- load
  if constexpr (first) {
    if constexpr (!INV) {  // natural order, strided per thread, coalesced across lanes
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int h = 0; h < S; ++h) {
          const int i = h * D + c[q];
          W val = 0;
          if (active) {
            if constexpr (GATHER) {
              const int hb = i >> ga.log_w, off = i & ((1 << ga.log_w) - 1);
              val = gin[(((size_t)hb << ga.log_rows_local) + row) << ga.log_w | off];
            } else {
              val = xb[i];
            }
          }
          v[q * S + h] = val;
        }
    } else {  // bit-reversed input, contiguous runs
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (active) load_run<W, S>(xb + blk[q] * S, v + q * S);
        else
#pragma unroll
          for (int h = 0; h < S; ++h) v[q * S + h] = 0;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) v[q * S + h] = sb[swz<W>(blk[q] * B + h * D + c[q])];
  }
  // ---- compute
  if constexpr (!INV) dif_round<W, LOGN, SR, LEVEL, G, PLO1>(v, c, tw, m);
  else dit_round<W, LOGN, SR, LEVEL, G, PLO1>(v, c, tw, m);
  // ---- store
  if constexpr (last) {
    if (norm) {
#pragma unroll
      for (int i = 0; i < Sh::E; ++i) v[i] = INV ? norm4<W>(v[i], p, p2) : norm2<W>(v[i], p);
    }
    if (active) {
      if constexpr (!INV) {
#pragma unroll
        for (int q = 0; q < G; ++q) store_run<W, S>(xb + blk[q] * S, v + q * S);
      } else {
#pragma unroll
        for (int q = 0; q < G; ++q)
#pragma unroll
          for (int h = 0; h < S; ++h) {
            const int i = h * D + c[q];
            if constexpr (GATHER) {  // scatter: element i of row `row` -> block i >> log_w
              const int hb = i >> ga.log_w, off = i & ((1 << ga.log_w) - 1);
              if (ga.p2p)
                reinterpret_cast<W*>(select_peer(ga.peer, (uint32_t)hb))[(((size_t)ga.src_rank << ga.log_rows_local) + row)
                                                                         << ga.log_w | off] =
                    v[q * S + h];
              else
                reinterpret_cast<W*>(ga.ext)[(((size_t)hb << ga.log_rows_local) + row) << ga.log_w | off] = v[q * S + h];
            } else {
              xb[i] = v[q * S + h];
            }
          }
      }
    }
  } else {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int h = 0; h < S; ++h) sb[swz<W>(blk[q] * B + h * D + c[q])] = v[q * S + h];
    __syncthreads();
    constexpr int nr = INV ? r - 1 : r + 1;
    contig_round<W, LOGN, LE, INV, GATHER, PLO1, nr>(v, xb, gin, row, ga, sb, t, active, tw, m, norm);
  }
}

template <class W, int LOGN, int LE, bool INV, bool GATHER, bool PLO1>
__global__ void __launch_bounds__(ContigShape<LOGN, LE>::THREADS, ContigShape<LOGN, LE>::MINB)
    k_contig(W* __restrict__ x, size_t batch, const TwPair<W>* __restrict__ tw, W p, int norm, GatherArgs ga) {
  using Sh = ContigShape<LOGN, LE>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);
  const int slot = threadIdx.x / Sh::T, t = threadIdx.x % Sh::T;
  const Mod<W> m = make_mod<W>(p);
  W v[Sh::E];
  for (size_t b0 = (size_t)blockIdx.x * Sh::K; b0 < batch; b0 += (size_t)gridDim.x * Sh::K) {
    const size_t b = b0 + slot;
    const bool active = b < batch;
    W* xb = x + b * Sh::N;
    constexpr int r0 = INV ? Sh::R - 1 : 0;
    contig_round<W, LOGN, LE, INV, GATHER, PLO1, r0>(v, xb, reinterpret_cast<const W*>(ga.ext), b, ga, sm + slot * Sh::N,
                                                     t, active, tw, m, norm != 0);
  }
}


// ----------------------------------------------------------------- pointwise, normalise
// c = a b L^{-1} mod p: Montgomery REDC in the Alg. 5 pattern gives
// a b beta^{-1} in (0,2p); a Shoup multiply by K = beta L^{-1} mod p (or beta mod p
// without scaling) restores the scale; then normalise.
template <class W>
__global__ void k_pointwise(W* __restrict__ c, const W* __restrict__ a, const W* __restrict__ b, size_t n, W p, W J,
                            W K, W Kp, int vec) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t done = 0;
  if (vec) {  // 16-byte vectors (all three pointers 16-byte aligned), streaming loads and stores
    constexpr int PER = 16 / (int)sizeof(W);
    const size_t nv = n / PER;
    for (size_t i = i0; i < nv; i += stride) {
      W av[PER], bv[PER], cv[PER];
      unpack16<W>(__ldcs(reinterpret_cast<const uint4*>(a) + i), av);
      unpack16<W>(__ldcs(reinterpret_cast<const uint4*>(b) + i), bv);
#pragma unroll
      for (int e = 0; e < PER; ++e) cv[e] = norm2<W>(shoup_mul<W>(mont_redc_mul<W>(av[e], bv[e], J, p), K, Kp, p), p);
      __stcs(reinterpret_cast<uint4*>(c) + i, pack16<W>(cv));
    }
    done = nv * PER;
  }
  for (size_t i = done + i0; i < n; i += stride) {
    W r = mont_redc_mul<W>(a[i], b[i], J, p);
    r = shoup_mul<W>(r, K, Kp, p);
    c[i] = norm2<W>(r, p);
  }
}

template <class W> __global__ void k_normalize(W* __restrict__ x, size_t n, W p, int from4p) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const W p2 = 2 * p;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    x[i] = from4p ? norm4<W>(x[i], p, p2) : norm2<W>(x[i], p);
}

template <class W, bool PLO1>
__global__ void k_debug_bfly(int alg, const W* __restrict__ Wv, const W* __restrict__ Wpv, W* __restrict__ X,
                             W* __restrict__ Y, size_t n, W p, W J) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  W x = X[i], y = Y[i];
  const Mod<W> m = make_mod<W>(p);
  const W p2 = m.p2;
  switch (alg) {  // the transform kernels' exact arithmetic (PLO1 when p = 1 mod 2^32)
    case 2: bfly_alg2<W>(x, y, Wv[i], Wpv[i], p); break;
    case 3: bfly_alg3<W, PLO1>(x, y, Wv[i], Wpv[i], m); break;
    case 31: bfly_alg3_w1<W>(x, y, p2); break;
    case 4: bfly_alg4<W, PLO1>(x, y, Wv[i], Wpv[i], m); break;
    case 41: bfly_alg4_w1<W>(x, y, p2); break;
    case 5: bfly_alg5<W>(x, y, Wpv[i], J, p, p2); break;
    default: break;
  }
  X[i] = x;
  Y[i] = y;
}

// ----------------------------------------------------------------- ALU calibration
// Register-only Algorithm 3 loop: 8 independent butterfly chains per thread.
template <class W, bool PLO1>
__global__ void __launch_bounds__(256) k_calib(W* sink, W p, W w, W wp, unsigned iters) {
  constexpr int CH = 8;
  W x[CH], y[CH];
  const Mod<W> m = make_mod<W>(p);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = (W)(threadIdx.x * 7 + c) % p;
    y[c] = (W)(threadIdx.x * 13 + 3 * c) % p;
  }
  for (unsigned i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) bfly_alg3<W, PLO1>(x[c], y[c], w, wp, m);
  W s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= x[c] ^ y[c];
  if (s == (W)0x12345678u) sink[0] = s;
}

// ----------------------------------------------------------------- launch plumbing
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

// per-(W, LOGN) elements-per-thread choice
template <class W, int LOGN> struct ContigLE {
  static constexpr int value = sizeof(W) == 8 ? (LOGN <= 4 ? LOGN : (LOGN <= 13 ? 4 : 5))
                                              : (LOGN <= 5 ? LOGN : 5);
};

template <class W, int LOGN, bool INV, bool GATHER, bool PLO1>
static cudaError_t run_contig(void* x, size_t batch, const void* tw, uint64_t p, bool norm, GatherArgs ga,
                              cudaStream_t s) {
  constexpr int LE = ContigLE<W, LOGN>::value;
  using Sh = ContigShape<LOGN, LE>;
  const size_t smem = Sh::R > 1 ? (size_t)Sh::K * Sh::N * sizeof(W) : 0;
  auto kern = k_contig<W, LOGN, LE, INV, GATHER, PLO1>;
  static PerDevice occ_cache;
  const int occ = occ_cache.get([&] { return occupancy(kern, Sh::THREADS, smem); });
  const size_t iters = (batch + Sh::K - 1) / Sh::K;
  const size_t maxg = (size_t)occ * num_sms();
  const unsigned grid = (unsigned)(iters < maxg ? iters : maxg);
  if (!grid) return cudaSuccess;
  kern<<<grid, Sh::THREADS, smem, s>>>(reinterpret_cast<W*>(x), batch, reinterpret_cast<const TwPair<W>*>(tw),
                                       (W)p, norm ? 1 : 0, ga);
  return cudaGetLastError();
}

template <class W, bool INV, bool GATHER, int LO, int HI>
static cudaError_t contig_dispatch(int logn, void* x, size_t batch, const void* tw, uint64_t p, bool norm,
                                   GatherArgs ga, cudaStream_t s) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (logn == LO) {
      if constexpr (sizeof(W) == 8) {
        if ((p & 0xffffffffull) == 1) return run_contig<W, LO, INV, GATHER, true>(x, batch, tw, p, norm, ga, s);
      }
      return run_contig<W, LO, INV, GATHER, false>(x, batch, tw, p, norm, ga, s);
    }
    return contig_dispatch<W, INV, GATHER, LO + 1, HI>(logn, x, batch, tw, p, norm, ga, s);
  }
}

cudaError_t launch_contig(int wbytes, int logn, bool inverse, bool normalize, void* x, size_t batch, const void* tw,
                          uint64_t p, cudaStream_t s) {
  GatherArgs ga{nullptr, 0, 0, 0u, 0u, {}};
  if (wbytes == 8) {
    return inverse ? contig_dispatch<uint64_t, true, false, 1, kContigMaxLog64>(logn, x, batch, tw, p, normalize, ga, s)
                   : contig_dispatch<uint64_t, false, false, 1, kContigMaxLog64>(logn, x, batch, tw, p, normalize, ga, s);
  }
  return inverse ? contig_dispatch<uint32_t, true, false, 1, kContigMaxLog32>(logn, x, batch, tw, p, normalize, ga, s)
                 : contig_dispatch<uint32_t, false, false, 1, kContigMaxLog32>(logn, x, batch, tw, p, normalize, ga, s);
}

cudaError_t launch_rows_gather(int wbytes, int logn2, void* out, const void* recv, uint32_t log_rows_local,
                               uint32_t log_world, const void* tw, uint64_t p, cudaStream_t s) {
  GatherArgs ga{const_cast<void*>(recv), (uint32_t)logn2 - log_world, log_rows_local, 0u, 0u, {}};
  const size_t rows = (size_t)1 << log_rows_local;
  if (wbytes == 8)
    return contig_dispatch<uint64_t, false, true, 5, kContigMaxLog64>(logn2, out, rows, tw, p, true, ga, s);
  return contig_dispatch<uint32_t, false, true, 5, kContigMaxLog32>(logn2, out, rows, tw, p, true, ga, s);
}

cudaError_t launch_rows_scatter(int wbytes, int logn2, const void* in, void* send, uint32_t log_rows_local,
                                uint32_t log_world, const void* tw_inv, uint64_t p, cudaStream_t s,
                                const uint64_t* peers, uint32_t src_rank) {
  GatherArgs ga{send, (uint32_t)logn2 - log_world, log_rows_local, 0u, 0u, {}};
  if (peers) {
    ga.p2p = 1;
    ga.src_rank = src_rank;
    for (uint32_t h = 0; h < (1u << log_world) && h < 8; ++h) ga.peer[h] = peers[h];
  }
  const size_t rows = (size_t)1 << log_rows_local;
  void* x = const_cast<void*>(in);  // read only: the inverse's scatter writes to `send`
  if (wbytes == 8)
    return contig_dispatch<uint64_t, true, true, 5, kContigMaxLog64>(logn2, x, rows, tw_inv, p, true, ga, s);
  return contig_dispatch<uint32_t, true, true, 5, kContigMaxLog32>(logn2, x, rows, tw_inv, p, true, ga, s);
}

// ----------------------------------------------------------------- block transpose
// dst[j][i][k] = src[i][j][k] (i < n0, j < n1, k < n2): the pack / unpack of the
// distributed four-step's contiguous-layout variants (F4).  HBM-bound copy; each warp
// moves one contiguous run of n2 words with 16-byte accesses when aligned.
template <class W>
__global__ void k_block_transpose(W* __restrict__ dst, const W* __restrict__ src, uint64_t n0, uint64_t n1,
                                  uint64_t n2) {
  const uint64_t runs = n0 * n1;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int PER = 16 / sizeof(W);
  const bool vec = (n2 % PER) == 0;
  for (uint64_t rr = warp; rr < runs; rr += nwarps) {
    const uint64_t i = rr / n1, j = rr % n1;
    const W* s = src + rr * n2;
    W* d = dst + (j * n0 + i) * n2;
    if (vec) {
      for (uint64_t k = (uint64_t)lane * PER; k < n2; k += 32 * PER)
        *reinterpret_cast<uint4*>(d + k) = __ldcs(reinterpret_cast<const uint4*>(s + k));
    } else {
      for (uint64_t k = lane; k < n2; k += 32) d[k] = s[k];
    }
  }
}

cudaError_t launch_block_transpose(int wbytes, void* dst, const void* src, uint64_t n0, uint64_t n1, uint64_t n2,
                                   cudaStream_t s) {
  if (!n0 || !n1 || !n2) return cudaSuccess;
  const int th = 256;
  const uint64_t warps = n0 * n1;
  uint64_t g = (warps * 32 + th - 1) / th;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  const unsigned grid = (unsigned)(g < cap ? g : cap);
  if (wbytes == 8)
    k_block_transpose<uint64_t><<<grid, th, 0, s>>>((uint64_t*)dst, (const uint64_t*)src, n0, n1, n2);
  else
    k_block_transpose<uint32_t><<<grid, th, 0, s>>>((uint32_t*)dst, (const uint32_t*)src, n0, n1, n2);
  return cudaGetLastError();
}

unsigned elementwise_grid(size_t n, int threads);

// ----------------------------------------------------------------- three-prime CRT (F3)
// Garner's mixed-radix reconstruction of x in [0, p0 p1 p2) from residues r_i < p_i
// (the RNS use of P:21): v0 = r0, v1 = (r1 - v0) p0^{-1} mod p1,
// v2 = ((r2 - v0) p0^{-1} - v1) p1^{-1} mod p2, x = v0 + v1 p0 + v2 p0 p1.  Every
// multiply by a constant is a Shoup multiply with a host-precomputed W';
// the subtractions add a multiple of the modulus so each Shoup input stays < 2^32.
__global__ void k_crt3(uint64_t* __restrict__ out, const uint32_t* __restrict__ r0, const uint32_t* __restrict__ r1,
                       const uint32_t* __restrict__ r2, size_t n, Crt3Consts k) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t v0 = __ldcs(r0 + i);
    uint32_t v1 = shoup_mul<uint32_t>(__ldcs(r1 + i) + k.K1 - v0, k.c01, k.c01p, k.p1);  // [0, 2 p1)
    v1 = csub<uint32_t>(v1, k.p1);
    uint32_t u = shoup_mul<uint32_t>(__ldcs(r2 + i) + k.K2 - v0, k.c02, k.c02p, k.p2);  // [0, 2 p2)
    uint32_t v2 = shoup_mul<uint32_t>(u + k.K3 - v1, k.c12, k.c12p, k.p2);
    v2 = csub<uint32_t>(v2, k.p2);
    // x = v0 + v1 p0 + v2 (p0 p1): the last term is up to 2^92, so 128-bit
    const uint64_t a = (uint64_t)v0 + (uint64_t)v1 * k.p0;  // < p0 p1 <= 2^62
    const uint64_t lo = (uint64_t)v2 * k.p01, hi = __umul64hi((uint64_t)v2, k.p01);
    const uint64_t xlo = lo + a;
    const uint64_t xhi = hi + (xlo < lo ? 1u : 0u);
    __stcs(reinterpret_cast<ulonglong2*>(out) + i, make_ulonglong2(xlo, xhi));
  }
}

cudaError_t launch_crt3(uint64_t* out, const uint32_t* r0, const uint32_t* r1, const uint32_t* r2, size_t n,
                        const Crt3Consts& k, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const int th = 256;
  k_crt3<<<elementwise_grid(n, th), th, 0, s>>>(out, r0, r1, r2, n, k);
  return cudaGetLastError();
}

cudaError_t launch_pointwise(int wbytes, void* c, const void* a, const void* b, size_t n, uint64_t p, uint64_t J,
                             uint64_t K, uint64_t Kp, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const int th = 256;
  const int vec = (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 15) == 0;
  const size_t nthreads = vec ? n / (16 / wbytes) + 1 : n;
  if (wbytes == 8)
    k_pointwise<uint64_t><<<elementwise_grid(nthreads, th), th, 0, s>>>(
        (uint64_t*)c, (const uint64_t*)a, (const uint64_t*)b, n, p, J, K, Kp, vec);
  else
    k_pointwise<uint32_t><<<elementwise_grid(nthreads, th), th, 0, s>>>(
        (uint32_t*)c, (const uint32_t*)a, (const uint32_t*)b, n, (uint32_t)p, (uint32_t)J, (uint32_t)K, (uint32_t)Kp,
        vec);
  return cudaGetLastError();
}

// Range-checking mode: flag[0] |= 1 if any word is >= bound.
template <class W>
__global__ void k_check_range(const W* __restrict__ x, size_t n, W bound, unsigned* flag) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) bad |= x[i] >= bound;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

cudaError_t launch_check_range(int wbytes, const void* x, size_t n, uint64_t bound, unsigned* flag, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const int th = 256;
  if (wbytes == 8)
    k_check_range<uint64_t><<<elementwise_grid(n, th), th, 0, s>>>((const uint64_t*)x, n, bound, flag);
  else
    k_check_range<uint32_t><<<elementwise_grid(n, th), th, 0, s>>>((const uint32_t*)x, n, (uint32_t)bound, flag);
  return cudaGetLastError();
}

cudaError_t launch_normalize(int wbytes, void* x, size_t n, uint64_t p, int from4p, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const int th = 256;
  if (wbytes == 8) k_normalize<uint64_t><<<elementwise_grid(n, th), th, 0, s>>>((uint64_t*)x, n, p, from4p);
  else k_normalize<uint32_t><<<elementwise_grid(n, th), th, 0, s>>>((uint32_t*)x, n, (uint32_t)p, from4p);
  return cudaGetLastError();
}

cudaError_t launch_calib(int wbytes, uint64_t p, uint64_t w, uint64_t wp, unsigned iters, void* sink,
                         uint64_t* n_bfly, cudaStream_t s) {
  const unsigned grid = (unsigned)num_sms() * 8, th = 256;
  *n_bfly = (uint64_t)grid * th * 8 * iters;
  if (wbytes == 8) {
    if ((p & 0xffffffffull) == 1) k_calib<uint64_t, true><<<grid, th, 0, s>>>((uint64_t*)sink, p, w, wp, iters);
    else k_calib<uint64_t, false><<<grid, th, 0, s>>>((uint64_t*)sink, p, w, wp, iters);
  } else {
    k_calib<uint32_t, false><<<grid, th, 0, s>>>((uint32_t*)sink, (uint32_t)p, (uint32_t)w, (uint32_t)wp, iters);
  }
  return cudaGetLastError();
}

cudaError_t launch_debug_bfly(int wbytes, int alg, const void* W, const void* Wp, void* X, void* Y, size_t n,
                              uint64_t p, uint64_t J, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const int th = 256;
  const unsigned grid = (unsigned)((n + th - 1) / th);
  if (wbytes == 8) {
    if ((p & 0xffffffffull) == 1)
      k_debug_bfly<uint64_t, true><<<grid, th, 0, s>>>(alg, (const uint64_t*)W, (const uint64_t*)Wp, (uint64_t*)X,
                                                        (uint64_t*)Y, n, p, J);
    else
      k_debug_bfly<uint64_t, false><<<grid, th, 0, s>>>(alg, (const uint64_t*)W, (const uint64_t*)Wp, (uint64_t*)X,
                                                         (uint64_t*)Y, n, p, J);
  } else {
    k_debug_bfly<uint32_t, false><<<grid, th, 0, s>>>(alg, (const uint32_t*)W, (const uint32_t*)Wp, (uint32_t*)X,
                                                       (uint32_t*)Y, n, (uint32_t)p, (uint32_t)J);
  }
  return cudaGetLastError();
}

}  // namespace nttb
