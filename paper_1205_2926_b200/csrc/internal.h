// internal.h -- declarations shared by the host plan code (plan.cu) and the
// kernel launchers (ntt_kernels.cu).  Not part of the public ABI.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace nttb {

// A launch-configuration value (SM count, occupancy) cached per CUDA device: computed on the first
// use on each device (cudaFuncSetAttribute and the occupancy queries are per device), read with
// relaxed atomics so concurrent callers are safe (a concurrent first use computes it twice, with
// the same result).  Devices beyond kMaxDevices are not cached.
struct PerDevice {
  static constexpr int kMaxDevices = 64;
  std::atomic<int> v[kMaxDevices];
  template <class F> int get(F compute) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) return compute();
    int x = v[d].load(std::memory_order_relaxed);
    if (!x) {
      x = compute();
      v[d].store(x, std::memory_order_relaxed);
    }
    return x;
  }
};

// Range-audit build (-DNTT_RANGE_AUDIT, modarith.cuh): each kernel translation unit registers the
// host accessors of its device counter; plan.cu sums them (ntt_audit_counts).
struct AuditTU {
  unsigned long long (*read)();
  void (*reset)();
  void (*mutate)(int);
};
void audit_register(const AuditTU& tu);

// Limits of the on-chip (single-pass) transform and of the column pass, as
// log2 of the sub-transform length, per word size.
constexpr int kContigMaxLog64 = 14;  // 2^14 u64 = 128 KiB smem, 512 threads x 32 words
constexpr int kContigMaxLog32 = 15;  // 2^15 u32 = 128 KiB smem, 1024 threads x 32 words
constexpr int kColsMaxLog64 = 9;     // 2^9 rows x 16 u64 columns = 64 KiB tile
constexpr int kColsMaxLog32 = 10;    // 2^10 rows x 32 u32 columns = 128 KiB tile
constexpr int kColsMinLog = 4;
constexpr int kColsTmaMaxLog = 9;    // TMA-staged column pass: N x 128-byte tiles <= 64 KiB, double-buffered
// TMA-staged single-pass kernel (ntt_contig_tma.cu): double-buffered tiles of <= 64 KiB
constexpr int kTmaMinLog = 8;
constexpr int kTmaMaxLog64 = 13;
constexpr int kTmaMaxLog32 = 14;

// Column-pass geometry (four-step pass j of the nested decomposition):
// the data is viewed as blocks of B = N*S words; inside a block, element
// (row r < N, column c < S) sits at r*S + c.  The pass runs length-N NTTs down
// every column and (forward) multiplies element (r, c) by omega_L^{e},
// e = (c * rev_logN(r)) << log_tw_mul, or (inverse) by omega_L^{-e} first.
struct ColsParams {
  uint64_t n_tiles;        // (#blocks) * (S / C)
  uint32_t log_S;          // row stride within a block (words)
  uint32_t log_colgroups;  // log2(S / C)
  uint32_t log_tw_mul;     // log2(L / B): converts block-root exponents to omega_L exponents
  uint32_t ell;            // log2 L
  uint32_t H;              // factored-table split (0 = direct table of L entries)
  uint32_t twiddle;        // 1: apply the four-step twiddle (always 1: k_cols_tma's forward applies it
                           // unconditionally, its last stage's W = 1 butterflies being left lazy for it)
  uint32_t normalize;      // 1: write canonical [0,p) output
  // distributed shard (config C5): global column = col_map(local column)
  uint32_t shard;          // 0: plain; 1: local columns map to global via the fields below
  uint32_t log_local_w;    // log2 of the local matrix width (N2/G)
  uint32_t log_n2;         // log2 N2 (global width)
  uint32_t col0;           // first global column of this shard
  // fused all-to-all (ntt_fourstep_cols_p2p, last column pass only): local row r goes to
  // peer[r >> log_rows_rank] at word (src_rank << (log_rows_rank + log_local_w)) +
  // ((r mod 2^log_rows_rank) << log_local_w) + local column, i.e. block src_rank of that
  // rank's all-to-all receive buffer, written over NVLink instead of in place
  uint32_t p2p;
  uint32_t log_rows_rank;  // log2(N1/G)
  uint32_t src_rank;
  uint64_t peer[8];        // receive buffers of the G <= 8 ranks (device addresses)
  // forward four-step twiddle from the pass's twiddle matrix DevTables::fm (N x S, row-major,
  // M[r][c] = omega_B^{c rev(r)}): one load and one Shoup product per element (k_cols_tma only;
  // other kernels use the factored tables fa/fb, which the plan always keeps)
  uint32_t matrix;
  // tile order: 0 = column groups fastest (tile = block * groups + group); 1 = blocks fastest within
  // runs of 2^log_cgi column groups, so the CTAs in flight share a few column groups' twiddle rows
  uint32_t bmajor;
  uint32_t log_cgi;
  // forward butterfly of the plan (3 = Algorithm 3; 2 / 5 = the ablations F1 / F2, forward only)
  uint32_t bf;
};

struct DevTables {
  const void* sub_fwd;  // omega_N^e, e < N/2, pairs (W, W')
  const void* sub_inv;  // omega_N^{-e}
  const void* fa;       // factored four-step table A (or the direct table when H == 0)
  const void* fb;       // factored four-step table B
  const void* fm = nullptr;  // forward four-step twiddle matrix (ColsParams::matrix)
};

// launchers (return cudaGetLastError of the launch)
cudaError_t launch_contig(int wbytes, int logn, bool inverse, bool normalize, void* x, size_t batch, const void* tw,
                          uint64_t p, cudaStream_t s);
bool tma_supported(int wbytes, int logn);
// bf: forward butterfly 3 (Algorithm 3), 2 (Algorithm 2) or 5 (Algorithm 5) -- F1/F2 ablations
cudaError_t launch_contig_tma(int wbytes, int logn, bool inverse, bool normalize, void* x, size_t batch,
                              const void* tw, uint64_t p, cudaStream_t s, int bf = 3);
// transforms of length 2 * (on-chip max) on 2-CTA clusters (ntt_split2.cu); pw_a != nullptr
// fuses the pointwise product a*b*L^{-1} into the inverse's load (cyclic convolution)
bool split2_supported(int wbytes, int logn);
cudaError_t launch_split2(int wbytes, int logn, bool inverse, void* x, size_t batch, const void* tw, uint64_t p,
                          const void* pw_a, const void* pw_b, uint64_t J, uint64_t K, uint64_t Kp, cudaStream_t s,
                          const void* tw1s = nullptr, int bf = 3);
cudaError_t launch_cols(int wbytes, int logn, bool inverse, void* x, const ColsParams& prm, const DevTables& t,
                        uint64_t p, cudaStream_t s);
// the same pass with TMA-staged, double-buffered tiles (ntt_cols_tma.cu)
bool cols_tma_supported(int wbytes, int logn, const ColsParams& prm, const void* x);
cudaError_t launch_cols_tma(int wbytes, int logn, bool inverse, void* x, const ColsParams& prm, const DevTables& t,
                            uint64_t p, cudaStream_t s);
cudaError_t launch_rows_gather(int wbytes, int logn2, void* out, const void* recv, uint32_t log_rows_local,
                               uint32_t log_world, const void* tw, uint64_t p, cudaStream_t s);
// distributed inverse (F4): inverse row NTTs, natural-order rows scattered into the send blocks
cudaError_t launch_rows_scatter(int wbytes, int logn2, const void* in, void* send, uint32_t log_rows_local,
                                uint32_t log_world, const void* tw_inv, uint64_t p, cudaStream_t s,
                                const uint64_t* peers = nullptr, uint32_t src_rank = 0);
cudaError_t launch_block_transpose(int wbytes, void* dst, const void* src, uint64_t n0, uint64_t n1, uint64_t n2,
                                   cudaStream_t s);
// three-prime CRT (Garner), constants precomputed on the host (plan.cu, ntt_crt3)
struct Crt3Consts {
  uint32_t p0, p1, p2;
  uint32_t c01, c01p;  // p0^{-1} mod p1 and its Shoup W' (beta = 2^32)
  uint32_t c02, c02p;  // p0^{-1} mod p2
  uint32_t c12, c12p;  // p1^{-1} mod p2
  uint32_t K1, K2, K3; // multiples of p1, p2, p2 that keep the Shoup inputs non-negative
  uint64_t p01;        // p0 p1
};
cudaError_t launch_crt3(uint64_t* out, const uint32_t* r0, const uint32_t* r1, const uint32_t* r2, size_t n,
                        const Crt3Consts& k, cudaStream_t s);
cudaError_t launch_pointwise(int wbytes, void* c, const void* a, const void* b, size_t n, uint64_t p, uint64_t J,
                             uint64_t K, uint64_t Kp, cudaStream_t s);
cudaError_t launch_normalize(int wbytes, void* x, size_t n, uint64_t p, int from4p, cudaStream_t s);
cudaError_t launch_check_range(int wbytes, const void* x, size_t n, uint64_t bound, unsigned* flag, cudaStream_t s);
cudaError_t launch_synth(int wbytes, void* x, size_t count, uint64_t seed, uint64_t tensor_id, uint64_t start,
                         uint64_t bound, unsigned bits, cudaStream_t s);
cudaError_t launch_calib(int wbytes, uint64_t p, uint64_t w, uint64_t wp, unsigned iters, void* sink,
                         uint64_t* n_bfly, cudaStream_t s);
cudaError_t launch_debug_bfly(int wbytes, int alg, const void* W, const void* Wp, void* X, void* Y, size_t n,
                              uint64_t p, uint64_t J, cudaStream_t s);

}  // namespace nttb
