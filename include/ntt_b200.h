/*
 * ntt_b200.h -- C ABI of the B200-native batched NTT engine.
 *
 * Implements the hot path of D. Harvey, "Faster arithmetic for number-theoretic
 * transforms" (arXiv:1205.2926): the radix-2 NTT over F_p (Algorithm 1, PAPER.md
 * P:27-46) with the lazy Shoup butterfly (Algorithm 3; operands in
 * [0,2p)) for the forward transform and the lazy inverse butterfly (Algorithm 4,
 * P:142-159; operands in [0,4p)) for the inverse, W' = floor(W beta / p).
 * Citations: P:n = line n of the paper text.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - beta (the machine word) is 2^32 or 2^64.  Data words are uint32_t for
 *   beta = 2^32 and uint64_t for beta = 2^64, in DEVICE memory owned by the
 *   caller, batch x L words, contiguous, transform b at offset b*L, 16-byte
 *   aligned.  The library never allocates in a transform call.
 * - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *   stream) and are stream-ordered.  Argument and plan errors are reported
 *   synchronously; an asynchronous CUDA fault surfaces as NTT_ERR_CUDA from a
 *   later call or a stream synchronisation.  No C++ exception crosses the ABI.
 * - Input ranges are preconditions (not checked in the hot path): forward
 *   needs x < 2p (Alg. 3 input), inverse needs x < 4p (Alg. 4).
 *   ntt_set_range_checks(1) turns on a checking mode in which ntt_forward /
 *   ntt_inverse first scan their input on the stream, synchronise, and return
 *   NTT_ERR_RANGE (data untouched) if any word is out of range.
 * - Outputs are always normalised to [0,p) ("normalise the final NTT
 *   output"); bit-exactness is defined on these canonical values.
 * - A plan is immutable after creation and may be shared by threads and
 *   streams; distinct buffers may be transformed concurrently with one plan.
 */
#ifndef NTT_B200_H
#define NTT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ntt_plan_s* ntt_plan_t;   /* opaque */
typedef struct CUstream_st* ntt_stream_t; /* identical to cudaStream_t */

typedef enum {
  NTT_OK = 0,
  NTT_ERR_ARG = -1,         /* null pointer, misaligned buffer, size overflow, bad flag */
  NTT_ERR_MODULUS = -2,     /* p even, composite, or p >= beta/4 (Alg. 3/4 precondition) */
  NTT_ERR_ROOT = -3,        /* omega^(L/2) != p-1, i.e. omega is not a primitive L-th root */
  NTT_ERR_LENGTH = -4,      /* ell > 28, or 2^ell does not divide p-1 ("p = 1 mod L") */
  NTT_ERR_WORD = -5,        /* log2_beta not in {32, 64} */
  NTT_ERR_CUDA = -6,        /* a CUDA runtime error (see ntt_last_cuda_error) */
  NTT_ERR_NOMEM = -7,       /* device or host allocation failed at plan creation */
  NTT_ERR_UNSUPPORTED = -8, /* valid request this build does not implement */
  NTT_ERR_RANGE = -9        /* range-checking mode: an input word is >= 2p (forward) / 4p (inverse) */
} ntt_status;

/* ntt_pointwise_mul flags */
#define NTT_SCALE_INV_L 1u /* multiply the products by L^{-1} mod p */

/* Plan: validates (p, omega, ell, beta) and precomputes the twiddle tables
 * W = omega^e, W' = floor(W beta / p) ("precomputed and reused").
 *   p         : odd prime, p < beta/4, p = 1 mod 2^ell
 *   omega     : primitive 2^ell-th root of unity mod p; checked as omega^(L/2) = p-1
 *   ell       : transform length L = 2^ell, 0 <= ell <= 28 (ell = 0 is the identity)
 *   log2_beta : 32 or 64 (word size)
 *   device    : CUDA device ordinal that owns the plan's tables
 * On success *out owns device tables on `device` (free with ntt_plan_destroy).
 * On error *out is set to NULL. */
ntt_status ntt_plan_create(ntt_plan_t* out, uint64_t p, uint64_t omega, unsigned ell, unsigned log2_beta, int device);
ntt_status ntt_plan_destroy(ntt_plan_t plan);

/* Same, with the forward butterfly selectable for the paper's own comparison (Table 1,
 * P:212-228): NTT_BFLY_ALG3 = Algorithm 3 (default, the hot
 * path), NTT_BFLY_ALG2 = Algorithm 2 (NTL, canonical operands; forward input must be
 * < p), NTT_BFLY_ALG5 = Algorithm 5 (Montgomery; its forward tables hold one word
 * W' = beta W mod p per entry, half the bytes of the Shoup pairs).  ALG2/ALG5 forward
 * transforms run in every forward kernel family: lengths 2^8..2^28 for beta = 2^64 (on-chip,
 * 2-CTA cluster and four-step column passes incl. the twiddle matrix) and 2^8..2^16 for
 * beta = 2^32; other lengths return NTT_ERR_UNSUPPORTED.  ntt_inverse always uses
 * Algorithm 4 (with the Shoup tables). */
#define NTT_BFLY_ALG2 2u
#define NTT_BFLY_ALG3 3u
#define NTT_BFLY_ALG5 5u
ntt_status ntt_plan_create_ex(ntt_plan_t* out, uint64_t p, uint64_t omega, unsigned ell, unsigned log2_beta,
                              int device, unsigned butterfly);

typedef struct {
  uint64_t p, omega, omega_inv, L_inv; /* L_inv = L^{-1} mod p */
  unsigned ell, log2_beta, word_bytes;
  unsigned n_passes;                   /* kernel passes per transform on one GPU (1 = fused on chip) */
  unsigned pass_log2[4];               /* log2 of each pass's sub-transform length, outermost first */
  int device;
} ntt_plan_info_t;
ntt_status ntt_plan_info(ntt_plan_t plan, ntt_plan_info_t* out);

/* Forward NTT, in place (Algorithm 1, with the Algorithm 3 butterfly):
 * natural-order input in [0,2p) -> output j = b_{rev(j)} (bit-reversed),
 * b_k = sum_i omega^{ik} a_i, normalised to [0,p).
 *   x     : device pointer, batch*L words
 *   batch : number of independent transforms (0 is a no-op) */
ntt_status ntt_forward(ntt_plan_t plan, void* x, size_t batch, ntt_stream_t stream);

/* Inverse NTT, in place: Algorithm 1 run backwards with the Algorithm 4
 * butterfly and twiddles omega^{-k}: bit-reversed input in [0,4p) -> natural
 * order, UNSCALED (ntt_inverse(ntt_forward(a)) = L*a mod p), normalised to [0,p). */
ntt_status ntt_inverse(ntt_plan_t plan, void* x, size_t batch, ntt_stream_t stream);

/* One kernel pass of the plan's schedule (ntt_plan_info_t.pass_log2, outermost first), so a
 * caller can time or interleave the passes of a multi-pass transform.  Running passes
 * 0, 1, ..., n_passes-1 with inverse = 0 is exactly ntt_forward; running n_passes-1, ..., 0
 * with inverse = 1 is exactly ntt_inverse (each in that order, on the same x; other orders
 * are undefined).  Forward pass j < n_passes-1 is a four-step column pass (Algorithm 1's
 * stages re-associated; four-step twiddle fused), the last one the
 * contiguous row pass with the normalisation; the inverse mirrors it.
 * Single-pass plans have one pass (0).  Same buffer contract and input ranges as
 * ntt_forward / ntt_inverse (before the first pass); intermediate buffers hold redundant
 * representatives (< 2p forward, < 4p inverse).  No range-checking mode here.
 * NTT_ERR_ARG for pass >= n_passes or inverse > 1. */
ntt_status ntt_transform_pass(ntt_plan_t plan, void* x, size_t batch, unsigned inverse, unsigned pass,
                              ntt_stream_t stream);

/* Pointwise product for the convolution use: c_k = a_k b_k [* L^{-1}]
 * mod p for k < batch*L.  Inputs in [0,2p); output canonical [0,p).  c may
 * alias a or b. */
ntt_status ntt_pointwise_mul(ntt_plan_t plan, void* c, const void* a, const void* b, size_t batch, unsigned flags,
                             ntt_stream_t stream);

/* Cyclic convolution of `batch` pairs (config C3 building block): a <- a * b
 * (cyclic, length L, mod p).  Runs forward(a), forward(b), pointwise with
 * L^{-1}, inverse(a).  For the 2-CTA cluster sizes (L = 2^16 u32, 2^15 u64) the
 * product is fused into the last round of b's forward, which then only reads b;
 * otherwise b is overwritten by its transform: b's contents are unspecified on
 * return.  Inputs in [0,2p). */
ntt_status ntt_cyclic_convolve(ntt_plan_t plan, void* a, void* b, size_t batch, ntt_stream_t stream);

/* Host-resident data (end-to-end use): ops is a bit set of NTT_OP_FORWARD and
 * NTT_OP_INVERSE (forward first when both).  host_in / host_out hold batch*L words
 * in HOST memory (page-locked for overlap; pageable works but serialises);
 * host_out may equal host_in.  dev_buf is caller-owned DEVICE scratch of
 * dev_buf_bytes >= L*word_bytes: the batch is streamed through it in chunks,
 * each chunk's H2D copy, transform(s) and D2H copy pipelined over the plan's own
 * streams so copies overlap compute.  Ordered after prior work on `stream`;
 * later work on `stream` waits for the whole call.  Thread safety: concurrent
 * calls on one plan are serialised (each enqueues its whole pipeline under the
 * plan's lock, on the plan's pipeline streams); they must use distinct dev_buf. */
#define NTT_OP_FORWARD 1u
#define NTT_OP_INVERSE 2u
ntt_status ntt_execute_host(ntt_plan_t plan, unsigned ops, const void* host_in, void* host_out, size_t batch,
                            void* dev_buf, size_t dev_buf_bytes, ntt_stream_t stream);

/* Copy the plan's forward twiddle table W_e = omega^e, W'_e = floor(W_e beta/p),
 * e < L/2, to host arrays of L/2 words each (test hook; W' check P:85).
 * Returns NTT_ERR_UNSUPPORTED when ell > 20 (tables are factored then). */
ntt_status ntt_plan_twiddles(ntt_plan_t plan, void* host_W, void* host_Wp);

/* Copy a device-resident twiddle table the kernels read to host memory (test hook for A1, P:58,
 * W' p <= W beta < (W'+1) p).  pass indexes ntt_plan_info_t.pass_log2.
 *   kind 0: the per-stage table of that pass's sub-transform (length N = 2^pass_log2[pass], root
 *           omega^(L/N)): stage i (1-based) at entry N - (N >> (i-1)) + (i-1), entries
 *           zeta_i^k, k <= N >> i (the inverse reads the same table, negated entries).
 *   kind 1, 2: the four-step twiddle factors of column pass `pass` (blocks of B = 2^(ell - sum of
 *           the earlier passes) words, root omega_B): table A = omega_B^(e << H), e < B >> H, and
 *           table B = omega_B^e, e < 2^H (H = log2 of B's entry count); a direct table has A = B.
 *   kind 3: the twiddle matrix of column pass `pass`: N rows x S columns, entry (r, c) =
 *           omega_B^(c rev(r)) (NTT_ERR_UNSUPPORTED when that level uses factors).
 * Entries are (W, W') pairs of the plan's word size; Algorithm 5 plans' forward tables hold
 * one word beta W mod p per entry.  *bytes receives the table size; host_out = NULL only
 * queries it; otherwise capacity must be >= *bytes.  Synchronous. */
ntt_status ntt_plan_table(ntt_plan_t plan, unsigned kind, unsigned pass, void* host_out, size_t capacity,
                          size_t* bytes);

/* ---- four-step pass entry points for a transform split over G GPUs (config C5) ----
 * View the length-L transform (L = 2^ell) as an N1 x N2 row-major matrix,
 * N1 = 2^ell1, N2 = L/N1, M[r][c] = x[N2 r + c].  Rank g of G holds the column
 * shard c in [g N2/G, (g+1) N2/G) as an N1 x (N2/G) row-major matrix.
 *   ntt_fourstep_cols: length-N1 NTTs down every local column (root omega^{N2}),
 *     then M[r][c] *= omega^{c rev_{ell1}(r)} (four-step twiddle); output in
 *     [0,2p).  This is stages 1..ell1 of Algorithm 1, re-associated.
 *   ntt_fourstep_rows: input `recv` holds G blocks; block h (h < G) is the
 *     (N1/G) x (N2/G) sub-matrix rows [g N1/G, (g+1) N1/G) x columns
 *     [h N2/G, (h+1) N2/G), row-major, blocks back to back (the all-to-all
 *     receive layout).  Runs length-N2 NTTs on the N1/G full rows (root
 *     omega^{N1}) and writes them, normalised, to `out` (N1/G x N2, row major):
 *     out = flat positions [g L/G, (g+1) L/G) of Algorithm 1's bit-reversed output.
 * Both need ell1 = ell/2 (ell even), G a power of two dividing N1 and N2/16. */
ntt_status ntt_fourstep_cols(ntt_plan_t plan, unsigned ell1, void* x_shard, unsigned rank, unsigned world,
                             ntt_stream_t stream);
ntt_status ntt_fourstep_rows(ntt_plan_t plan, unsigned ell1, const void* recv, void* out, unsigned rank, unsigned world,
                             ntt_stream_t stream);

/* Fused compute + collective (SURVEY.md §8(e) "fused variant"): ntt_fourstep_cols with the
 * all-to-all folded into its last column pass.  Instead of writing the shard in place, the
 * pass stores row r of this rank's N1 x (N2/G) result straight into block `rank` of rank
 * h = r / (N1/G)'s receive buffer, peer_recv[h] (device addresses valid on this device,
 * e.g. symmetric-memory / P2P-mapped buffers of L/G words; peer_recv is a HOST array of
 * `world` <= 8 addresses), over NVLink.  After every rank's call and a cross-rank barrier
 * that orders these stores (stream-ordered, e.g. a symmetric-memory barrier), each
 * rank's buffer holds exactly what all_to_all_single would have delivered, ready for
 * ntt_fourstep_rows.  x_shard is used as scratch by the earlier column passes.
 * NTT_ERR_UNSUPPORTED when the last column pass has no TMA-staged kernel (tiles > 64 KiB). */
ntt_status ntt_fourstep_cols_p2p(ntt_plan_t plan, unsigned ell1, void* x_shard, const uint64_t* peer_recv,
                                 unsigned rank, unsigned world, ntt_stream_t stream);

/* ---- the same split run backwards, and layout helpers ----
 *   ntt_fourstep_rows_inv: `in` holds this rank's N1/G rows of Algorithm 1's
 *     bit-reversed output (flat positions [g L/G, (g+1) L/G), i.e. what
 *     ntt_fourstep_rows wrote), each in [0,4p).  Runs the inverse (Algorithm 1
 *     backwards, Algorithm 4 butterfly) of length N2 on every row (root
 *     omega^{-N1}), natural order out, and writes row r's columns
 *     [h N2/G, (h+1) N2/G) to block h of `send` (G blocks of (N1/G) x (N2/G) words,
 *     row-major, back to back): the all-to-all send layout.  `in` is not modified;
 *     `send` must not alias it.
 *   ntt_fourstep_cols_inv: after the all-to-all, x_shard is this rank's column
 *     shard (N1 x N2/G, row-major).  Multiplies M[r][c] by omega^{-c rev_{ell1}(r)}
 *     then runs inverse NTTs of length N1 down every local column (root
 *     omega^{-N2}); output normalised to [0,p), natural order: the column shard of
 *     L*a when the spectrum was ntt_forward(a) (unscaled, like ntt_inverse).
 * Same size constraints as ntt_fourstep_cols / ntt_fourstep_rows. */
ntt_status ntt_fourstep_rows_inv(ntt_plan_t plan, unsigned ell1, const void* in, void* send, unsigned rank,
                                 unsigned world, ntt_stream_t stream);
ntt_status ntt_fourstep_cols_inv(ntt_plan_t plan, unsigned ell1, void* x_shard, unsigned rank, unsigned world,
                                 ntt_stream_t stream);
/* ntt_fourstep_rows_inv with the all-to-all fused: block h of every row goes straight into
 * block `rank` of rank h's receive buffer peer_recv[h] (peer memory over NVLink; HOST array of
 * `world` <= 8 device addresses) instead of a local send buffer.  After every rank's call and
 * a stream-ordered cross-rank barrier, each receive buffer is the column shard that
 * ntt_fourstep_cols_inv takes. */
ntt_status ntt_fourstep_rows_inv_p2p(ntt_plan_t plan, unsigned ell1, const void* in, const uint64_t* peer_recv,
                                     unsigned rank, unsigned world, ntt_stream_t stream);

/* Block transpose dst[j][i][k] = src[i][j][k] for i < n0, j < n1, k < n2 (words of
 * word_bytes = 4 or 8; device buffers, 16-byte aligned, not aliasing).  The pack /
 * unpack between a contiguous shard (rows of N2 words) and the all-to-all block
 * layout for the contiguous-input / contiguous-output distributed transforms
 * (n0 = N1/G rows, n1 = G blocks, n2 = N2/G words, or n0 and n1 swapped). */
ntt_status ntt_block_transpose(void* dst, const void* src, size_t n0, size_t n1, size_t n2, unsigned word_bytes,
                               ntt_stream_t stream);

/* Three-prime CRT (the RNS use of P:21): for i < n,
 * out[2i] + 2^64 out[2i+1] = the unique x in [0, p0 p1 p2) with x = r_k[i] mod p_k
 * (Garner's mixed-radix form, every constant multiply a Shoup multiply).
 * p0, p1, p2: distinct odd primes < 2^30; r_k: device arrays of n canonical residues
 * (uint32_t, < p_k, not checked); out: device array of 2n uint64_t, 16-byte aligned.
 * With the residues of a three-prime cyclic convolution (config C3) whose true
 * coefficients are < p0 p1 p2, out is the exact integer product. */
ntt_status ntt_crt3(uint64_t* out, const uint32_t* r0, const uint32_t* r1, const uint32_t* r2, size_t n, uint32_t p0,
                    uint32_t p1, uint32_t p2, ntt_stream_t stream);

/* Seeded counter-based generator (test/bench infrastructure; same definition as
 * synth/__init__.py): x[i] = element (start+i) of stream (seed, tensor_id),
 * uniform in [0, bound) by rejection if bound != 0, else uniform in [0, 2^bits).
 * word_bytes = 4 or 8. */
ntt_status ntt_synth_uniform(void* x, size_t count, unsigned word_bytes, uint64_t seed, uint64_t tensor_id,
                             uint64_t start, uint64_t bound, unsigned bits, ntt_stream_t stream);

/* Debug/ablation hook: run one butterfly algorithm of the paper element-wise on
 * device arrays (alg 2 = Algorithm 2, 3 = Algorithm 3, 4 = Algorithm 4,
 * 5 = Algorithm 5 with Wp = beta W mod p and J = p^{-1} mod beta, 31 = the W = 1
 * fast path of Algorithm 3).  All arrays hold n words of the plan's width. */
ntt_status ntt_debug_butterfly(ntt_plan_t plan, int alg, const void* W, const void* Wp, void* X, void* Y, size_t n,
                               ntt_stream_t stream);

/* ALU-roofline calibration (bench infrastructure): launches a register-only loop of
 * Algorithm 3 butterflies -- no memory traffic -- so that the caller can
 * time the sustained butterfly rate of the integer pipes at the live clocks.
 * *n_butterflies receives the number of butterflies the launch performs.
 * sink: device buffer of >= 16 bytes (defeats dead-code elimination). */
ntt_status ntt_calibrate_butterfly(unsigned log2_beta, uint64_t p, uint64_t W, uint64_t Wp, unsigned iters,
                                   void* sink, uint64_t* n_butterflies, ntt_stream_t stream);

/* Range-checking mode (process-wide, default off): when on, ntt_forward / ntt_inverse
 * verify their input against the Algorithm 3 / 4 preconditions (x < 2p, x < 4p; P:114,
 * P:146) with a device scan and a stream synchronisation before transforming, and return
 * NTT_ERR_RANGE without modifying x on a violation.  A debugging aid: it costs a full
 * read of the data and a host round trip per call.  Returns the previous setting. */
unsigned ntt_set_range_checks(unsigned on);

/* Range audit (a debugging build, libntt_b200_audit.so, compiled with
 * -DNTT_RANGE_AUDIT).  In that build every butterfly checks the intervals of its theorem --
 * Theorem 2: Algorithm 3 inputs/outputs in [0,2p) and T = X - Y + 2p in [0,4p);
 * Theorem 3: Algorithm 4 in [0,4p); Theorem 4: Algorithm 5 outputs in
 * [0,2p); Algorithm 2 canonical -- every column pass checks the buffer it leaves in HBM (< 2p
 * forward, < 4p inverse) and every normalised output is checked < p; each violation increments a
 * device counter.
 *   ntt_build_flags: NTT_BUILD_RANGE_AUDIT when this library is the audit build.
 *   ntt_audit_counts: synchronises `device` and returns the violations counted since the last
 *     reset.  NTT_ERR_UNSUPPORTED in the production build.
 *   ntt_audit_reset: synchronises, zeroes the counters; mutate bit 0 drops the "+2p" of Algorithm 3
 *     line 3 in every kernel (the mutation control), which the audit must report; bit 1
 *     turns on race stress: every round of every kernel starts with a per-warp pseudo-random delay,
 *     so a missing barrier around a shared-memory exchange or a staging buffer would show up as wrong
 *     results.  NTT_ERR_UNSUPPORTED in the production build. */
#define NTT_BUILD_RANGE_AUDIT 1u
unsigned ntt_build_flags(void);
ntt_status ntt_audit_counts(int device, uint64_t* violations);
ntt_status ntt_audit_reset(int device, int mutate);

/* Number of kernel launches the last transform entry point on this thread issued. */
unsigned ntt_last_launch_count(void);
const char* ntt_status_str(ntt_status s);
const char* ntt_last_cuda_error(void);
unsigned ntt_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NTT_B200_H */
