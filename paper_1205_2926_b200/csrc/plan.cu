// plan.cu -- host side of the C ABI (include/ntt_b200.h): plan validation,
// twiddle precompute, the pass schedule, and the entry points.
//
// Twiddle precompute ("W and W' ... can be precomputed and reused"):
// W_e = omega^e by repeated multiplication, W'_e = floor(W_e beta / p) by a
// 128-bit division, so W' p <= W beta < (W'+1) p exactly (the bound used in the
// proof of Theorem 1).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "../../include/ntt_b200.h"
#include "internal.h"

using u128 = unsigned __int128;

namespace {

thread_local unsigned t_launches = 0;
thread_local char t_cuda_err[256] = "";

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((u128)a * b % p); }
uint64_t powmod(uint64_t b, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  b %= p;
  for (; e; e >>= 1, b = mulmod(b, b, p))
    if (e & 1) r = mulmod(r, b, p);
  return r;
}

// Deterministic Miller-Rabin for 64-bit n (the first 12 prime bases suffice).
bool is_prime_u64(uint64_t n) {
  if (n < 2) return false;
  static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t q : small) {
    if (n % q == 0) return n == q;
  }
  uint64_t d = n - 1;
  int s = 0;
  while (!(d & 1)) d >>= 1, ++s;
  for (uint64_t a : small) {
    uint64_t x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < s; ++i) {
      x = mulmod(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}

// Table of (root^e, floor(root^e beta / p)) for e < count, interleaved pairs of
// the plan's word width.
std::vector<uint8_t> make_table(uint64_t p, uint64_t root, uint64_t count, unsigned bits, uint64_t scale = 1) {
  const size_t wb = bits / 8;
  std::vector<uint8_t> out(count * 2 * wb);
  uint64_t w = scale % p;  // entries scale * root^e
  for (uint64_t e = 0; e < count; ++e) {
    const uint64_t wp = (uint64_t)(((u128)w << bits) / p);
    if (wb == 8) {
      memcpy(&out[(2 * e) * 8], &w, 8);
      memcpy(&out[(2 * e + 1) * 8], &wp, 8);
    } else {
      const uint32_t w32 = (uint32_t)w, wp32 = (uint32_t)wp;
      memcpy(&out[(2 * e) * 4], &w32, 4);
      memcpy(&out[(2 * e + 1) * 4], &wp32, 4);
    }
    w = mulmod(w, root, p);
  }
  return out;
}

}  // namespace

// Per-stage table of an N = 2^logn point transform with root `root` (rounds.cuh stage_off):
// stage i (1-based) holds zeta_i^k = root^{2^{i-1} k}, k <= m_i = N >> i, at offset
// N - (N >> (i-1)) + (i-1).  The first N/2 entries (stage 1) are root^e, e < N/2.  The extra entry
// k = m_i (= -1) lets the inverse read zeta_i^{-k} = -zeta_i^{m_i - k} from this same table
// (rounds.cuh inv_index), so no inverse table is built.
std::vector<uint8_t> make_stage_table(uint64_t p, uint64_t root, unsigned logn, unsigned bits) {
  const uint64_t N = (uint64_t)1 << logn;
  std::vector<uint8_t> out;
  if (logn == 0) return out;
  out.reserve((N - 1 + logn) * 2 * (bits / 8));
  uint64_t zeta = root;
  for (unsigned i = 1; i <= logn; ++i) {
    std::vector<uint8_t> t = make_table(p, zeta, (N >> i) + 1, bits);
    out.insert(out.end(), t.begin(), t.end());
    zeta = mulmod(zeta, zeta, p);
  }
  return out;
}

// Algorithm 5 form of a table of (W, W') pairs: one word per entry, W'_mont = beta W mod p (P:174,
// "only a single value W' must be stored") -- half the bytes of the Shoup pairs.
std::vector<uint8_t> to_mont_words(const std::vector<uint8_t>& pairs, uint64_t p, unsigned bits) {
  const size_t wb = bits / 8, n = pairs.size() / (2 * wb);
  const uint64_t bmodp = (uint64_t)(((u128)1 << bits) % p);
  std::vector<uint8_t> out(n * wb);
  for (size_t e = 0; e < n; ++e) {
    uint64_t w = 0;
    memcpy(&w, &pairs[2 * e * wb], wb);
    const uint64_t wm = mulmod(w, bmodp, p);
    memcpy(&out[e * wb], &wm, wb);
  }
  return out;
}

// Algorithm 5 variant of the per-stage table (same layout, one word per entry).
std::vector<uint8_t> make_stage_table_mont(uint64_t p, uint64_t root, unsigned logn, unsigned bits) {
  return to_mont_words(make_stage_table(p, root, logn, bits), p, bits);
}

// Four-step twiddle matrix of a column pass: N = 2^logn rows x S = 2^logs columns,
// row-major, entry (r, c) = (W, W') of W = rootB^{c rev_logn(r)} (rootB = omega_B, B = N S).  Built by
// rows on the host's cores: row r is the geometric sequence of rootB^{rev(r)}.
std::vector<uint8_t> make_fourstep_matrix(uint64_t p, uint64_t rootB, unsigned logn, unsigned logs, unsigned bits) {
  const uint64_t N = (uint64_t)1 << logn, S = (uint64_t)1 << logs;
  const size_t wb = bits / 8;
  std::vector<uint8_t> out(N * S * 2 * wb);
  auto rows = [&](uint64_t r0, uint64_t r1) {
    for (uint64_t r = r0; r < r1; ++r) {
      uint64_t rv = 0;
      for (unsigned b = 0; b < logn; ++b) rv |= ((r >> b) & 1) << (logn - 1 - b);
      const uint64_t base = powmod(rootB, rv, p);
      uint64_t w = 1;
      uint8_t* dst = &out[r * S * 2 * wb];
      for (uint64_t c = 0; c < S; ++c) {
        const uint64_t wp = (uint64_t)(((u128)w << bits) / p);
        memcpy(dst + (2 * c) * wb, &w, wb);  // little-endian: the low wb bytes
        memcpy(dst + (2 * c + 1) * wb, &wp, wb);
        w = mulmod(w, base, p);
      }
    }
  };
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (N * S < ((uint64_t)1 << 16)) nt = 1;
  std::vector<std::thread> th;
  for (unsigned i = 0; i < nt; ++i) th.emplace_back(rows, N * i / nt, N * (i + 1) / nt);
  for (auto& t : th) t.join();
  return out;
}

bool tma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NTT_DISABLE_TMA");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

struct ntt_plan_s {
  int device = 0;
  uint64_t p = 0, omega = 0, omega_inv = 0, L_inv = 0, J = 0;
  unsigned ell = 0, bits = 0, wbytes = 0;
  unsigned bfly = 3;  // forward butterfly (NTT_BFLY_ALG*)
  // schedule: log2 sub-lengths of the passes, outermost first
  std::vector<unsigned> passes;
  // device tables
  void* tw_fwd = nullptr;  // single pass: omega^e, e < L/2
  void* tw1s = nullptr;    // cluster sizes: stage-1 entries omega^e K_scale, e < L/2 (fused convolution)
  void* tw_inv = nullptr;  // single pass, read by the inverse (negated entries): tw_fwd itself, or for
                           // Algorithm 5 plans (Montgomery tw_fwd) the Shoup table of omega
  std::vector<void*> sub_fwd, sub_inv;  // per pass sub-length tables (sub_inv[j] == sub_fwd[j])
  std::vector<void*> owned;
  std::map<const void*, size_t> table_bytes;  // size of every uploaded table (ntt_plan_table)
  // lazily built tables for the distributed four-step entry points (guarded by mu)
  std::mutex mu;
  std::map<unsigned, void*> extra_sub;      // log2 N -> omega_N^e per-stage table (forward and inverse)
  // four-step twiddle tables per block level: log2 B -> (table A, table B, H) for omega_B^e, e < B
  struct FsTables { void* fa; void* fb; unsigned H; };
  std::map<unsigned, FsTables> fs_level;
  std::map<unsigned, void*> fs_matrix;  // (bf << 16 | log2 B << 8 | log2 N) -> forward twiddle matrix of that pass
  std::map<unsigned, FsTables> fs_level_bf;  // ablation plans' forward four-step factors (bf << 8 | log2 B)
  // host-buffer executor (ntt_execute_host): pipeline streams and events
  static constexpr int kRing = 8;           // max device buffers in the host pipeline's ring
  static constexpr int kDefaultRing = 4;
  static constexpr int kDefaultChunks = 8;
  std::mutex host_mu;                        // held for a whole ntt_execute_host call (streams, ring events)
  cudaStream_t pipe[3] = {};                 // H2D, compute, D2H
  cudaEvent_t pipe_done[3] = {};
  cudaEvent_t ring_ev[3 * kRing] = {};       // loaded / computed / freed per ring buffer
  cudaEvent_t start_ev = nullptr;
  // pointwise constants: K = beta mod p (plain) / beta L^{-1} mod p (scaled) and K'
  uint64_t K_plain = 0, Kp_plain = 0, K_scale = 0, Kp_scale = 0;
};

namespace {

ntt_status cuda_fail(cudaError_t e) {
  snprintf(t_cuda_err, sizeof t_cuda_err, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return NTT_ERR_CUDA;
}

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

ntt_status upload(ntt_plan_s* pl, const std::vector<uint8_t>& host, void** out) {
  void* d = nullptr;
  const size_t n = host.empty() ? 16 : host.size();
  cudaError_t e = cudaMalloc(&d, n);
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? NTT_ERR_NOMEM : cuda_fail(e);
  pl->owned.push_back(d);
  pl->table_bytes[d] = host.size();
  if (!host.empty()) {
    e = cudaMemcpy(d, host.data(), host.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  *out = d;
  return NTT_OK;
}

void free_plan(ntt_plan_s* pl) {
  if (!pl) return;
  {
    DeviceGuard g(pl->device);
    for (void* d : pl->owned) cudaFree(d);
    for (int i = 0; i < 3; ++i) {
      if (pl->pipe[i]) cudaStreamDestroy(pl->pipe[i]);
      if (pl->pipe_done[i]) cudaEventDestroy(pl->pipe_done[i]);
    }
    for (int i = 0; i < 3 * ntt_plan_s::kRing; ++i)
      if (pl->ring_ev[i]) cudaEventDestroy(pl->ring_ev[i]);
    if (pl->start_ev) cudaEventDestroy(pl->start_ev);
  }
  delete pl;
}

// Pass schedule: one on-chip pass when the
// transform fits; otherwise column passes of <= kColsMax stages followed by one
// contiguous row pass of <= kContigMax stages, stage counts balanced.
constexpr unsigned kRowPassLog64 = 12;  // row pass of >= 3-pass beta = 2^64 schedules

std::vector<unsigned> make_schedule(unsigned ell, unsigned wbytes) {
  // experiment hook: NTT_SCHEDULE="a,b[,c]" (outermost first, must sum to ell) overrides the schedule
  if (const char* e = getenv("NTT_SCHEDULE")) {
    std::vector<unsigned> s;
    unsigned sum = 0;
    for (const char* q = e; *q;) {
      const unsigned v = (unsigned)strtoul(q, const_cast<char**>(&q), 10);
      s.push_back(v);
      sum += v;
      if (*q == ',') ++q;
      else if (*q) break;
    }
    if (sum == ell && !s.empty()) return s;
  }
  const unsigned cmax = wbytes == 8 ? nttb::kContigMaxLog64 : nttb::kContigMaxLog32;
  const unsigned colmax = wbytes == 8 ? nttb::kColsMaxLog64 : nttb::kColsMaxLog32;
  // the contiguous pass reaches 2 * (on-chip max) on a 2-CTA cluster (ntt_split2.cu)
  if (ell <= cmax + 1) return {ell};
  for (unsigned np = 2;; ++np) {
    const unsigned col = std::min(colmax, ell / np);
    const unsigned last = ell - col * (np - 1);
    if (last <= cmax + 1) {
      if (np >= 3 && wbytes == 8 && ell - kRowPassLog64 <= (np - 1) * colmax) {
        // three or more passes: a 2^12 row pass in the TMA-staged kernel and balanced column
        // passes, larger first (measured C5 2^28: [8,8,12] 6.90 ms vs [9,9,10] 7.28 ms)
        const unsigned rest = ell - kRowPassLog64, nc = np - 1;
        std::vector<unsigned> s(np, rest / nc);
        for (unsigned i = 0; i < rest % nc; ++i) s[i] += 1;
        s[np - 1] = kRowPassLog64;
        if (s[nc - 1] >= (unsigned)nttb::kColsMinLog) return s;
      }
      std::vector<unsigned> s(np, col);
      s[np - 1] = last;
      return s;
    }
  }
}

// Per-stage table of omega_N for N = 2^logn, built once per plan (distributed entry points); the
// inverse kernels read the same table (negated entries, rounds.cuh inv_index).
ntt_status sub_table(ntt_plan_s* pl, unsigned logn, void** out, bool inverse = false) {
  (void)inverse;
  std::lock_guard<std::mutex> lk(pl->mu);
  auto& cache = pl->extra_sub;
  auto it = cache.find(logn);
  if (it != cache.end()) { *out = it->second; return NTT_OK; }
  const uint64_t L = (uint64_t)1 << pl->ell, Nn = (uint64_t)1 << logn;
  void* d = nullptr;
  const uint64_t root = powmod(pl->omega, L / Nn, pl->p);
  ntt_status st = upload(pl, make_stage_table(pl->p, root, logn, pl->bits), &d);
  if (st != NTT_OK) return st;
  cache[logn] = d;
  *out = d;
  return NTT_OK;
}

// Four-step twiddles of a column pass whose blocks hold B = 2^lb words: omega_B^e, e < B (omega_B =
// omega^{L/B}), so a pass indexes its own tables with e = c rev(r) instead of e << log2(L/B) into
// one L-level table (whose entries a warp's neighbouring columns then hit far apart: C5's second
// column pass).  Direct table for lb <= 16, else factored omega_B^e = omega_B^{(e >> H) << H} *
// omega_B^{e & (2^H - 1)} (two Shoup multiplies) with H = min(ceil(lb / 2), 10): the low factor
// (indexed by e mod 2^H, scattered across a warp) stays in L1, the high one (indexed by e >> H,
// nearly uniform across neighbouring columns) in L2.  Measured C5: H = 14 6.37 ms, H = 10 6.06 ms.
// bf = 2 / 5 (forward column passes of the ablation plans, F1 / F2): always factored (H >= 1; the
// ablation kernels have no direct-table form), Shoup pairs for Algorithm 2, one-word Montgomery
// factors for Algorithm 5 (its twiddle product is Alg. 5's multiply).
ntt_status fourstep_level_tables(ntt_plan_s* pl, unsigned lb, ntt_plan_s::FsTables* out, unsigned bf = 3) {
  std::lock_guard<std::mutex> lk(pl->mu);
  auto& cache = bf == 3 ? pl->fs_level : pl->fs_level_bf;
  const unsigned key = bf == 3 ? lb : ((bf << 8) | lb);
  auto it = cache.find(key);
  if (it != cache.end()) { *out = it->second; return NTT_OK; }
  auto form = [&](std::vector<uint8_t> pairs) { return bf == 5 ? to_mont_words(pairs, pl->p, pl->bits) : pairs; };
  const uint64_t B = (uint64_t)1 << lb;
  const uint64_t root = powmod(pl->omega, ((uint64_t)1 << pl->ell) >> lb, pl->p);
  ntt_plan_s::FsTables t{nullptr, nullptr, 0};
  ntt_status st;
  // experiment hook: largest level with a direct table.  Measured: direct 2^20-entry tables (16 MiB,
  // L2-resident) instead of two factors make C5 5.5% and a batched 2^20 forward 12% slower.
  static const unsigned direct_max = [] {
    const char* e = getenv("NTT_FS_DIRECT_MAX");
    return e ? (unsigned)atoi(e) : 16u;
  }();
  if (lb <= direct_max && bf == 3) {
    st = upload(pl, make_table(pl->p, root, B, pl->bits), &t.fa);
    t.fb = t.fa;
  } else {
    t.H = std::min((lb + 1) / 2, 10u);
    if (const char* e = getenv("NTT_FOURSTEP_H")) {  // experiment hook
      const unsigned h = (unsigned)atoi(e);
      if (h >= 1 && h < lb) t.H = h;
    }
    st = upload(pl, form(make_table(pl->p, powmod(root, (uint64_t)1 << t.H, pl->p), B >> t.H, pl->bits)), &t.fa);
    if (st == NTT_OK) st = upload(pl, form(make_table(pl->p, root, (uint64_t)1 << t.H, pl->bits)), &t.fb);
  }
  if (st != NTT_OK) return st;
  cache[key] = t;
  *out = t;
  return NTT_OK;
}

// Largest block level with a forward twiddle matrix (env NTT_FS_MATRIX_MAX, default 24: C4's 2^24 level
// takes 256 MiB; C5's 2^28 level would take 4 GiB and keeps the factored tables).
unsigned fs_matrix_max() {
  static const unsigned v = [] {
    const char* e = getenv("NTT_FS_MATRIX_MAX");
    return e ? (unsigned)atoi(e) : 24u;
  }();
  return v;
}

// Forward twiddle matrix of the column pass with blocks of 2^lb words and 2^logn rows (nullptr when
// the level uses a direct table or exceeds fs_matrix_max()).
ntt_status fourstep_matrix(ntt_plan_s* pl, unsigned lb, unsigned logn, void** out, unsigned bf = 3) {
  *out = nullptr;
  static const unsigned direct_max = [] {
    const char* e = getenv("NTT_FS_DIRECT_MAX");
    return e ? (unsigned)atoi(e) : 16u;
  }();
  if (lb <= direct_max || lb > fs_matrix_max() || logn >= lb) return NTT_OK;
  std::lock_guard<std::mutex> lk(pl->mu);
  const unsigned key = (bf << 16) | (lb << 8) | logn;
  auto it = pl->fs_matrix.find(key);
  if (it != pl->fs_matrix.end()) { *out = it->second; return NTT_OK; }
  const uint64_t rootB = powmod(pl->omega, ((uint64_t)1 << pl->ell) >> lb, pl->p);
  void* d = nullptr;
  std::vector<uint8_t> mat = make_fourstep_matrix(pl->p, rootB, logn, lb - logn, pl->bits);
  if (bf == 5) mat = to_mont_words(mat, pl->p, pl->bits);  // Algorithm 5: one word per entry
  ntt_status st = upload(pl, mat, &d);
  if (st != NTT_OK) return st;
  pl->fs_matrix[key] = d;
  *out = d;
  return NTT_OK;
}

unsigned env_uint(const char* name, unsigned dflt) {
  const char* e = getenv(name);
  return e ? (unsigned)atoi(e) : dflt;
}

}  // namespace

extern "C" {

unsigned ntt_abi_version(void) { return 1; }

const char* ntt_status_str(ntt_status s) {
  switch (s) {
    case NTT_OK: return "ok";
    case NTT_ERR_ARG: return "invalid argument";
    case NTT_ERR_MODULUS: return "modulus must be an odd prime p < beta/4";
    case NTT_ERR_ROOT: return "omega is not a primitive 2^ell-th root of unity mod p";
    case NTT_ERR_LENGTH: return "2^ell must divide p-1 and ell <= 28";
    case NTT_ERR_WORD: return "log2_beta must be 32 or 64";
    case NTT_ERR_CUDA: return "CUDA error";
    case NTT_ERR_NOMEM: return "out of memory";
    case NTT_ERR_UNSUPPORTED: return "unsupported";
    case NTT_ERR_RANGE: return "input word out of the butterfly's accepted range";
  }
  return "unknown status";
}

const char* ntt_last_cuda_error(void) { return t_cuda_err; }
unsigned ntt_last_launch_count(void) { return t_launches; }

ntt_status ntt_plan_create(ntt_plan_t* out, uint64_t p, uint64_t omega, unsigned ell, unsigned log2_beta, int device) {
  return ntt_plan_create_ex(out, p, omega, ell, log2_beta, device, NTT_BFLY_ALG3);
}

ntt_status ntt_plan_create_ex(ntt_plan_t* out, uint64_t p, uint64_t omega, unsigned ell, unsigned log2_beta,
                              int device, unsigned butterfly) {
  if (!out) return NTT_ERR_ARG;
  if (butterfly != NTT_BFLY_ALG2 && butterfly != NTT_BFLY_ALG3 && butterfly != NTT_BFLY_ALG5) return NTT_ERR_ARG;
  *out = nullptr;
  if (log2_beta != 32 && log2_beta != 64) return NTT_ERR_WORD;
  // P:114 / P:146: p < beta/4; p odd prime ("word-sized prime", Alg. 5 "p odd")
  const u128 beta = (u128)1 << log2_beta;
  if (p < 3 || !(p & 1) || (u128)p * 4 >= beta || !is_prime_u64(p)) return NTT_ERR_MODULUS;
  if (ell > 28) return NTT_ERR_LENGTH;
  const uint64_t L = (uint64_t)1 << ell;
  if ((p - 1) % L != 0) return NTT_ERR_LENGTH;  // p = 1 mod L
  if (omega >= p) return NTT_ERR_ROOT;
  if (ell == 0) {
    if (omega != 1) return NTT_ERR_ROOT;
  } else if (powmod(omega, L / 2, p) != p - 1) {
    return NTT_ERR_ROOT;  // primitive L-th root <=> omega^(L/2) = -1
  }
  ntt_plan_s* pl = new (std::nothrow) ntt_plan_s();
  if (!pl) return NTT_ERR_NOMEM;
  pl->device = device;
  pl->p = p;
  pl->omega = omega;
  pl->omega_inv = powmod(omega, p - 2, p);
  pl->L_inv = powmod(L % p, p - 2, p);
  pl->ell = ell;
  pl->bits = log2_beta;
  pl->wbytes = log2_beta / 8;
  pl->bfly = butterfly;
  {
    // J = p^{-1} mod beta by Newton iteration
    uint64_t j = p;  // correct to 3 bits for odd p
    for (int i = 0; i < 6; ++i) j *= 2 - p * j;
    pl->J = log2_beta == 32 ? (uint64_t)(uint32_t)j : j;
  }
  {
    const uint64_t bmodp = (uint64_t)(beta % p);
    pl->K_plain = bmodp;
    pl->Kp_plain = (uint64_t)(((u128)bmodp << log2_beta) / p);
    pl->K_scale = mulmod(bmodp, pl->L_inv, p);
    pl->Kp_scale = (uint64_t)(((u128)pl->K_scale << log2_beta) / p);
  }
  pl->passes = make_schedule(ell, pl->wbytes);
  DeviceGuard g(device);
  if (!g.ok) { delete pl; return cuda_fail(cudaGetLastError()); }
  ntt_status st = NTT_OK;
  const unsigned bits = log2_beta;
  if (pl->passes.size() == 1) {
    if ((st = upload(pl, butterfly == NTT_BFLY_ALG5 ? make_stage_table_mont(p, omega, ell, bits)
                                                    : make_stage_table(p, omega, ell, bits),
                     &pl->tw_fwd)) != NTT_OK) {
      free_plan(pl);
      return st;
    }
    // the inverse (Algorithm 4, Shoup pairs) reads the forward table's negated entries
    pl->tw_inv = pl->tw_fwd;
    if (butterfly == NTT_BFLY_ALG5 &&
        (st = upload(pl, make_stage_table(p, omega, ell, bits), &pl->tw_inv)) != NTT_OK) {
      free_plan(pl);
      return st;
    }
    if (nttb::split2_supported((int)pl->wbytes, (int)ell) &&
        (st = upload(pl, make_table(p, omega, (uint64_t)1 << (ell - 1), bits, pl->K_scale), &pl->tw1s)) != NTT_OK) {
      free_plan(pl);
      return st;
    }
  } else {
    for (unsigned n : pl->passes) {
      const uint64_t Nn = (uint64_t)1 << n;
      const uint64_t rootN = powmod(omega, L / Nn, p);
      void *f = nullptr, *fi = nullptr;
      if ((st = upload(pl, make_stage_table(p, rootN, n, bits), &fi)) != NTT_OK ||
          (butterfly == NTT_BFLY_ALG5 && (st = upload(pl, make_stage_table_mont(p, rootN, n, bits), &f)) != NTT_OK)) {
        free_plan(pl);
        return st;
      }
      pl->sub_fwd.push_back(butterfly == NTT_BFLY_ALG5 ? f : fi);
      pl->sub_inv.push_back(fi);  // the inverse reads the Shoup table (negated entries)
    }
    unsigned outer = 0;
    for (size_t j = 0; j + 1 < pl->passes.size(); ++j) {
      ntt_plan_s::FsTables t;
      void* fm = nullptr;
      if ((st = fourstep_level_tables(pl, ell - outer, &t)) != NTT_OK ||
          (butterfly != NTT_BFLY_ALG3 && (st = fourstep_level_tables(pl, ell - outer, &t, butterfly)) != NTT_OK) ||
          (st = fourstep_matrix(pl, ell - outer, pl->passes[j], &fm, butterfly)) != NTT_OK) {
        free_plan(pl);
        return st;
      }
      outer += pl->passes[j];
    }
  }
  *out = pl;
  return NTT_OK;
}

ntt_status ntt_plan_destroy(ntt_plan_t plan) {
  if (!plan) return NTT_ERR_ARG;
  free_plan(plan);
  return NTT_OK;
}

ntt_status ntt_plan_info(ntt_plan_t pl, ntt_plan_info_t* out) {
  if (!pl || !out) return NTT_ERR_ARG;
  memset(out, 0, sizeof *out);
  out->p = pl->p;
  out->omega = pl->omega;
  out->omega_inv = pl->omega_inv;
  out->L_inv = pl->L_inv;
  out->ell = pl->ell;
  out->log2_beta = pl->bits;
  out->word_bytes = pl->wbytes;
  out->n_passes = (unsigned)pl->passes.size();
  for (size_t i = 0; i < pl->passes.size() && i < 4; ++i) out->pass_log2[i] = pl->passes[i];
  out->device = pl->device;
  return NTT_OK;
}

ntt_status ntt_plan_twiddles(ntt_plan_t pl, void* host_W, void* host_Wp) {
  if (!pl || !host_W || !host_Wp) return NTT_ERR_ARG;
  if (pl->ell > 20) return NTT_ERR_UNSUPPORTED;
  const uint64_t half = ((uint64_t)1 << pl->ell) / 2;
  std::vector<uint8_t> t;
  if (pl->tw_fwd) {  // the device table the kernels read (its stage-1 block is omega^e, e < L/2)
    DeviceGuard g(pl->device);
    t.resize(half * 2 * pl->wbytes);
    if (half) {
      cudaError_t e = cudaMemcpy(t.data(), pl->tw_fwd, t.size(), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(e);
    }
  } else {
    t = make_table(pl->p, pl->omega, half, pl->bits);
  }
  const size_t wb = pl->wbytes;
  for (uint64_t e = 0; e < half; ++e) {
    memcpy((uint8_t*)host_W + e * wb, &t[(2 * e) * wb], wb);
    memcpy((uint8_t*)host_Wp + e * wb, &t[(2 * e + 1) * wb], wb);
  }
  return NTT_OK;
}

static bool aligned16(const void* x) { return ((uintptr_t)x & 15) == 0; }

ntt_status ntt_plan_table(ntt_plan_t pl, unsigned kind, unsigned pass, void* host_out, size_t capacity,
                          size_t* bytes) {
  if (!pl || !bytes || kind > 3) return NTT_ERR_ARG;
  *bytes = 0;
  const unsigned np = (unsigned)pl->passes.size();
  if (pass >= np || pl->ell == 0) return NTT_ERR_ARG;
  const void* d = nullptr;
  if (kind == 0) {
    d = np == 1 ? pl->tw_fwd : pl->sub_fwd[pass];
  } else {
    if (pass + 1 >= np) return NTT_ERR_ARG;  // the row pass has no four-step twiddle
    unsigned outer = 0;
    for (unsigned i = 0; i < pass; ++i) outer += pl->passes[i];
    const unsigned lb = pl->ell - outer;
    if (kind == 3) {
      void* fm = nullptr;
      if (ntt_status st = fourstep_matrix(pl, lb, pl->passes[pass], &fm, pl->bfly); st != NTT_OK) return st;
      d = fm;
    } else {
      ntt_plan_s::FsTables t{};
      if (ntt_status st = fourstep_level_tables(pl, lb, &t, pl->bfly); st != NTT_OK) return st;
      d = kind == 1 ? t.fa : t.fb;
    }
  }
  if (!d) return NTT_ERR_UNSUPPORTED;  // e.g. no matrix at this level
  std::lock_guard<std::mutex> lk(pl->mu);
  auto it = pl->table_bytes.find(d);
  if (it == pl->table_bytes.end()) return NTT_ERR_UNSUPPORTED;
  *bytes = it->second;
  if (!host_out) return NTT_OK;  // size query
  if (capacity < it->second) return NTT_ERR_ARG;
  DeviceGuard g(pl->device);
  cudaError_t e = cudaMemcpy(host_out, d, it->second, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

// On-chip transform of `batch` contiguous N-point transforms: the TMA-staged
// kernel where it applies (NTT_DISABLE_TMA=1 forces the register-direct one).
static cudaError_t launch_contig_any(int wbytes, int logn, bool inverse, bool normalize, void* x, size_t batch,
                                     const void* tw, uint64_t p, cudaStream_t s) {
  if (nttb::split2_supported(wbytes, logn)) {  // always normalises; fine for every caller (A5)
    (void)normalize;
    return nttb::launch_split2(wbytes, logn, inverse, x, batch, tw, p, nullptr, nullptr, 0, 0, 0, s);
  }
  if (tma_enabled() && nttb::tma_supported(wbytes, logn))
    return nttb::launch_contig_tma(wbytes, logn, inverse, normalize, x, batch, tw, p, s);
  return nttb::launch_contig(wbytes, logn, inverse, normalize, x, batch, tw, p, s);
}

// Four-step column pass: the TMA-staged kernel where it applies (NTT_DISABLE_TMA=1
// forces the register-direct one).
static cudaError_t launch_cols_any(int wbytes, int logn, bool inverse, void* x, const nttb::ColsParams& prm,
                                   const nttb::DevTables& t, uint64_t p, cudaStream_t s) {
  if (tma_enabled() && nttb::cols_tma_supported(wbytes, logn, prm, x))
    return nttb::launch_cols_tma(wbytes, logn, inverse, x, prm, t, p, s);
  return nttb::launch_cols(wbytes, logn, inverse, x, prm, t, p, s);
}

static std::atomic<unsigned> g_range_checks{0};

#ifdef NTT_RANGE_AUDIT
// Range-audit build: every translation unit with kernels registers its counter accessors
// (modarith.cuh); a function-local static so registration from other TUs' static initialisers is
// safe regardless of initialisation order.
static std::vector<nttb::AuditTU>& audit_tus() {
  static std::vector<nttb::AuditTU> v;
  return v;
}
}  // extern "C"
void nttb::audit_register(const nttb::AuditTU& tu) { audit_tus().push_back(tu); }
extern "C" {
#endif

// Range-checking mode: scan x for words >= bound; NTT_ERR_RANGE on a violation.
static ntt_status check_range(ntt_plan_t pl, const void* x, size_t n, uint64_t bound, cudaStream_t s) {
  unsigned* flag = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&flag, sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, sizeof(unsigned), s);
  if (e == cudaSuccess) e = nttb::launch_check_range((int)pl->wbytes, x, n, bound, flag, s);
  unsigned h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, flag, sizeof h, cudaMemcpyDeviceToHost, s);
  if (flag) cudaFreeAsync(flag, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e);
  return h ? NTT_ERR_RANGE : NTT_OK;
}

// One kernel pass of the schedule (no argument checks; callers validate).  Pass j indexes the
// schedule outermost first: forward runs j = 0 .. np-1 (column passes, then the contiguous row pass,
// which normalises), the inverse j = np-1 .. 0 (row pass first, the j = 0 column pass normalises).
static cudaError_t run_pass(ntt_plan_t pl, void* x, size_t batch, cudaStream_t s, bool inverse, unsigned j) {
  const uint64_t L = (uint64_t)1 << pl->ell;
  const unsigned np = (unsigned)pl->passes.size();
  if (pl->ell == 0)  // identity; only the normalisation remains
    return nttb::launch_normalize(pl->wbytes, x, batch, pl->p, inverse ? 1 : 0, s);
  const bool abl = pl->bfly != NTT_BFLY_ALG3 && !inverse;  // F1/F2 ablation forward: BF-templated kernels only
  if (abl && (np == 1 || j + 1 == np)) {
    const unsigned n = np == 1 ? pl->ell : pl->passes[np - 1];
    const size_t rows = np == 1 ? batch : batch * (L >> n);
    const void* tw = np == 1 ? pl->tw_fwd : pl->sub_fwd[np - 1];
    if (nttb::split2_supported(pl->wbytes, (int)n))
      return nttb::launch_split2(pl->wbytes, (int)n, false, x, rows, tw, pl->p, nullptr, nullptr, 0, 0, 0, s,
                                 nullptr, (int)pl->bfly);
    if (!nttb::tma_supported(pl->wbytes, (int)n)) return cudaErrorNotSupported;
    return nttb::launch_contig_tma(pl->wbytes, (int)n, false, true, x, rows, tw, pl->p, s, (int)pl->bfly);
  }
  if (np == 1)
    return launch_contig_any(pl->wbytes, (int)pl->ell, inverse, true, x, batch, inverse ? pl->tw_inv : pl->tw_fwd,
                             pl->p, s);
  if (j + 1 == np) {  // contiguous row pass
    const size_t rows = batch * (L >> pl->passes[np - 1]);
    return launch_contig_any(pl->wbytes, (int)pl->passes[np - 1], inverse, !inverse, x, rows,
                             inverse ? pl->sub_inv[np - 1] : pl->sub_fwd[np - 1], pl->p, s);
  }
  // column pass j of the nested four-step
  const unsigned C = 128 / pl->wbytes;
  nttb::ColsParams prm{};
  unsigned outer = 0;
  for (unsigned i = 0; i < j; ++i) outer += pl->passes[i];
  const unsigned logB = pl->ell - outer, logN = pl->passes[j], logS = logB - logN;
  unsigned logC = 0;
  while ((1u << logC) < C) ++logC;
  prm.log_S = logS;
  prm.log_colgroups = logS - logC;
  prm.n_tiles = ((uint64_t)batch << outer) << prm.log_colgroups;
  // per-level tables: exponent e = c rev(r) of omega_B, B = 2^logB (log_tw_mul = 0, ell = logB)
  prm.log_tw_mul = 0;
  prm.ell = logB;
  prm.twiddle = 1;
  prm.normalize = (inverse && j == 0) ? 1 : 0;
  ntt_plan_s::FsTables t{};
  if (fourstep_level_tables(pl, prm.ell, &t) != NTT_OK)  // built at plan creation: a cache hit
    return cudaErrorMemoryAllocation;
  if (abl && fourstep_level_tables(pl, prm.ell, &t, pl->bfly) != NTT_OK) return cudaErrorMemoryAllocation;
  prm.H = t.H;
  prm.bf = inverse ? 3 : pl->bfly;
  nttb::DevTables tb{pl->sub_fwd[j], pl->sub_inv[j], t.fa, t.fb};
  if (!inverse) {
    void* fm = nullptr;
    if (fourstep_matrix(pl, logB, logN, &fm, pl->bfly) != NTT_OK) return cudaErrorMemoryAllocation;  // cache hit
    if (fm) {
      tb.fm = fm;
      prm.matrix = 1;
      // blocks fastest within runs of 2^log_cgi column groups: the CTAs in flight read the same few
      // column groups' matrix rows (L2-resident) for every transform of the batch
      static const unsigned bmajor = env_uint("NTT_COLS_BMAJOR", 1), cgi = env_uint("NTT_COLS_CGI", 2);
      const unsigned groups_log = prm.log_colgroups;
      prm.bmajor = bmajor;
      prm.log_cgi = std::min(cgi, groups_log);
    }
  }
  if (abl) {  // the ablation butterflies exist in the TMA-staged column kernel only (no fallback)
    if (!nttb::cols_tma_supported(pl->wbytes, (int)pl->passes[j], prm, x)) return cudaErrorNotSupported;
    return nttb::launch_cols_tma(pl->wbytes, (int)pl->passes[j], false, x, prm, tb, pl->p, s);
  }
  return launch_cols_any(pl->wbytes, (int)pl->passes[j], inverse, x, prm, tb, pl->p, s);
}

static ntt_status check_transform_args(ntt_plan_t pl, void* x, size_t batch) {
  if (!pl || (!x && batch) || (x && !aligned16(x))) return NTT_ERR_ARG;
  const uint64_t L = (uint64_t)1 << pl->ell;
  if (batch > (SIZE_MAX / pl->wbytes) / L) return NTT_ERR_ARG;
  return NTT_OK;
}

static ntt_status run_transform(ntt_plan_t pl, void* x, size_t batch, cudaStream_t s, bool inverse) {
  t_launches = 0;
  if (ntt_status st = check_transform_args(pl, x, batch); st != NTT_OK) return st;
  if (!batch) return NTT_OK;
  const uint64_t L = (uint64_t)1 << pl->ell;
  DeviceGuard g(pl->device);
  if (!g.ok) return cuda_fail(cudaGetLastError());
  if (g_range_checks.load(std::memory_order_relaxed)) {
    // Alg. 3 takes [0,2p) (Alg. 2 plans canonical [0,p)), Alg. 4 [0,4p)
    const uint64_t bound = inverse ? 4 * pl->p : (pl->bfly == NTT_BFLY_ALG2 ? pl->p : 2 * pl->p);
    ntt_status st = check_range(pl, x, batch * L, bound, s);
    if (st != NTT_OK) return st;
  }
  const unsigned np = pl->ell == 0 ? 1u : (unsigned)pl->passes.size();
  cudaError_t e = cudaSuccess;
  for (unsigned k = 0; k < np && e == cudaSuccess; ++k) {
    e = run_pass(pl, x, batch, s, inverse, inverse ? np - 1 - k : k);
    ++t_launches;
  }
  if (e == cudaErrorNotSupported) {  // a size the ablation kernels do not cover (before any launch)
    cudaGetLastError();
    return NTT_ERR_UNSUPPORTED;
  }
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

// Host-buffer pipeline: three role streams -- H2D copies, transforms, D2H copies -- over a ring of
// NB device buffers carved from dev_buf.  Chunk k uses buffer k mod NB; its H2D waits until the
// D2H of chunk k - NB has drained that buffer, so both copy directions stay busy back to back
// (C2 end to end: 3.33 ms vs 3.46 ms for per-chunk streams doing all three stages; the copies
// alone pipeline in 3.06 ms, tools/e2e_probe.py).
ntt_status ntt_execute_host(ntt_plan_t pl, unsigned ops, const void* host_in, void* host_out, size_t batch,
                            void* dev_buf, size_t dev_buf_bytes, ntt_stream_t stream) {
  if (!pl || !ops || (ops & ~(NTT_OP_FORWARD | NTT_OP_INVERSE))) return NTT_ERR_ARG;
  if (!batch) { t_launches = 0; return NTT_OK; }
  if (!host_in || !host_out || !dev_buf || !aligned16(dev_buf)) return NTT_ERR_ARG;
  const uint64_t L = (uint64_t)1 << pl->ell;
  const size_t tbytes = (size_t)L * pl->wbytes;
  if (batch > SIZE_MAX / tbytes || dev_buf_bytes < tbytes) return NTT_ERR_ARG;
  DeviceGuard g(pl->device);
  using P = ntt_plan_s;
  // the pipeline streams and the ring events are per plan: one call enqueues at a time, so a
  // concurrent call on another thread waits (its copies would otherwise interleave with this
  // call's event records); the work itself is ordered through the shared pipeline streams
  std::lock_guard<std::mutex> call_lk(pl->host_mu);
  {
    std::lock_guard<std::mutex> lk(pl->mu);
    if (!pl->start_ev) {
      for (int i = 0; i < 3; ++i) {
        cudaError_t e = cudaStreamCreateWithFlags(&pl->pipe[i], cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(e);
      }
      for (int i = 0; i < 3 * P::kRing; ++i) {
        cudaError_t e = cudaEventCreateWithFlags(&pl->ring_ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e);
      }
      for (int i = 0; i < 3; ++i) {
        cudaError_t e = cudaEventCreateWithFlags(&pl->pipe_done[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e);
      }
      cudaError_t e = cudaEventCreateWithFlags(&pl->start_ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e);
    }
  }
  static int env_nb = -1, env_chunks = -1;
  if (env_nb < 0) {
    const char* e1 = getenv("NTT_HOST_RING");
    const char* e2 = getenv("NTT_HOST_CHUNKS");
    env_nb = (e1 && atoi(e1) > 0) ? std::min(atoi(e1), P::kRing) : P::kDefaultRing;
    env_chunks = (e2 && atoi(e2) > 0) ? atoi(e2) : P::kDefaultChunks;
  }
  // ring of NB buffers of `chunk` transforms each; aim for env_chunks chunks, none below ~1 MiB
  const int nb = (int)std::max<size_t>(1, std::min<size_t>((size_t)env_nb, dev_buf_bytes / tbytes));
  const size_t per_buf = dev_buf_bytes / nb / tbytes;
  const size_t min_chunk = std::max<size_t>(1, ((size_t)1 << 20) / tbytes);
  const size_t want = std::max(min_chunk, (batch + (size_t)env_chunks - 1) / (size_t)env_chunks);
  const size_t chunk = std::max<size_t>(1, std::min(per_buf, want));
  cudaStream_t user = (cudaStream_t)stream;
  cudaStream_t h2d = pl->pipe[0], comp = pl->pipe[1], d2h = pl->pipe[2];
  cudaEvent_t* loaded = pl->ring_ev;
  cudaEvent_t* computed = pl->ring_ev + P::kRing;
  cudaEvent_t* freed = pl->ring_ev + 2 * P::kRing;
  cudaError_t e = cudaEventRecord(pl->start_ev, user);
  for (int i = 0; e == cudaSuccess && i < 3; ++i) e = cudaStreamWaitEvent(pl->pipe[i], pl->start_ev, 0);
  if (e != cudaSuccess) return cuda_fail(e);
  unsigned launches = 0;
  size_t k = 0;
  for (size_t b0 = 0; b0 < batch; b0 += chunk, ++k) {
    const size_t n = std::min(chunk, batch - b0);
    const int b = (int)(k % (size_t)nb);
    void* d = (uint8_t*)dev_buf + (size_t)b * per_buf * tbytes;
    if (k >= (size_t)nb && (e = cudaStreamWaitEvent(h2d, freed[b], 0)) != cudaSuccess) return cuda_fail(e);
    e = cudaMemcpyAsync(d, (const uint8_t*)host_in + b0 * tbytes, n * tbytes, cudaMemcpyHostToDevice, h2d);
    if (e == cudaSuccess) e = cudaEventRecord(loaded[b], h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(comp, loaded[b], 0);
    if (e != cudaSuccess) return cuda_fail(e);
    if (ops & NTT_OP_FORWARD) {
      ntt_status st = run_transform(pl, d, n, comp, false);
      launches += t_launches;
      if (st != NTT_OK) return st;
    }
    if (ops & NTT_OP_INVERSE) {
      ntt_status st = run_transform(pl, d, n, comp, true);
      launches += t_launches;
      if (st != NTT_OK) return st;
    }
    e = cudaEventRecord(computed[b], comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(d2h, computed[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync((uint8_t*)host_out + b0 * tbytes, d, n * tbytes, cudaMemcpyDeviceToHost, d2h);
    if (e == cudaSuccess) e = cudaEventRecord(freed[b], d2h);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  for (int i = 0; e == cudaSuccess && i < 3; ++i) {
    e = cudaEventRecord(pl->pipe_done[i], pl->pipe[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(user, pl->pipe_done[i], 0);
  }
  t_launches = launches;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

unsigned ntt_set_range_checks(unsigned on) { return g_range_checks.exchange(on ? 1u : 0u); }

unsigned ntt_build_flags(void) {
#ifdef NTT_RANGE_AUDIT
  return NTT_BUILD_RANGE_AUDIT;
#else
  return 0;
#endif
}

ntt_status ntt_audit_counts(int device, uint64_t* violations) {
  if (!violations) return NTT_ERR_ARG;
  *violations = 0;
#ifdef NTT_RANGE_AUDIT
  DeviceGuard g(device);
  if (!g.ok) return cuda_fail(cudaGetLastError());
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e);
  for (const auto& tu : audit_tus()) *violations += tu.read();
  return NTT_OK;
#else
  (void)device;
  return NTT_ERR_UNSUPPORTED;
#endif
}

ntt_status ntt_audit_reset(int device, int mutate) {
#ifdef NTT_RANGE_AUDIT
  DeviceGuard g(device);
  if (!g.ok) return cuda_fail(cudaGetLastError());
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e);
  for (const auto& tu : audit_tus()) {
    tu.reset();
    tu.mutate(mutate & 3);  // bit 0: mutation control, bit 1: race stress
  }
  return NTT_OK;
#else
  (void)device;
  (void)mutate;
  return NTT_ERR_UNSUPPORTED;
#endif
}

ntt_status ntt_forward(ntt_plan_t plan, void* x, size_t batch, ntt_stream_t stream) {
  return run_transform(plan, x, batch, (cudaStream_t)stream, false);
}

ntt_status ntt_inverse(ntt_plan_t plan, void* x, size_t batch, ntt_stream_t stream) {
  return run_transform(plan, x, batch, (cudaStream_t)stream, true);
}

ntt_status ntt_transform_pass(ntt_plan_t pl, void* x, size_t batch, unsigned inverse, unsigned pass,
                              ntt_stream_t stream) {
  t_launches = 0;
  if (ntt_status st = check_transform_args(pl, x, batch); st != NTT_OK) return st;
  if (inverse > 1 || pass >= pl->passes.size()) return NTT_ERR_ARG;
  if (!batch) return NTT_OK;
  DeviceGuard g(pl->device);
  if (!g.ok) return cuda_fail(cudaGetLastError());
  cudaError_t e = run_pass(pl, x, batch, (cudaStream_t)stream, inverse != 0, pass);
  ++t_launches;
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    return NTT_ERR_UNSUPPORTED;
  }
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

ntt_status ntt_pointwise_mul(ntt_plan_t pl, void* c, const void* a, const void* b, size_t batch, unsigned flags,
                             ntt_stream_t stream) {
  t_launches = 0;
  if (!pl || flags > NTT_SCALE_INV_L) return NTT_ERR_ARG;
  if (!batch) return NTT_OK;
  if (!c || !a || !b) return NTT_ERR_ARG;
  const uint64_t L = (uint64_t)1 << pl->ell;
  if (batch > (SIZE_MAX / pl->wbytes) / L) return NTT_ERR_ARG;
  DeviceGuard g(pl->device);
  const bool sc = flags & NTT_SCALE_INV_L;
  cudaError_t e = nttb::launch_pointwise(pl->wbytes, c, a, b, batch * L, pl->p, pl->J, sc ? pl->K_scale : pl->K_plain,
                                         sc ? pl->Kp_scale : pl->Kp_plain, (cudaStream_t)stream);
  ++t_launches;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

ntt_status ntt_cyclic_convolve(ntt_plan_t pl, void* a, void* b, size_t batch, ntt_stream_t stream) {
  if (!pl) return NTT_ERR_ARG;
  unsigned total = 0;
  ntt_status st = ntt_forward(pl, a, batch, stream);
  total += t_launches;
  static const bool inv_pw = getenv("NTT_CONV_INV_PW") != nullptr;  // A/B hook: product fused into the inverse
  if (st == NTT_OK && batch && !inv_pw && pl->passes.size() == 1 && pl->bfly == NTT_BFLY_ALG3 &&
      nttb::split2_supported((int)pl->wbytes, (int)pl->ell) && aligned16(b)) {
    // forward of b with the pointwise product (x L^{-1}) fused into its last round, written over
    // a-hat; then the plain inverse of a.  b is only read.
    DeviceGuard g(pl->device);
    cudaError_t e = nttb::launch_split2((int)pl->wbytes, (int)pl->ell, false, b, batch, pl->tw_fwd, pl->p, a, b, pl->J,
                                        pl->K_scale, pl->Kp_scale, (cudaStream_t)stream, pl->tw1s);
    if (e != cudaErrorNotSupported) {
      if (e != cudaSuccess) return cuda_fail(e);
      st = ntt_inverse(pl, a, batch, stream);
      t_launches += total + 1;
      return st;
    }
    cudaGetLastError();
  }
  if (st == NTT_OK) { st = ntt_forward(pl, b, batch, stream); total += t_launches; }
  if (st == NTT_OK && pl->passes.size() == 1 && nttb::split2_supported((int)pl->wbytes, (int)pl->ell)) {
    // pointwise product (x L^{-1}) fused into the inverse's load
    DeviceGuard g(pl->device);
    cudaError_t e = nttb::launch_split2((int)pl->wbytes, (int)pl->ell, true, a, batch, pl->tw_inv, pl->p, a, b, pl->J,
                                        pl->K_scale, pl->Kp_scale, (cudaStream_t)stream);
    t_launches = total + 1;
    return e == cudaSuccess ? NTT_OK : cuda_fail(e);
  }
  if (st == NTT_OK) { st = ntt_pointwise_mul(pl, a, a, b, batch, NTT_SCALE_INV_L, stream); total += t_launches; }
  if (st == NTT_OK) { st = ntt_inverse(pl, a, batch, stream); total += t_launches; }
  t_launches = total;
  return st;
}

// Column half of the distributed four-step (forward: column NTTs then the twiddle;
// inverse: the inverse twiddle then inverse column NTTs, passes in reverse order).
static ntt_status fourstep_cols_impl(ntt_plan_t pl, unsigned ell1, void* x, unsigned rank, unsigned world,
                                     ntt_stream_t stream, bool inverse, const uint64_t* peers = nullptr) {
  t_launches = 0;
  if (!pl || !x || !aligned16(x) || world == 0 || (world & (world - 1)) || rank >= world) return NTT_ERR_ARG;
  if (ell1 == 0 || ell1 >= pl->ell) return NTT_ERR_ARG;
  const unsigned ell2 = pl->ell - ell1;
  unsigned lw = 0;
  while ((1u << lw) < world) ++lw;
  const unsigned C = 128 / pl->wbytes;
  if (lw > ell1 || (ell2 < lw) || ((1u << (ell2 - lw)) < C)) return NTT_ERR_ARG;
  const unsigned colmax = pl->wbytes == 8 ? nttb::kColsMaxLog64 : nttb::kColsMaxLog32;
  // split the length-N1 column DFT into column passes of <= colmax stages
  const unsigned nc = (ell1 + colmax - 1) / colmax;
  std::vector<unsigned> cp(nc, ell1 / nc);
  for (unsigned i = 0; i < ell1 % nc; ++i) cp[nc - 1 - i] += 1;
  const unsigned log_wl = ell2 - lw;  // local width N2/G
  unsigned logC = 0;
  while ((1u << logC) < C) ++logC;
  DeviceGuard g(pl->device);
  std::vector<nttb::ColsParams> prms(nc);
  std::vector<ntt_plan_s::FsTables> tabs(nc);
  unsigned outer = 0;
  for (unsigned j = 0; j < nc; ++j) {
    const unsigned logN = cp[j];
    // local block = rows of this sub-level x local width
    const unsigned logS = (ell1 - outer - logN) + log_wl;
    nttb::ColsParams& prm = prms[j];
    prm = nttb::ColsParams{};
    prm.log_S = logS;
    prm.log_colgroups = logS - logC;
    prm.n_tiles = ((uint64_t)1 << outer) << prm.log_colgroups;
    // per-level tables of omega_B, B = 2^(ell - outer): e = c rev(r) (c: global column of the block)
    prm.log_tw_mul = 0;
    prm.ell = pl->ell - outer;
    if (ntt_status st = fourstep_level_tables(pl, prm.ell, &tabs[j]); st != NTT_OK) return st;
    prm.H = tabs[j].H;
    prm.twiddle = 1;
    prm.normalize = (inverse && j == 0) ? 1 : 0;  // the inverse's last pass writes canonical values
    prm.shard = 1;
    prm.log_local_w = log_wl;
    prm.log_n2 = ell2;
    prm.col0 = rank << log_wl;
    outer += logN;
  }
  if (peers) {  // fused all-to-all: the last column pass scatters into the peers' receive buffers
    if (world > 8) return NTT_ERR_UNSUPPORTED;
    nttb::ColsParams& last = prms[nc - 1];
    if (!tma_enabled() || !nttb::cols_tma_supported((int)pl->wbytes, (int)cp[nc - 1], last, x))
      return NTT_ERR_UNSUPPORTED;
    for (unsigned h = 0; h < world; ++h)
      if (!peers[h] || (peers[h] & 15)) return NTT_ERR_ARG;
    last.p2p = 1;
    last.log_rows_rank = ell1 - lw;
    last.src_rank = rank;
    for (unsigned h = 0; h < world; ++h) last.peer[h] = peers[h];
  }
  cudaError_t e = cudaSuccess;
  for (unsigned jj = 0; jj < nc && e == cudaSuccess; ++jj) {
    const unsigned j = inverse ? nc - 1 - jj : jj;
    void* sub = nullptr;
    ntt_status st = sub_table(pl, cp[j], &sub, inverse);
    if (st != NTT_OK) return st;
    nttb::DevTables t{sub, sub, tabs[j].fa, tabs[j].fb};
    e = prms[j].p2p ? nttb::launch_cols_tma(pl->wbytes, (int)cp[j], inverse, x, prms[j], t, pl->p, (cudaStream_t)stream)
                    : launch_cols_any(pl->wbytes, (int)cp[j], inverse, x, prms[j], t, pl->p, (cudaStream_t)stream);
    ++t_launches;
  }
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

ntt_status ntt_fourstep_cols(ntt_plan_t pl, unsigned ell1, void* x, unsigned rank, unsigned world,
                             ntt_stream_t stream) {
  return fourstep_cols_impl(pl, ell1, x, rank, world, stream, false);
}

ntt_status ntt_fourstep_cols_inv(ntt_plan_t pl, unsigned ell1, void* x, unsigned rank, unsigned world,
                                 ntt_stream_t stream) {
  return fourstep_cols_impl(pl, ell1, x, rank, world, stream, true);
}

ntt_status ntt_fourstep_cols_p2p(ntt_plan_t pl, unsigned ell1, void* x, const uint64_t* peer_recv, unsigned rank,
                                 unsigned world, ntt_stream_t stream) {
  if (!peer_recv) { t_launches = 0; return NTT_ERR_ARG; }
  return fourstep_cols_impl(pl, ell1, x, rank, world, stream, false, peer_recv);
}

ntt_status ntt_fourstep_rows(ntt_plan_t pl, unsigned ell1, const void* recv, void* out, unsigned rank, unsigned world,
                             ntt_stream_t stream) {
  t_launches = 0;
  if (!pl || !recv || !out || !aligned16(out) || world == 0 || (world & (world - 1)) || rank >= world)
    return NTT_ERR_ARG;
  if (ell1 == 0 || ell1 >= pl->ell) return NTT_ERR_ARG;
  const unsigned ell2 = pl->ell - ell1;
  const unsigned cmax = pl->wbytes == 8 ? nttb::kContigMaxLog64 : nttb::kContigMaxLog32;
  if (ell2 > cmax || ell2 < 5) return NTT_ERR_UNSUPPORTED;
  unsigned lw = 0;
  while ((1u << lw) < world) ++lw;
  if (lw > ell1 || lw > ell2) return NTT_ERR_ARG;
  DeviceGuard g(pl->device);
  void* subf = nullptr;
  ntt_status st = sub_table(pl, ell2, &subf);
  if (st != NTT_OK) return st;
  cudaError_t e = nttb::launch_rows_gather(pl->wbytes, (int)ell2, out, recv, ell1 - lw, lw, subf, pl->p,
                                           (cudaStream_t)stream);
  ++t_launches;
  (void)rank;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

static ntt_status fourstep_rows_inv_impl(ntt_plan_t pl, unsigned ell1, const void* in, void* send, unsigned rank,
                                         unsigned world, ntt_stream_t stream, const uint64_t* peers) {
  t_launches = 0;
  if (!pl || !in || (!send && !peers) || !aligned16(in) || in == send || world == 0 || (world & (world - 1)) ||
      rank >= world)
    return NTT_ERR_ARG;
  if (peers) {
    if (world > 8) return NTT_ERR_UNSUPPORTED;
    for (unsigned h = 0; h < world; ++h)
      if (!peers[h] || (peers[h] & 15)) return NTT_ERR_ARG;
  }
  if (ell1 == 0 || ell1 >= pl->ell) return NTT_ERR_ARG;
  const unsigned ell2 = pl->ell - ell1;
  const unsigned cmax = pl->wbytes == 8 ? nttb::kContigMaxLog64 : nttb::kContigMaxLog32;
  if (ell2 > cmax || ell2 < 5) return NTT_ERR_UNSUPPORTED;
  unsigned lw = 0;
  while ((1u << lw) < world) ++lw;
  if (lw > ell1 || lw > ell2) return NTT_ERR_ARG;
  DeviceGuard g(pl->device);
  void* subi = nullptr;
  ntt_status st = sub_table(pl, ell2, &subi, true);
  if (st != NTT_OK) return st;
  cudaError_t e = nttb::launch_rows_scatter(pl->wbytes, (int)ell2, in, send, ell1 - lw, lw, subi, pl->p,
                                            (cudaStream_t)stream, peers, rank);
  ++t_launches;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

ntt_status ntt_fourstep_rows_inv(ntt_plan_t pl, unsigned ell1, const void* in, void* send, unsigned rank,
                                 unsigned world, ntt_stream_t stream) {
  return fourstep_rows_inv_impl(pl, ell1, in, send, rank, world, stream, nullptr);
}

ntt_status ntt_fourstep_rows_inv_p2p(ntt_plan_t pl, unsigned ell1, const void* in, const uint64_t* peer_recv,
                                     unsigned rank, unsigned world, ntt_stream_t stream) {
  if (!peer_recv) { t_launches = 0; return NTT_ERR_ARG; }
  return fourstep_rows_inv_impl(pl, ell1, in, nullptr, rank, world, stream, peer_recv);
}

ntt_status ntt_block_transpose(void* dst, const void* src, size_t n0, size_t n1, size_t n2, unsigned word_bytes,
                               ntt_stream_t stream) {
  t_launches = 0;
  if ((word_bytes != 4 && word_bytes != 8)) return NTT_ERR_ARG;
  if (!n0 || !n1 || !n2) return NTT_OK;
  if (!dst || !src || dst == src || !aligned16(dst) || !aligned16(src)) return NTT_ERR_ARG;
  if (n0 > SIZE_MAX / n1 || n0 * n1 > SIZE_MAX / n2 || n0 * n1 * n2 > SIZE_MAX / word_bytes) return NTT_ERR_ARG;
  cudaError_t e = nttb::launch_block_transpose((int)word_bytes, dst, src, n0, n1, n2, (cudaStream_t)stream);
  ++t_launches;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

ntt_status ntt_crt3(uint64_t* out, const uint32_t* r0, const uint32_t* r1, const uint32_t* r2, size_t n,
                    uint32_t p0, uint32_t p1, uint32_t p2, ntt_stream_t stream) {
  t_launches = 0;
  const uint32_t ps[3] = {p0, p1, p2};
  for (uint32_t q : ps)
    if (q < 3 || !(q & 1) || q >= (1u << 30) || !is_prime_u64(q)) return NTT_ERR_MODULUS;
  if (p0 == p1 || p0 == p2 || p1 == p2) return NTT_ERR_MODULUS;
  if (!n) return NTT_OK;
  if (!out || !r0 || !r1 || !r2 || !aligned16(out) || n > SIZE_MAX / 16) return NTT_ERR_ARG;
  nttb::Crt3Consts k{};
  k.p0 = p0; k.p1 = p1; k.p2 = p2;
  auto shoup32 = [](uint64_t w, uint64_t p) { return (uint32_t)(((u128)w << 32) / p); };
  k.c01 = (uint32_t)powmod(p0 % p1, p1 - 2, p1); k.c01p = shoup32(k.c01, p1);
  k.c02 = (uint32_t)powmod(p0 % p2, p2 - 2, p2); k.c02p = shoup32(k.c02, p2);
  k.c12 = (uint32_t)powmod(p1 % p2, p2 - 2, p2); k.c12p = shoup32(k.c12, p2);
  // K_i = ceil(bound / p) * p >= the subtracted value's bound; every Shoup input
  // (< K + p < 2^31 + 2^30) stays below beta = 2^32 (any T < beta)
  k.K1 = (uint32_t)(((uint64_t)p0 + p1 - 1) / p1 * p1);
  k.K2 = (uint32_t)(((uint64_t)p0 + p2 - 1) / p2 * p2);
  k.K3 = (uint32_t)(((uint64_t)p1 + p2 - 1) / p2 * p2);
  k.p01 = (uint64_t)p0 * p1;
  cudaError_t e = nttb::launch_crt3(out, r0, r1, r2, n, k, (cudaStream_t)stream);
  ++t_launches;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

ntt_status ntt_synth_uniform(void* x, size_t count, unsigned word_bytes, uint64_t seed, uint64_t tensor_id,
                             uint64_t start, uint64_t bound, unsigned bits, ntt_stream_t stream) {
  t_launches = 0;
  if ((word_bytes != 4 && word_bytes != 8) || (!x && count)) return NTT_ERR_ARG;
  if (bound == 0 && (bits == 0 || bits > 8 * word_bytes)) return NTT_ERR_ARG;
  if (bound != 0 && word_bytes == 4 && bound > 0xFFFFFFFFull + 1) return NTT_ERR_ARG;
  cudaError_t e = nttb::launch_synth((int)word_bytes, x, count, seed, tensor_id, start, bound, bits,
                                     (cudaStream_t)stream);
  ++t_launches;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

ntt_status ntt_calibrate_butterfly(unsigned log2_beta, uint64_t p, uint64_t W, uint64_t Wp, unsigned iters,
                                   void* sink, uint64_t* n_butterflies, ntt_stream_t stream) {
  t_launches = 0;
  if ((log2_beta != 32 && log2_beta != 64) || !sink || !n_butterflies || !iters) return NTT_ERR_ARG;
  cudaError_t e = nttb::launch_calib((int)(log2_beta / 8), p, W, Wp, iters, sink, n_butterflies, (cudaStream_t)stream);
  ++t_launches;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

ntt_status ntt_debug_butterfly(ntt_plan_t pl, int alg, const void* W, const void* Wp, void* X, void* Y, size_t n,
                               ntt_stream_t stream) {
  t_launches = 0;
  if (!pl || (n && (!X || !Y))) return NTT_ERR_ARG;
  if (alg != 2 && alg != 3 && alg != 4 && alg != 5 && alg != 31 && alg != 41) return NTT_ERR_ARG;
  if (n && alg != 31 && alg != 41 && (!W || !Wp)) return NTT_ERR_ARG;
  DeviceGuard g(pl->device);
  cudaError_t e = nttb::launch_debug_bfly((int)pl->wbytes, alg, W, Wp, X, Y, n, pl->p, pl->J, (cudaStream_t)stream);
  ++t_launches;
  return e == cudaSuccess ? NTT_OK : cuda_fail(e);
}

}  // extern "C"
