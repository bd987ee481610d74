/*
 * ntt_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the batched NTT hot path of
 * D. Harvey, "Faster arithmetic for number-theoretic transforms" (arXiv:1205.2926).
 * Citations "P:n" are lines of the paper text with the section /
 * algorithm they fall in.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  The product path (paper_1205_2926_b200/) never
 * links, imports or calls it, and this file shares no code, header, table or
 * constant generator with the CUDA path.
 *
 * Arithmetic: every modular operation is fully reduced with a 128-bit `%`
 * (reading 4 of DESIGN.md: bit-exactness is defined on canonical outputs).
 * Twiddles are recomputed here by iterated multiplication, never read from the
 * plan of the product library.
 *
 * Functions and the passages they follow:
 *   orc_powmod            -- plain square-and-multiply.
 *   orc_dft_direct        -- P:24 (Section 1): b_j = sum_i omega^{ij} a_i, O(L^2).
 *   orc_ntt_forward       -- P:27-46 (Algorithm 1, "Simple FFT"), fully reduced
 *                            butterflies, output in bit-reversed order.
 *   orc_ntt_inverse       -- P:141 (Section 4): "running Algorithm 1 backwards"
 *                            with the DIT butterfly (X,Y) -> (X+WY, X-WY),
 *                            W = zeta^{-k}; unscaled (result L*a, DESIGN reading 2).
 *   orc_pointwise         -- P:21 (convolution use): c_k = a_k b_k [L^{-1}] mod p.
 *   orc_cyclic_conv_coeff -- definition of cyclic convolution, one coefficient.
 *   orc_schoolbook_mod    -- schoolbook (linear) product mod p, O(n_a n_b).
 *   orc_bfly              -- the paper's butterflies written step by step over a
 *                            generic word size beta = 2^bb (bb <= 64):
 *                            alg 2 = Algorithm 2, alg 3 = Algorithm 3
 *                            (P:110-127), alg 4 = Algorithm 4,
 *                            alg 5 = Algorithm 5.  Used to pin
 *                            Theorems 1-4 (P:77-89, P:129-135, P:161-167,
 *                            P:191-199) exhaustively at small beta.
 * Batch and multi-threaded entry points only distribute independent transforms
 * (or the independent butterflies of one stage) over threads; the arithmetic
 * is the same per-butterfly code.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((u128)a * b) % p); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((u128)a + b) % p); }
/* (a - b) mod p for any a, b (not only canonical ones) */
static uint64_t submod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((u128)(a % p) + p - (b % p)) % p); }

uint64_t orc_powmod(uint64_t b, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  b %= p;
  while (e) {
    if (e & 1) r = mulmod(r, b, p);
    b = mulmod(b, b, p);
    e >>= 1;
  }
  return r;
}

/* b_j = sum_{i<L} omega^{ij} a_i, natural order.  O(L^2). */
void orc_dft_direct(uint64_t p, uint64_t omega, uint64_t L, const uint64_t* a, uint64_t* b) {
  for (uint64_t j = 0; j < L; ++j) {
    uint64_t wj = orc_powmod(omega, j, p); /* omega^j */
    uint64_t pw = 1 % p;                   /* omega^{ij}, i = 0 */
    uint64_t acc = 0;
    for (uint64_t i = 0; i < L; ++i) {
      acc = addmod(acc, mulmod(pw, a[i] % p, p), p);
      pw = mulmod(pw, wj, p);
    }
    b[j] = acc;
  }
}

/* One DIF stage of Algorithm 1, butterflies q in [q0, q1) of the L/2
 * butterflies of stage i, enumerated as q = j*m + k (j < 2^{i-1}, k < m). */
static void alg1_stage_range(uint64_t p, uint64_t zeta, uint64_t m, uint64_t* x, uint64_t q0, uint64_t q1) {
  uint64_t k = q0 % m;
  uint64_t zk = orc_powmod(zeta, k, p); /* zeta^k */
  for (uint64_t q = q0; q < q1; ++q) {
    uint64_t j = q / m;
    uint64_t t = 2 * j * m;
    uint64_t X = x[t + k], Y = x[t + k + m];
    x[t + k] = addmod(X, Y, p);                      /* x_{t+k} + x_{t+k+m} */
    x[t + k + m] = mulmod(zk, submod(X, Y, p), p);   /* zeta^k (x_{t+k} - x_{t+k+m}) */
    if (++k == m) { k = 0; zk = 1 % p; } else zk = mulmod(zk, zeta, p);
  }
}

/* One stage of Algorithm 1 run backwards: (X,Y) -> (X + W Y, X - W Y),
 * W = zeta_inv^k with zeta_inv = omega^{-2^{i-1}}. */
static void alg1_inv_stage_range(uint64_t p, uint64_t zeta_inv, uint64_t m, uint64_t* x, uint64_t q0, uint64_t q1) {
  uint64_t k = q0 % m;
  uint64_t zk = orc_powmod(zeta_inv, k, p);
  for (uint64_t q = q0; q < q1; ++q) {
    uint64_t j = q / m;
    uint64_t t = 2 * j * m;
    uint64_t X = x[t + k], Y = x[t + k + m];
    uint64_t WY = mulmod(zk, Y % p, p);
    x[t + k] = addmod(X, WY, p);
    x[t + k + m] = submod(X, WY, p);
    if (++k == m) { k = 0; zk = 1 % p; } else zk = mulmod(zk, zeta_inv, p);
  }
}

/* Algorithm 1: in place, natural in, bit-reversed out, canonical. */
void orc_ntt_forward(uint64_t p, uint64_t omega, unsigned ell, uint64_t* x) {
  uint64_t L = (uint64_t)1 << ell;
  for (uint64_t i = 0; i < L; ++i) x[i] %= p;
  for (unsigned i = 1; i <= ell; ++i) {
    uint64_t zeta = orc_powmod(omega, (uint64_t)1 << (i - 1), p); /* zeta <- omega^{2^{i-1}} */
    uint64_t m = (uint64_t)1 << (ell - i);                          /* m <- 2^{ell-i} */
    alg1_stage_range(p, zeta, m, x, 0, L / 2);
  }
}

/* Algorithm 1 backwards: bit-reversed in, natural out, result L*a. */
void orc_ntt_inverse(uint64_t p, uint64_t omega, unsigned ell, uint64_t* x) {
  uint64_t L = (uint64_t)1 << ell;
  uint64_t omega_inv = orc_powmod(omega, p - 2, p); /* p prime (Fermat) */
  for (uint64_t i = 0; i < L; ++i) x[i] %= p;
  for (unsigned i = ell; i >= 1; --i) {
    uint64_t zeta_inv = orc_powmod(omega_inv, (uint64_t)1 << (i - 1), p);
    uint64_t m = (uint64_t)1 << (ell - i);
    alg1_inv_stage_range(p, zeta_inv, m, x, 0, L / 2);
  }
}

/* ---- multi-threaded drivers (independent work only) ---- */
typedef struct {
  uint64_t p, omega;
  unsigned ell;
  uint64_t* x;
  uint64_t b0, b1;
  int inverse;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  uint64_t L = (uint64_t)1 << j->ell;
  for (uint64_t b = j->b0; b < j->b1; ++b) {
    if (j->inverse) orc_ntt_inverse(j->p, j->omega, j->ell, j->x + b * L);
    else orc_ntt_forward(j->p, j->omega, j->ell, j->x + b * L);
  }
  return NULL;
}

/* `batch` independent transforms, contiguous (transform b at b*L), over nthreads. */
void orc_ntt_batch(uint64_t p, uint64_t omega, unsigned ell, uint64_t* x, uint64_t batch, int inverse, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > batch) nthreads = (int)(batch ? batch : 1);
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  batch_job* jobs = (batch_job*)calloc((size_t)nthreads, sizeof(batch_job));
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (batch_job){p, omega, ell, x, batch * (uint64_t)t / nthreads, batch * (uint64_t)(t + 1) / nthreads, inverse};
    pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

typedef struct {
  uint64_t p, omega;
  unsigned ell;
  uint64_t* x;
  int tid, nthreads, inverse;
  pthread_barrier_t* bar;
} stage_job;

static void* stage_worker(void* arg) {
  stage_job* s = (stage_job*)arg;
  uint64_t L = (uint64_t)1 << s->ell, half = L / 2;
  uint64_t q0 = half * (uint64_t)s->tid / s->nthreads, q1 = half * (uint64_t)(s->tid + 1) / s->nthreads;
  for (uint64_t i = q0 * 2; i < q1 * 2; ++i) s->x[i] %= s->p;
  pthread_barrier_wait(s->bar);
  if (!s->inverse) {
    for (unsigned i = 1; i <= s->ell; ++i) {
      uint64_t zeta = orc_powmod(s->omega, (uint64_t)1 << (i - 1), s->p);
      if (q1 > q0) alg1_stage_range(s->p, zeta, (uint64_t)1 << (s->ell - i), s->x, q0, q1);
      pthread_barrier_wait(s->bar);
    }
  } else {
    uint64_t omega_inv = orc_powmod(s->omega, s->p - 2, s->p);
    for (unsigned i = s->ell; i >= 1; --i) {
      uint64_t zeta_inv = orc_powmod(omega_inv, (uint64_t)1 << (i - 1), s->p);
      if (q1 > q0) alg1_inv_stage_range(s->p, zeta_inv, (uint64_t)1 << (s->ell - i), s->x, q0, q1);
      pthread_barrier_wait(s->bar);
    }
  }
  return NULL;
}

/* One transform, the L/2 independent butterflies of each stage split over threads. */
void orc_ntt_single_mt(uint64_t p, uint64_t omega, unsigned ell, uint64_t* x, int inverse, int nthreads) {
  if (ell == 0) { x[0] %= p; return; }
  if (nthreads < 1) nthreads = 1;
  pthread_barrier_t bar;
  pthread_barrier_init(&bar, NULL, (unsigned)nthreads);
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  stage_job* jobs = (stage_job*)calloc((size_t)nthreads, sizeof(stage_job));
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (stage_job){p, omega, ell, x, t, nthreads, inverse, &bar};
    pthread_create(&th[t], NULL, stage_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_barrier_destroy(&bar);
  free(th);
  free(jobs);
}

/* P:21 convolution use: c_k = a_k b_k (times L^{-1} if scale_L != 0) mod p. */
void orc_pointwise(uint64_t p, const uint64_t* a, const uint64_t* b, uint64_t* c, uint64_t n, uint64_t scale_L) {
  uint64_t s = scale_L ? orc_powmod(scale_L % p, p - 2, p) : 1 % p;
  for (uint64_t k = 0; k < n; ++k) c[k] = mulmod(mulmod(a[k] % p, b[k] % p, p), s, p);
}

/* Cyclic convolution, one coefficient: c_k = sum_i a_i b_{(k-i) mod L} mod p. */
uint64_t orc_cyclic_conv_coeff(uint64_t p, const uint64_t* a, const uint64_t* b, uint64_t L, uint64_t k) {
  uint64_t acc = 0;
  for (uint64_t i = 0; i < L; ++i) acc = addmod(acc, mulmod(a[i] % p, b[(k + L - i) % L] % p, p), p);
  return acc;
}

/* Schoolbook (linear) product mod p: out has na + nb - 1 entries. */
void orc_schoolbook_mod(uint64_t p, const uint64_t* a, uint64_t na, const uint64_t* b, uint64_t nb, uint64_t* out) {
  if (!na || !nb) return;
  memset(out, 0, sizeof(uint64_t) * (na + nb - 1));
  for (uint64_t i = 0; i < na; ++i)
    for (uint64_t j = 0; j < nb; ++j) out[i + j] = addmod(out[i + j], mulmod(a[i] % p, b[j] % p, p), p);
}

/* ---- the paper's butterflies over beta = 2^bb, step by step (bb in 2..64) ---- */
static u128 wrapb(u128 v, unsigned bb) { return bb >= 128 ? v : (v & ((((u128)1) << bb) - 1)); }

/* Returns the outputs through Xo/Yo; all word operations wrap modulo beta, as
 * a machine word would, so a violated precondition shows up in the checks.
 *   alg 2: Algorithm 2.  T <- X - Y, "if T < 0" read as X < Y.
 *   alg 3: Algorithm 3.
 *   alg 4: Algorithm 4.
 *   alg 5: Algorithm 5; Wp is beta*W mod p, J = p^{-1} mod beta. */
int orc_bfly(int alg, unsigned bb, uint64_t p, uint64_t W, uint64_t Wp, uint64_t J, uint64_t X, uint64_t Y,
             uint64_t* Xo, uint64_t* Yo) {
  u128 Xp, Yp, T, Q;
  switch (alg) {
    case 2:
      Xp = wrapb((u128)X + Y, bb);                    /* X' <- X + Y */
      if (Xp >= p) Xp = wrapb(Xp - p, bb);            /* if X' >= p then X' <- X' - p */
      if (X < Y) T = wrapb((u128)X + p - Y, bb);      /* T <- X - Y; if T < 0 then T <- T + p */
      else T = wrapb((u128)X - Y, bb);
      Q = ((u128)Wp * T) >> bb;                       /* Q <- floor(W'T / beta) */
      Yp = wrapb((u128)W * T - (u128)Q * p, bb);      /* Y' <- (WT - Qp) mod beta */
      if (Yp >= p) Yp = wrapb(Yp - p, bb);            /* if Y' >= p then Y' <- Y' - p */
      break;
    case 3:
      Xp = wrapb((u128)X + Y, bb);                    /* X' <- X + Y */
      if (Xp >= 2 * (u128)p) Xp = wrapb(Xp - 2 * (u128)p, bb); /* if X' >= 2p then X' <- X' - 2p */
      T = wrapb((u128)X + (((u128)1) << bb) - Y + 2 * (u128)p, bb); /* T <- X - Y + 2p */
      Q = ((u128)Wp * T) >> bb;                       /* Q <- floor(W'T / beta) */
      Yp = wrapb((u128)W * T - (u128)Q * p, bb);      /* Y' <- (WT - Qp) mod beta */
      break;
    case 4: {
      u128 Xr = X;
      if (Xr >= 2 * (u128)p) Xr = wrapb(Xr - 2 * (u128)p, bb); /* if X >= 2p then X <- X - 2p */
      Q = ((u128)Wp * Y) >> bb;                        /* Q <- floor(W'Y / beta) */
      T = wrapb((u128)W * Y - (u128)Q * p, bb);        /* T <- (WY - Qp) mod beta */
      Xp = wrapb(Xr + T, bb);                          /* X' <- X + T */
      Yp = wrapb(Xr + (((u128)1) << bb) - T + 2 * (u128)p, bb); /* Y' <- X - T + 2p */
      break;
    }
    case 5: {
      Xp = wrapb((u128)X + Y, bb);
      if (Xp >= 2 * (u128)p) Xp = wrapb(Xp - 2 * (u128)p, bb);
      T = wrapb((u128)X + (((u128)1) << bb) - Y + 2 * (u128)p, bb); /* T <- X - Y + 2p */
      u128 R = (u128)Wp * T;                           /* R1 beta + R0 <- W'T */
      u128 R1 = R >> bb, R0 = wrapb(R, bb);
      Q = wrapb(R0 * J, bb);                           /* Q <- R0 J mod beta */
      u128 H = ((u128)Q * p) >> bb;                    /* H <- floor(Qp / beta) */
      Yp = wrapb(R1 + (((u128)1) << bb) - H + p, bb);  /* Y' <- R1 - H + p */
      break;
    }
    default:
      return -1;
  }
  *Xo = (uint64_t)Xp;
  *Yo = (uint64_t)Yp;
  return 0;
}

/* Array form of orc_bfly (W, Wp per element). */
int orc_bfly_batch(int alg, unsigned bb, uint64_t p, uint64_t J, uint64_t n, const uint64_t* W, const uint64_t* Wp,
                   const uint64_t* X, const uint64_t* Y, uint64_t* Xo, uint64_t* Yo) {
  for (uint64_t i = 0; i < n; ++i)
    if (orc_bfly(alg, bb, p, W[i], Wp[i], J, X[i], Y[i], &Xo[i], &Yo[i])) return -1;
  return 0;
}

/* P:24, second form: the NTT evaluates a(x) = a_0 + a_1 x + ... + a_{L-1} x^{L-1}
 * at the powers of omega.  Horner evaluation of a(x) mod p, O(L). */
uint64_t orc_poly_eval(uint64_t p, const uint64_t* a, uint64_t L, uint64_t x) {
  uint64_t acc = 0;
  for (uint64_t i = L; i-- > 0;) acc = addmod(mulmod(acc, x % p, p), a[i] % p, p);
  return acc;
}
