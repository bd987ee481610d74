"""Pins for the CPU oracle (oracle/), against what the paper and mathematics fix.

No pin here re-types the oracle's own formula: each checks the oracle against a
worked example, a second algorithm (direct DFT vs Algorithm 1), a closed form,
an invariant, or an exhaustive theorem statement.  Citations: P:n = PAPER.md
line n, S:n = SPEC.md line n.
"""
import random

import numpy as np
import pytest

import oracle
from conftest import read_golden

P30 = 998244353                    # 119*2^23 + 1 (configs C1, C3)
P62 = 29 * 2**57 + 1               # 4179340454199820289 (configs C2, C4, C5)
RNS = (469762049, 167772161, 998244353)  # config C3


def root(p, L):
    """omega = 3^((p-1)/L): the BASELINE.json rule (reading 1)."""
    return pow(3, (p - 1) // L, p)


def bitrev(j, ell):
    return int(format(j, f"0{ell}b")[::-1], 2) if ell else 0


# ---------------------------------------------------------------- worked example
def test_worked_example_p13():
    g = read_golden("worked_example_p13.txt")
    p, w, a = g["p"], g["omega"], g["input"]
    assert list(oracle.dft_direct(p, w, a)) == g["dft_natural"]
    assert list(oracle.ntt_forward(p, w, a)) == g["forward_bitrev"]      # P:33 (Alg. 1)
    assert list(oracle.ntt_inverse(p, w, g["forward_bitrev"])) == g["inverse_unscaled"]


# ---------------------------------------------------------------- two algorithms agree
@pytest.mark.parametrize("p", [P30, P62, 469762049, 167772161, 97, 257])
def test_alg1_equals_direct_dft_bitreversed(p):
    """Algorithm 1 output j holds b_{rev(j)} of the direct sum, every L <= 2^10."""
    rng = np.random.default_rng(p)
    max_ell = min(10, ((p - 1) & -(p - 1)).bit_length() - 1)
    for ell in range(0, max_ell + 1):
        L = 1 << ell
        w = root(p, L) if p not in (97, 257) else pow(5 if p == 97 else 3, (p - 1) // L, p)
        a = rng.integers(0, p, size=L, dtype=np.uint64) if p < 2**63 else None
        b = oracle.dft_direct(p, w, a)
        out = oracle.ntt_forward(p, w, a)
        assert [int(out[j]) for j in range(L)] == [int(b[bitrev(j, ell)]) for j in range(L)], (p, ell)


def test_L2_special_case():
    """L = 2: omega = -1, b = (a0 + a1, a0 - a1)."""
    for p in (P30, P62):
        a0, a1 = p - 1, p - 2
        out = oracle.ntt_forward(p, p - 1, [a0, a1])
        assert [int(v) for v in out] == [(a0 + a1) % p, (a0 - a1) % p]


# ---------------------------------------------------------------- closed forms at larger L
@pytest.mark.parametrize("p,ell", [(P30, 16), (P62, 16), (P62, 20)])
def test_closed_forms(p, ell):
    L = 1 << ell
    w = root(p, L)
    assert pow(w, L // 2, p) == p - 1 and pow(w, L, p) == 1  # primitive L-th root
    # delta -> all ones
    d = np.zeros(L, dtype=np.uint64); d[0] = 1
    assert (oracle.ntt_forward(p, w, d) == 1).all()
    # shifted delta e_s -> out[j] = omega^{s*rev(j)}
    s = 12345 % L
    e = np.zeros(L, dtype=np.uint64); e[s] = 1
    out = oracle.ntt_forward(p, w, e)
    for j in random.Random(ell).sample(range(L), 64):
        assert int(out[j]) == pow(w, s * bitrev(j, ell), p)
    # constant c -> (L*c, 0, ..., 0)
    c = p - 3
    out = oracle.ntt_forward(p, w, np.full(L, c, dtype=np.uint64))
    assert int(out[0]) == (L * c) % p and not out[1:].any()
    # chirp a_i = omega^{-m i} -> L at position rev(m), zero elsewhere
    m = 777 % L
    winv_m = pow(w, (L - m) % L, p)
    chirp = np.empty(L, dtype=np.uint64)
    v = 1
    for i in range(L):
        chirp[i] = v
        v = v * winv_m % p
    out = oracle.ntt_forward(p, w, chirp)
    nz = np.flatnonzero(out)
    assert list(nz) == [bitrev(m, ell)] and int(out[nz[0]]) == L % p


@pytest.mark.parametrize("p,ell", [(P30, 14), (P62, 14)])
def test_spot_evaluation_horner(p, ell):
    """P:24 second form: output j is the polynomial a(x) evaluated at omega^{rev(j)}."""
    L = 1 << ell
    w = root(p, L)
    rng = np.random.default_rng(7)
    a = rng.integers(0, p, size=L, dtype=np.uint64)
    out = oracle.ntt_forward(p, w, a)
    coeffs = [int(v) for v in a]
    for j in [0, 1, L - 1] + random.Random(3).sample(range(L), 8):
        x = pow(w, bitrev(j, ell), p)
        acc = 0
        for cf in reversed(coeffs):  # Horner
            acc = (acc * x + cf) % p
        assert int(out[j]) == acc
    # out[0] = sum a_i ; out[1] = b_{L/2} = sum (-1)^i a_i
    assert int(out[0]) == sum(coeffs) % p
    assert int(out[1]) == sum(cf if i % 2 == 0 else -cf for i, cf in enumerate(coeffs)) % p


def test_linearity():
    """NTT(alpha x + y) = alpha NTT(x) + NTT(y) mod p."""
    p, ell = P62, 12
    L = 1 << ell
    w = root(p, L)
    rng = np.random.default_rng(11)
    x = rng.integers(0, p, size=L, dtype=np.uint64)
    y = rng.integers(0, p, size=L, dtype=np.uint64)
    alpha = 123456789123456789
    comb = np.array([(alpha * int(u) + int(v)) % p for u, v in zip(x, y)], dtype=np.uint64)
    fx, fy, fc = (oracle.ntt_forward(p, w, t) for t in (x, y, comb))
    assert all(int(c) == (alpha * int(u) + int(v)) % p for u, v, c in zip(fx, fy, fc))


# ---------------------------------------------------------------- inverse
@pytest.mark.parametrize("p,ell", [(P30, 10), (P62, 12), (RNS[0], 16), (RNS[1], 13)])
def test_inverse_of_forward_is_L_times_identity(p, ell):
    """P:141 (Algorithm 1 run backwards, unscaled): inverse(forward(x)) = L x (config C2 check)."""
    L = 1 << ell
    w = root(p, L)
    x = np.random.default_rng(ell).integers(0, p, size=(3, L), dtype=np.uint64)
    y = oracle.ntt_inverse(p, w, oracle.ntt_forward(p, w, x))
    assert np.array_equal(y.astype(object), (x.astype(object) * L) % p)


def test_multithreaded_single_transform_matches():
    p, ell = P62, 16
    L = 1 << ell
    w = root(p, L)
    x = np.random.default_rng(5).integers(0, p, size=L, dtype=np.uint64)
    a = oracle.ntt_forward(p, w, x, nthreads=1)
    b = oracle.ntt_forward(p, w, x, nthreads=4)
    assert np.array_equal(a, b)
    assert np.array_equal(oracle.ntt_inverse(p, w, a, nthreads=4), oracle.ntt_inverse(p, w, a, nthreads=1))


# ---------------------------------------------------------------- convolution
def test_schoolbook_closed_forms():
    assert list(oracle.schoolbook_mod(13, [1, 1], [1, 1])) == [1, 2, 1]
    assert list(oracle.schoolbook_mod(10**9 + 7, [1, 2, 3, 4], [4, 3, 2, 1])) == [4, 11, 20, 30, 20, 11, 4]
    # (1+x)^n binomial coefficients
    p, n = P30, 40
    poly = [1]
    for _ in range(n):
        poly = [int(v) for v in oracle.schoolbook_mod(p, poly, [1, 1])]
    from math import comb
    assert poly == [comb(n, k) % p for k in range(n + 1)]


@pytest.mark.parametrize("p", RNS + (P62,))
def test_convolution_theorem(p):
    """forward, forward, pointwise (x L^{-1}), inverse = cyclic convolution = schoolbook (deg < L)."""
    ell = 10
    L = 1 << ell
    w = root(p, L)
    rng = np.random.default_rng(p % 1000)
    a = np.zeros(L, dtype=np.uint64); b = np.zeros(L, dtype=np.uint64)
    a[: L // 2] = rng.integers(0, 2**20, size=L // 2)   # config C3 shape: coeffs < 2^20, zero-padded
    b[: L // 2] = rng.integers(0, 2**20, size=L // 2)
    c = oracle.ntt_inverse(p, w, oracle.pointwise(p, oracle.ntt_forward(p, w, a), oracle.ntt_forward(p, w, b), scale_L=L))
    ref = oracle.schoolbook_mod(p, a[: L // 2], b[: L // 2])
    assert np.array_equal(c[: ref.size], ref) and not c[ref.size:].any()
    for k in (0, 1, L // 2, L - 1):
        assert oracle.cyclic_conv_coeff(p, a, b, k) == int(c[k])


def test_cyclic_conv_wraps():
    p, L = 97, 8
    a = [0] * L; a[3] = 1          # x^3
    b = list(range(1, L + 1))
    # multiplying by x^3 cyclically shifts b by 3
    assert [oracle.cyclic_conv_coeff(p, a, b, k) for k in range(L)] == [b[(k - 3) % L] for k in range(L)]


# ---------------------------------------------------------------- butterflies (Theorems 1-4)
def _odd_primes_below(n):
    return [q for q in range(3, n) if all(q % d for d in range(2, int(q**0.5) + 1))]


def test_butterfly_traces_p17():
    g = read_golden("butterfly_traces_p17.txt")
    bb, p, W = g["beta_bits"], g["p"], g["W"]
    assert g["Wp_shoup"] == (W << bb) // p and g["J"] * p % (1 << bb) == 1
    for alg, X, Y, Xo, Yo in g["rows"]:
        Wp = g["Wp_mont"] if alg == 5 else g["Wp_shoup"]
        xo, yo = oracle.bfly(alg, bb, p, W, Wp, [X], [Y], J=g["J"])
        assert (int(xo[0]), int(yo[0])) == (Xo, Yo), alg


def _check_theorem(alg, bb, p, in_bound, out_bound):
    """Exhaustive over W in (0,p) and legal (X,Y): congruence + interval contracts.
    Returns the number of violations."""
    beta = 1 << bb
    J = pow(p, -1, beta) if p % 2 else 0
    side = np.arange(in_bound * p, dtype=np.int64)
    X, Y = (g.ravel() for g in np.meshgrid(side, side, indexing="ij"))
    bad = 0
    for W in range(1, p):
        Wp = (W * beta) % p if alg == 5 else (W * beta) // p
        xo, yo = oracle.bfly(alg, bb, p, W, Wp, X.astype(np.uint64), Y.astype(np.uint64), J=J)
        xo, yo = xo.astype(np.int64), yo.astype(np.int64)
        if alg in (2, 3, 5):
            want_x, want_y = (X + Y) % p, (W * (X - Y)) % p
        else:  # alg 4: (X + WY, X - WY)
            want_x, want_y = (X + W * Y) % p, (X - W * Y) % p
        ok = (xo % p == want_x) & (yo % p == want_y) & (xo < out_bound * p) & (yo < out_bound * p)
        bad += int((~ok).sum())
    return bad


@pytest.mark.parametrize("alg,pmax,in_b,out_b", [
    (2, 128, 1, 1),   # Thm 1: p < beta/2, [0,p) -> [0,p)
    (3, 64, 2, 2),    # Thm 2: p < beta/4, [0,2p) -> [0,2p)
    (4, 64, 4, 4),    # Thm 3: p < beta/4, [0,4p) -> [0,4p)
    (5, 64, 2, 2),    # Thm 4: p odd, p < beta/4, [0,2p) -> [0,2p)
])
def test_theorems_exhaustive_beta8(alg, pmax, in_b, out_b):
    primes = _odd_primes_below(pmax)
    if alg == 4:
        primes = [q for q in primes if q < 32] + [61]  # keep the run short; 61 is the largest legal p
    assert sum(_check_theorem(alg, 8, q, in_b, out_b) for q in primes) == 0


def test_theorem2_negative_control():
    """Alg. 3 with p in (beta/4, beta/2) must violate its contract (the hypothesis matters)."""
    assert sum(_check_theorem(3, 8, q, 2, 2) for q in (67, 97, 127)) > 0


def test_theorem2_input_range_control():
    """Feeding Alg. 3 inputs outside [0,2p) (here [0,4p)) must show violations: the checker has power."""
    bad = 0
    for p in (53, 61):
        beta = 256
        side = np.arange(4 * p, dtype=np.uint64)
        X, Y = (g.ravel() for g in np.meshgrid(side, side, indexing="ij"))
        for W in (1, 2, p - 1):
            xo, yo = oracle.bfly(3, 8, p, W, (W * beta) // p, X, Y)
            bad += int(((xo >= 2 * p) | (yo >= 2 * p)).sum())
    assert bad > 0


@pytest.mark.parametrize("alg", [2, 3, 4, 5])
def test_theorems_random_beta64(alg):
    """Same contracts at the native beta = 2^64 with the 62-bit config prime (p < beta/4)."""
    bb, p = 64, P62
    beta = 1 << bb
    rng = random.Random(alg)
    J = pow(p, -1, beta)
    in_b = {2: 1, 3: 2, 4: 4, 5: 2}[alg]
    for _ in range(3000):
        W = rng.randrange(1, p)
        Wp = (W * beta) % p if alg == 5 else (W * beta) // p
        X, Y = rng.randrange(in_b * p), rng.randrange(in_b * p)
        xo, yo = oracle.bfly(alg, bb, p, W, Wp, [X], [Y], J=J)
        xo, yo = int(xo[0]), int(yo[0])
        if alg == 4:
            assert xo % p == (X + W * Y) % p and yo % p == (X - W * Y) % p
        else:
            assert xo % p == (X + Y) % p and yo % p == W * (X - Y) % p
        assert xo < in_b * p and yo < in_b * p


def test_theorem1_bound_shoup_any_T():
    """P:85 / P:104: 0 <= WT - Qp < 2p for ANY 0 <= T < beta (exhaustive at beta = 2^8)."""
    bb, beta = 8, 256
    for p in _odd_primes_below(128):
        T = np.arange(beta, dtype=np.int64)
        for W in range(1, p):
            Wp = (W * beta) // p
            Q = (Wp * T) >> bb
            r = W * T - Q * p
            assert ((r >= 0) & (r < 2 * p)).all()


# ---- F3: three-prime CRT (the RNS use of P:21)
RNS3 = (469762049, 167772161, 998244353)


def test_crt_recovers_known_integers():
    """Residues of known integers (taken with Python's %, not the oracle) lift back to the integers,
    including the range ends 0 and p0 p1 p2 - 1."""
    M = RNS3[0] * RNS3[1] * RNS3[2]
    rng = np.random.default_rng(11)
    xs = [0, 1, M - 1, M // 2, RNS3[0], RNS3[0] * RNS3[1]] + [int(v) for v in rng.integers(0, 2**62, 50)]
    xs += [(int(a) << 40) + int(b) for a, b in zip(rng.integers(0, 2**40, 20), rng.integers(0, 2**40, 20))]
    xs = [x % M for x in xs]
    res = [np.array([x % q for x in xs], dtype=np.uint64) for q in RNS3]
    assert oracle.crt(res, RNS3) == xs


def test_crt_gives_exact_integer_product():
    """Config C3 in miniature: the CRT of the three residue convolutions (oracle NTT route) is the exact
    integer product computed by numpy's integer convolution (coefficients < 2^55 < p0 p1 p2)."""
    ell, half = 8, 128
    L = 1 << ell
    rng = np.random.default_rng(5)
    a = rng.integers(0, 2**20, half, dtype=np.uint64)
    b = rng.integers(0, 2**20, half, dtype=np.uint64)
    exact = np.convolve(a.astype(np.int64), b.astype(np.int64))  # 2*half - 1 < L coefficients
    pa = np.zeros(L, dtype=np.uint64); pa[:half] = a
    pb = np.zeros(L, dtype=np.uint64); pb[:half] = b
    res = []
    for q in RNS3:
        w = pow(3, (q - 1) // L, q)
        res.append(oracle.ntt_inverse(q, w, oracle.pointwise(q, oracle.ntt_forward(q, w, pa),
                                                            oracle.ntt_forward(q, w, pb), scale_L=L)))
    got = oracle.crt(res, RNS3)
    assert got[:2 * half - 1] == [int(v) for v in exact] and got[2 * half - 1:] == [0] * (L - 2 * half + 1)


# ---------------------------------------------------------------- poly_eval / ntt_output_at
# orc_poly_eval (Horner) and its wrapper ntt_output_at are the oracle's route to sampled outputs of
# long transforms (2^22-2^28, the C4 sample) in the GPU parity tests; pinned here against the direct
# DFT (P:24 sum form), closed forms of the evaluation form ("evaluation at 1, omega, ...") and a
# mutation control.
@pytest.mark.parametrize("p", [P30, P62, 469762049])
def test_output_at_equals_direct_dft(p):
    """ntt_output_at(p, omega, a, j) = b_{rev(j)} of the O(L^2) direct sum, every j, L <= 2^10."""
    rng = np.random.default_rng(p & 0xFFFF)
    for ell in (0, 1, 2, 5, 10):
        L = 1 << ell
        w = root(p, L)
        a = rng.integers(0, p, size=L, dtype=np.uint64)
        b = oracle.dft_direct(p, w, a)
        got = [oracle.ntt_output_at(p, w, a, j) for j in range(L)]
        assert got == [int(b[bitrev(j, ell)]) for j in range(L)], (p, ell)


def test_poly_eval_small_values():
    """a(x) = 1 + 2x + 3x^2: a(5) = 86 = 8 mod 13; a(0) = a_0; a(1) = sum a_i; a(-1) alternating sum."""
    assert oracle.poly_eval(13, [1, 2, 3], 5) == 8
    assert oracle.poly_eval(13, [1, 2, 3], 0) == 1
    assert oracle.poly_eval(P62, [P62 - 1, P62 - 1, 5], 1) == (2 * (P62 - 1) + 5) % P62
    assert oracle.poly_eval(P62, [7, 11, 13, 17], P62 - 1) == (7 - 11 + 13 - 17) % P62
    assert oracle.poly_eval(P30, [], 5) == 0


@pytest.mark.parametrize("p", [P62, P30])
def test_output_at_closed_forms_2p20(p):
    """L = 2^20: shifted delta e_s gives omega^{s rev(j)}; all-ones gives L at j = 0 and 0 elsewhere."""
    ell = 20
    L = 1 << ell
    w = root(p, L)
    s = 987654
    e = np.zeros(L, dtype=np.uint64)
    e[s] = 1
    ones = np.ones(L, dtype=np.uint64)
    for j in [0, 1, L - 1] + random.Random(5).sample(range(L), 6):
        assert oracle.ntt_output_at(p, w, e, j) == pow(w, s * bitrev(j, ell), p)
        assert oracle.ntt_output_at(p, w, ones, j) == (L % p if j == 0 else 0)


def test_output_at_mutation_control():
    """A reversed coefficient order (a_{L-1-i}) must not reproduce the transform."""
    p, ell = P62, 8
    L = 1 << ell
    w = root(p, L)
    a = np.random.default_rng(9).integers(0, p, size=L, dtype=np.uint64)
    b = oracle.dft_direct(p, w, a)
    rev_a = a[::-1].copy()
    mism = sum(oracle.ntt_output_at(p, w, rev_a, j) != int(b[bitrev(j, ell)]) for j in range(L))
    assert mism > L // 2
