"""Randomised parity sweep: primes drawn at random (p = k 2^m + 1 < beta/4, both word sizes, generic and
p = 1 mod 2^32 forms), every schedule shape up to 2^20 and ragged batches -- forward and inverse bit-exact
against the oracle, inverse o forward = L x.  Seeded, so a failure reproduces."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from gpu_util import rand_residues, to_dev, to_host  # noqa: E402


def _is_prime(n):
    if n < 2:
        return False
    for q in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % q == 0:
            return n == q
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _draw_case(rng, bits):
    """(p, omega, ell, batch): p prime, p < 2^(bits-2), 2^ell | p - 1, omega primitive 2^ell-th root."""
    ell = rng.choice([1, 3, 6, 9, 11, 12, 13, 14, 15, 16, 17, 18, 20] if bits == 64 else
                     [1, 4, 7, 10, 12, 14, 15, 16, 17, 19])
    top = bits - 2
    while True:
        m = rng.randint(ell, min(ell + 12, top - 2))
        k = rng.randrange(1, 1 << (top - m))
        p = k * (1 << m) + 1
        if p >= 1 << top or not _is_prime(p):
            continue
        for g in range(2, 200):
            w = pow(g, (p - 1) >> ell, p)
            if ell == 0 or pow(w, 1 << (ell - 1), p) == p - 1:
                batch = rng.choice([1, 2, 3, 5]) if ell >= 16 else rng.choice([1, 7, 33, 130])
                return p, w, ell, batch


@pytest.fixture(scope="module")
def ntt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1205_2926_b200 as P
    return P


@pytest.mark.parametrize("seed", range(24))
def test_random_prime_sweep(ntt, seed):
    rng = random.Random(0x5EED + seed)
    bits = 64 if seed % 3 else 32
    p, w, ell, batch = _draw_case(rng, bits)
    L = 1 << ell
    plan = ntt.Plan(p, w, ell, bits)
    x = rand_residues(np.random.default_rng(seed), 2 * p, (batch, L))  # Alg. 3 accepts [0, 2p)
    d = to_dev(x, bits)
    plan.forward(d)
    f = to_host(d)
    nthr = oracle.default_threads()
    assert np.array_equal(f, oracle.ntt_forward(p, w, x % np.uint64(p), nthreads=nthr)), (p, ell, batch)
    plan.inverse(d)
    assert np.array_equal(to_host(d), ((x.astype(object) % p) * L % p).astype(np.uint64)), (p, ell, batch)
