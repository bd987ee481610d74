"""CPU oracle for the batched NTT hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct reference for D. Harvey, "Faster arithmetic for
number-theoretic transforms" (arXiv:1205.2926).  The arithmetic lives in
``ntt_oracle.c`` (fully reduced 128-bit ``%`` arithmetic, see its header for
the per-function PAPER.md citations); this module only compiles it with gcc
and marshals numpy arrays.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_1205_2926_b200`` never imports it; the two share no
code.  Nothing here is pinned by itself: ``tests/test_oracle_pins.py`` pins it
against the paper's definition, its worked examples, closed forms and
Theorems 1-4 (exhaustively at beta = 2^8).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ntt_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

U64P = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    """Compile ntt_oracle.c into liboracle.so (gcc -O2, pthreads)."""
    stale = (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)
    if force or stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, c_int, c_uint = ctypes.c_uint64, ctypes.c_int, ctypes.c_uint
        lib.orc_powmod.restype = u64
        lib.orc_powmod.argtypes = [u64, u64, u64]
        lib.orc_dft_direct.argtypes = [u64, u64, u64, U64P, U64P]
        lib.orc_ntt_forward.argtypes = [u64, u64, c_uint, U64P]
        lib.orc_ntt_inverse.argtypes = [u64, u64, c_uint, U64P]
        lib.orc_ntt_batch.argtypes = [u64, u64, c_uint, U64P, u64, c_int, c_int]
        lib.orc_ntt_single_mt.argtypes = [u64, u64, c_uint, U64P, c_int, c_int]
        lib.orc_pointwise.argtypes = [u64, U64P, U64P, U64P, u64, u64]
        lib.orc_cyclic_conv_coeff.restype = u64
        lib.orc_cyclic_conv_coeff.argtypes = [u64, U64P, U64P, u64, u64]
        lib.orc_schoolbook_mod.argtypes = [u64, U64P, u64, U64P, u64, U64P]
        lib.orc_poly_eval.restype = u64
        lib.orc_poly_eval.argtypes = [u64, U64P, u64, u64]
        lib.orc_bfly_batch.restype = c_int
        lib.orc_bfly_batch.argtypes = [c_int, c_uint, u64, u64, u64, U64P, U64P, U64P, U64P, U64P, U64P]
        _lib = lib
    return _lib


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(U64P)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))


def powmod(b: int, e: int, p: int) -> int:
    return int(_load().orc_powmod(b, e, p))


def dft_direct(p: int, omega: int, a) -> np.ndarray:
    """b_j = sum_i omega^{ij} a_i, natural order, O(L^2)."""
    a = _u64(a)
    b = np.empty_like(a)
    _load().orc_dft_direct(p, omega, a.size, _ptr(a), _ptr(b))
    return b


def ntt_forward(p: int, omega: int, x, nthreads: int = 1) -> np.ndarray:
    """Algorithm 1 on the last axis: natural in, bit-reversed out, canonical."""
    x = _u64(x).copy()
    L = x.shape[-1]
    ell = L.bit_length() - 1
    assert L == 1 << ell
    batch = x.size // L if L else 0
    if batch == 1 and nthreads > 1 and ell >= 16:
        _load().orc_ntt_single_mt(p, omega, ell, _ptr(x), 0, nthreads)
    else:
        _load().orc_ntt_batch(p, omega, ell, _ptr(x), batch, 0, nthreads)
    return x


def ntt_inverse(p: int, omega: int, x, nthreads: int = 1) -> np.ndarray:
    """Algorithm 1 run backwards: bit-reversed in, natural out, unscaled (L*a)."""
    x = _u64(x).copy()
    L = x.shape[-1]
    ell = L.bit_length() - 1
    assert L == 1 << ell
    batch = x.size // L if L else 0
    if batch == 1 and nthreads > 1 and ell >= 16:
        _load().orc_ntt_single_mt(p, omega, ell, _ptr(x), 1, nthreads)
    else:
        _load().orc_ntt_batch(p, omega, ell, _ptr(x), batch, 1, nthreads)
    return x


def pointwise(p: int, a, b, scale_L: int = 0) -> np.ndarray:
    """c_k = a_k b_k (times L^{-1} when scale_L = L != 0) mod p."""
    a, b = _u64(a), _u64(b)
    assert a.shape == b.shape
    c = np.empty_like(a)
    _load().orc_pointwise(p, _ptr(a), _ptr(b), _ptr(c), a.size, scale_L)
    return c


def cyclic_conv_coeff(p: int, a, b, k: int) -> int:
    """c_k = sum_i a_i b_{(k-i) mod L} mod p (definition, one coefficient)."""
    a, b = _u64(a), _u64(b)
    return int(_load().orc_cyclic_conv_coeff(p, _ptr(a), _ptr(b), a.size, k))


def schoolbook_mod(p: int, a, b) -> np.ndarray:
    """Linear product mod p, len(a) + len(b) - 1 coefficients."""
    a, b = _u64(a), _u64(b)
    out = np.zeros(a.size + b.size - 1, dtype=np.uint64)
    _load().orc_schoolbook_mod(p, _ptr(a), a.size, _ptr(b), b.size, _ptr(out))
    return out


def poly_eval(p: int, a, x: int) -> int:
    """P:24 (evaluation form): a(x) mod p by Horner."""
    a = _u64(a)
    return int(_load().orc_poly_eval(p, _ptr(a), a.size, x))


def ntt_output_at(p: int, omega: int, a, j: int) -> int:
    """Algorithm 1 output position j (bit-reversed order) = a(omega^{rev(j)})."""
    a = _u64(a)
    ell = a.size.bit_length() - 1
    rj = int(format(j, f"0{ell}b")[::-1], 2) if ell else 0
    return poly_eval(p, a, powmod(omega, rj, p))


def bfly(alg: int, bb: int, p: int, W, Wp, X, Y, J: int = 0):
    """The paper's butterfly `alg` in {2,3,4,5} over beta = 2^bb, element-wise."""
    X = _u64(X)
    n = X.size
    W = np.broadcast_to(_u64(W), X.shape).copy()
    Wp = np.broadcast_to(_u64(Wp), X.shape).copy()
    Y = np.broadcast_to(_u64(Y), X.shape).copy()
    Xo, Yo = np.empty_like(X), np.empty_like(X)
    rc = _load().orc_bfly_batch(alg, bb, p, J, n, _ptr(W), _ptr(Wp), _ptr(X), _ptr(Y), _ptr(Xo), _ptr(Yo))
    if rc:
        raise ValueError(f"unknown butterfly algorithm {alg}")
    return Xo, Yo


def crt(residues, primes):
    """The plain definition behind F3 (RNS use): for each index, the unique integer x in
    [0, prod(primes)) with x = residues[k] mod primes[k], by the textbook CRT formula
    x = sum_k r_k M_k (M_k^{-1} mod p_k) mod M, M_k = M / p_k, in Python integers.
    Returns a list of Python ints."""
    M = 1
    for q in primes:
        M *= q
    terms = []
    for q in primes:
        Mk = M // q
        terms.append(Mk * pow(Mk % q, -1, q))
    cols = [np.asarray(r, dtype=np.uint64).reshape(-1) for r in residues]
    return [sum(int(c[i]) * t for c, t in zip(cols, terms)) % M for i in range(cols[0].size)]
