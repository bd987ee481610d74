"""CPU-only checks of the C ABI boundary: the library loads, exports every symbol the
header declares, and plan validation rejects what the paper's preconditions exclude
(validation happens before any device call, so it runs without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ntt():
    import paper_1205_2926_b200 as P
    return P


def header_functions():
    src = open(os.path.join(ROOT, "include", "ntt_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ntt_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(ntt):
    names = header_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(ntt.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(ntt.EXPORTED)


def test_abi_version_and_status_strings(ntt):
    lib = ntt.lib()
    assert lib.ntt_abi_version() == 1
    for s in range(-9, 1):
        assert lib.ntt_status_str(s)


def _create(ntt, p, w, ell, bits):
    h = ctypes.c_void_p()
    st = ntt.lib().ntt_plan_create(ctypes.byref(h), p, w, ell, bits, 0)
    return st, h


P30 = 998244353
P62 = 29 * 2**57 + 1


@pytest.mark.parametrize("p,w,ell,bits,want", [
    (998244354, 1, 1, 32, -2),             # even
    (998244351, 1, 1, 32, -2),             # odd composite (3 * 332748117)
    (3221225473, 5, 1, 32, -2),            # prime 3*2^30+1 >= beta/4 = 2^30 (Alg. 3 needs p < beta/4)
    ((1 << 62) + 135, 3, 1, 64, -2),       # p >= 2^62 = beta/4 for beta = 2^64
    (13, 3, 2, 32, -3),                    # 3^1 has order 3: not a primitive 4th root
    (13, 1, 2, 32, -3),                    # omega = 1 (the 3^((p-1)/L) rule fails for p = 13)
    (13, 5, 3, 32, -4),                    # 8 does not divide 12
    (P30, 3, 29, 32, -4),                  # ell > 28
    (P30, 3, 10, 16, -5),                  # beta = 2^16 unsupported
    (P30, P30 + 1, 10, 32, -3),            # omega >= p
])
def test_plan_validation(ntt, p, w, ell, bits, want):
    st, h = _create(ntt, p, w, ell, bits)
    assert st == want
    assert not h.value


def test_valid_plan_reaches_device(ntt):
    """A valid plan passes validation and only then needs the device (NTT_ERR_CUDA here if none)."""
    import torch
    st, h = _create(ntt, 13, 5, 2, 32)
    if torch.cuda.is_available():
        assert st == 0
        ntt.lib().ntt_plan_destroy(h)
    else:
        assert st == -6


def test_pointer_checks_without_device(ntt):
    lib = ntt.lib()
    assert lib.ntt_forward(None, None, 1, None) == -1
    assert lib.ntt_synth_uniform(None, 10, 3, 0, 0, 0, 7, 0, None) == -1


RNS = (469762049, 167772161, 998244353)


def test_crt3_validation_without_device(ntt):
    """ntt_crt3 (F3) checks its moduli and pointers before touching the device."""
    lib = ntt.lib()
    assert lib.ntt_crt3(None, None, None, None, 0, *RNS, None) == 0               # n = 0: no-op
    assert lib.ntt_crt3(None, None, None, None, 5, *RNS, None) == -1              # null buffers
    assert lib.ntt_crt3(None, None, None, None, 5, RNS[0], RNS[0], RNS[2], None) == -2  # equal primes
    assert lib.ntt_crt3(None, None, None, None, 5, 998244351, RNS[1], RNS[2], None) == -2  # composite
    assert lib.ntt_crt3(None, None, None, None, 5, 3221225473, RNS[1], RNS[2], None) == -2  # >= 2^30


def test_block_transpose_validation_without_device(ntt):
    lib = ntt.lib()
    assert lib.ntt_block_transpose(None, None, 0, 4, 4, 8, None) == 0     # empty: no-op
    assert lib.ntt_block_transpose(None, None, 2, 4, 4, 8, None) == -1    # null buffers
    assert lib.ntt_block_transpose(16, 32, 2, 4, 4, 3, None) == -1        # word size
    assert lib.ntt_block_transpose(16, 16, 2, 4, 4, 8, None) == -1        # aliasing
    assert lib.ntt_block_transpose(16, 40, 2, 4, 4, 8, None) == -1        # misaligned source


def test_fourstep_entry_points_reject_null_plan(ntt):
    lib = ntt.lib()
    assert lib.ntt_fourstep_cols_inv(None, 7, None, 0, 2, None) == -1
    assert lib.ntt_fourstep_rows_inv(None, 7, None, None, 0, 2, None) == -1


def test_audit_build_exports_and_production_refuses(ntt):
    """The range-audit debug build exports the same ABI; the production build has no audit counters."""
    audit = os.path.join(ROOT, "paper_1205_2926_b200", "libntt_b200_audit.so")
    assert os.path.exists(audit)
    lib = ctypes.CDLL(audit)
    for n in header_functions():
        assert hasattr(lib, n), n
    lib.ntt_build_flags.restype = ctypes.c_uint
    assert lib.ntt_build_flags() & 1
    prod = ntt.lib()
    assert prod.ntt_build_flags() == 0
    v = ctypes.c_uint64(7)
    assert prod.ntt_audit_counts(0, ctypes.byref(v)) == -8 and v.value == 0
    assert prod.ntt_audit_reset(0, 0) == -8
