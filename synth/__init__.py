"""Seeded, counter-based synthetic input generator.

Shared by the tests, the oracle legs and bench.py; holds none of the NTT
arithmetic.  The CUDA library implements the SAME generator on the device
(``ntt_synth_uniform`` in ``paper_1205_2926_b200/csrc/synth.cu``) so that large
inputs (8 GiB for config C4) can be produced in HBM; ``tests/test_synth.py``
checks the two bit-for-bit.

Definition (reading 10 of DESIGN.md).  For a stream (seed, tensor_id) and a
global element index i, attempt a = 0, 1, 2, ...:

    key   = mix64(seed ^ (tensor_id * 0xD1B54A32D192ED03))
    draw  = mix64(key + (i * 64 + a) * 0x9E3779B97F4A7C15)        (mod 2^64)
    mix64 = SplitMix64 finaliser: z ^= z>>30; z *= 0xBF58476D1CE4E5B9;
                                  z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31

* uniform [0, p):  v = draw >> (64 - bitlen(p)); accept the first attempt with
  v < p (rejection, so unbiased); attempt 63 is taken as v mod p (probability
  < 2^-63, never observed).
* uniform [0, 2^k): v = draw(a=0) >> (64 - k).

Because every element depends only on (seed, tensor_id, i), any shard or
thread mapping regenerates identical data.
"""
from __future__ import annotations

import numpy as np

M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
TID_MUL = np.uint64(0xD1B54A32D192ED03)
MAX_ATTEMPTS = 64

# one seed per BASELINE.json config (0x12052926 xor config number)
SEED_BASE = 0x12052926


def config_seed(cfg: int) -> int:
    return SEED_BASE ^ cfg


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * M1
        z = z ^ (z >> np.uint64(27))
        z = z * M2
        z = z ^ (z >> np.uint64(31))
    return z


def _key(seed: int, tensor_id: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(tensor_id & 0xFFFFFFFFFFFFFFFF) * TID_MUL)
    return mix64(np.array([k], dtype=np.uint64))[0]


def draw(seed: int, tensor_id: int, idx: np.ndarray, attempt: int) -> np.ndarray:
    key = _key(seed, tensor_id)
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = idx * np.uint64(64) + np.uint64(attempt)
        return mix64(key + ctr * GOLDEN)


def uniform_mod(seed: int, tensor_id: int, start: int, count: int, p: int) -> np.ndarray:
    """Elements [start, start+count) of the uniform-[0,p) stream, as uint64."""
    bits = int(p).bit_length()
    shift = np.uint64(64 - bits)
    pu = np.uint64(p)
    idx = np.arange(start, start + count, dtype=np.uint64)
    out = np.empty(count, dtype=np.uint64)
    pending = np.arange(count)
    for a in range(MAX_ATTEMPTS):
        v = draw(seed, tensor_id, idx[pending], a) >> shift
        if a == MAX_ATTEMPTS - 1:
            out[pending] = v % pu
            break
        ok = v < pu
        out[pending[ok]] = v[ok]
        pending = pending[~ok]
        if pending.size == 0:
            break
    return out


def uniform_bits(seed: int, tensor_id: int, start: int, count: int, k: int) -> np.ndarray:
    """Elements [start, start+count) of the uniform-[0,2^k) stream, as uint64."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    return draw(seed, tensor_id, idx, 0) >> np.uint64(64 - k)
