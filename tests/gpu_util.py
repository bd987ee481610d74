"""Helpers for the GPU parity tests: numpy <-> device tensors, config constants."""
import numpy as np

P30 = 998244353                    # 119*2^23 + 1 (configs C1, C3)
P62 = 29 * 2**57 + 1               # configs C2, C4, C5
RNS = (469762049, 167772161, 998244353)
P62G = 2305843009146585089        # 62-bit, 2^24 | p-1, p != 1 mod 2^32: exercises the generic u64 Shoup tail


def root(p, L):
    """omega = 3^((p-1)/L), the BASELINE.json rule (reading 1)."""
    return pow(3, (p - 1) // L, p)


def word_dtype(log2_beta):
    return np.uint64 if log2_beta == 64 else np.uint32


def to_dev(a, log2_beta):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=word_dtype(log2_beta))).cuda()


def to_host(t):
    return t.cpu().numpy().astype(np.uint64)


def rand_residues(rng, p, shape, bound=None):
    hi = bound if bound is not None else p
    return rng.integers(0, hi, size=shape, dtype=np.uint64)


def bitrev(j, ell):
    return int(format(j, f"0{ell}b")[::-1], 2) if ell else 0
