"""F1/F2: the transform with Algorithm 2 (NTL) or Algorithm 5 (Montgomery)
butterflies is bit-exact against the oracle, like the Algorithm 3 product path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from gpu_util import P30, P62, rand_residues, root, to_dev, to_host  # noqa: E402


@pytest.fixture(scope="module")
def ntt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1205_2926_b200 as P
    return P


@pytest.mark.parametrize("alg", [2, 5, 3])
@pytest.mark.parametrize("p,bits,ell", [(P62, 64, 12), (P62, 64, 8), (P62, 64, 11), (P30, 32, 10), (P30, 32, 14),
                                        (167772161, 32, 12), (2305843009146585089, 64, 12)])
def test_forward_butterfly_variants(ntt, alg, p, bits, ell):
    L = 1 << ell
    if (p - 1) % L:
        pytest.skip("p != 1 mod L")
    w = pow(3, (p - 1) // L, p) if pow(pow(3, (p - 1) // L, p), L // 2, p) == p - 1 else None
    if w is None:
        pytest.skip("3 is not a generator for this p")
    plan = ntt.Plan(p, w, ell, bits, butterfly=alg)
    x = rand_residues(np.random.default_rng(alg * 100 + ell), p, (5, L))  # canonical (Alg. 2 input range)
    d = to_dev(x, bits)
    plan.forward(d)
    assert np.array_equal(to_host(d), oracle.ntt_forward(p, w, x))
    plan.inverse(d)  # Algorithm 4 regardless of the forward butterfly
    assert np.array_equal(to_host(d), ((x.astype(object) * L) % p).astype(np.uint64))


def test_unsupported_combinations(ntt):
    p, ell = P62, 16  # multi-pass: ablation butterflies only on the on-chip kernel
    plan = ntt.Plan(p, root(p, 1 << ell), ell, 64, butterfly=2)
    d = torch.zeros(1 << ell, dtype=torch.uint64, device="cuda")
    with pytest.raises(ntt.NttError):
        plan.forward(d)
