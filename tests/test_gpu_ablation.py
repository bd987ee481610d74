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
                                        (167772161, 32, 12), (2305843009146585089, 64, 12),
                                        # 2-CTA cluster sizes (k_splitk), multi-pass u64 (k_cols_tma + row pass):
                                        # direct-level [8, 8], matrix level 2^20 [9, 11], generic-p 2^18
                                        (P30, 32, 16), (P62, 64, 15), (P62, 64, 16), (P62, 64, 20),
                                        (2305843009146585089, 64, 18), (2305843009146585089, 64, 15)])
def test_forward_butterfly_variants(ntt, alg, p, bits, ell):
    L = 1 << ell
    if (p - 1) % L:
        pytest.skip("p != 1 mod L")
    w = pow(3, (p - 1) // L, p) if pow(pow(3, (p - 1) // L, p), L // 2, p) == p - 1 else None
    if w is None:
        pytest.skip("3 is not a generator for this p")
    plan = ntt.Plan(p, w, ell, bits, butterfly=alg)
    x = rand_residues(np.random.default_rng(alg * 100 + ell), p, (5 if ell <= 16 else 2, L))  # canonical (Alg. 2)
    d = to_dev(x, bits)
    plan.forward(d)
    assert np.array_equal(to_host(d), oracle.ntt_forward(p, w, x, nthreads=oracle.default_threads()))
    plan.inverse(d)  # Algorithm 4 regardless of the forward butterfly
    assert np.array_equal(to_host(d), ((x.astype(object) * L) % p).astype(np.uint64))


def test_unsupported_combinations(ntt):
    # beta = 2^32 multi-pass and lengths below the TMA kernels' 2^8: no ablation kernels
    for p, bits, ell, dt in ((P30, 32, 17, torch.uint32), (P62, 64, 6, torch.uint64)):
        plan = ntt.Plan(p, root(p, 1 << ell), ell, bits, butterfly=5)
        d = torch.zeros(1 << ell, dtype=dt, device="cuda")
        with pytest.raises(ntt.NttError):
            plan.forward(d)


@pytest.mark.parametrize("alg", [2, 5])
@pytest.mark.parametrize("ell,batch", [(24, 2), (28, 1)])
def test_ablation_config_shapes(ntt, alg, ell, batch):
    """F1/F2 at the C4 (2^24: column pass with the twiddle matrix, 2^15 cluster row pass) and C5
    (2^28: factored column passes, 2^12 row pass) shapes: the Algorithm 2 / 5 forward equals the
    Algorithm 3 forward (canonical outputs are unique), which the parity tests pin to the oracle;
    sampled outputs also against the oracle's evaluation form."""
    import synth
    p = P62
    L = 1 << ell
    w = root(p, L)
    x = torch.empty(batch * L, dtype=torch.uint64, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(4), 9, bound=p)
    ref = x.clone()
    ntt.Plan(p, w, ell, 64).forward(ref)
    got = x.clone()
    ntt.Plan(p, w, ell, 64, butterfly=alg).forward(got)
    assert torch.equal(got.view(torch.int64), ref.view(torch.int64))
    xh = to_host(x[:L])
    gh = to_host(got[:L])
    for j in (0, 1, L - 1, 777777):
        assert int(gh[j]) == oracle.ntt_output_at(p, w, xh, j)
