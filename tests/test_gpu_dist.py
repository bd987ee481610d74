"""The distributed four-step (config C5) on one GPU: G virtual ranks run the real kernels
(ntt_fourstep_cols / ntt_fourstep_rows) on their shards; the all-to-all is emulated by device copies
with exactly the layout of all_to_all_single (checked on gloo in test_dist_cpu.py).  The assembled
output must equal the single-GPU forward transform bit for bit (itself bit-exact vs the oracle)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P30 = 998244353
P62 = 29 * 2**57 + 1


@pytest.fixture(scope="module")
def ntt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1205_2926_b200 as P
    return P


@pytest.mark.parametrize("p,bits,ell,ell1,G", [
    (P62, 64, 12, 6, 2), (P62, 64, 12, 6, 4), (P62, 64, 16, 8, 4), (P30, 32, 16, 8, 2),
    (P62, 64, 20, 10, 8), (P62, 64, 28, 14, 8), (P62, 64, 28, 14, 2),
])
def test_fourstep_virtual_ranks(ntt, p, bits, ell, ell1, G):
    from paper_1205_2926_b200.dist import FourStepLayout
    import synth
    lay = FourStepLayout(ell, ell1, G)
    L, N1, N2, Wl, R = lay.L, lay.N1, lay.N2, lay.local_width, lay.rows_per_rank
    w = pow(3, (p - 1) // L, p)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(5), 0, bound=p)
    ref = x.clone()
    plan.forward(ref)
    shards = [x.view(N1, N2)[:, g * Wl:(g + 1) * Wl].contiguous().view(-1) for g in range(G)]
    del x
    for g in range(G):
        plan.fourstep_cols(ell1, shards[g], g, G)
    outs = []
    for h in range(G):  # all_to_all_single: rank h receives chunk h of every rank g, in rank order
        recv = torch.cat([shards[g].view(N1, Wl)[h * R:(h + 1) * R].reshape(-1) for g in range(G)])
        out = torch.empty(lay.shard_words, dtype=dt, device="cuda")
        plan.fourstep_rows(ell1, recv, out, h, G)
        outs.append(out)
        del recv
    got = torch.cat(outs)
    assert torch.equal(got.view(torch.int64 if bits == 64 else torch.int32),
                       ref.view(torch.int64 if bits == 64 else torch.int32))
