"""Out-of-bounds write detection for every entry point, without a sanitizer.

compute-sanitizer is not available on the GPU pool, so each call runs on views placed inside
larger allocations whose guard words (both sides, 32 KiB each) hold a byte sentinel.  After the
call the guards must be intact, and the result must equal the same call on a fresh tensor (the
parity tests pin that result to the oracle).  Shapes cover each kernel family -- the persistent
TMA kernel and its latency variant, the 2-CTA cluster kernel (forward, inverse, fused pointwise),
two- and three-pass four-step schedules, the four-step halves of the multi-GPU path -- with ragged
batches (not multiples of the SM or cluster count).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from gpu_util import P30, P62, P62G, RNS, root  # noqa: E402

GUARD_BYTES = 32 * 1024
SENT = 0xA5


@pytest.fixture(scope="module")
def ntt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1205_2926_b200 as P
    return P


def _dt(bits):
    return torch.uint64 if bits == 64 else torch.uint32


def _ival(t):
    return t.view(torch.int64 if t.element_size() == 8 else torch.int32)


class Guarded:
    """n words of dtype inside a sentinel-filled allocation."""

    def __init__(self, n, dtype):
        wb = torch.empty(0, dtype=dtype).element_size()
        self.g = GUARD_BYTES // wb
        self.raw = torch.full((n * wb + 2 * GUARD_BYTES,), SENT, dtype=torch.uint8, device="cuda")
        self.all = self.raw.view(dtype)
        self.t = self.all[self.g:self.g + n]

    def check(self, what):
        torch.cuda.synchronize()
        b = self.raw
        lo, hi = b[:GUARD_BYTES], b[b.numel() - GUARD_BYTES:]
        assert bool((lo == SENT).all()), f"{what}: write below the buffer"
        assert bool((hi == SENT).all()), f"{what}: write past the end of the buffer"


def _fill(ntt, x, p, tid):
    ntt.synth_uniform(x, synth.config_seed(2), tid, bound=p)


@pytest.mark.parametrize("p,bits,ell,batch", [
    (P30, 32, 1, 5), (P30, 32, 4, 37), (P30, 32, 10, 37), (P30, 32, 12, 149), (P30, 32, 14, 3), (P30, 32, 15, 3),
    (P62, 64, 1, 5), (P62, 64, 5, 37), (P62, 64, 12, 150), (P62, 64, 14, 3),
    (P30, 32, 16, 3), (P30, 32, 16, 75), (P62, 64, 15, 3), (P62, 64, 15, 77),
    (RNS[0], 32, 17, 2), (RNS[1], 32, 20, 1), (P62, 64, 16, 2), (P62, 64, 18, 1), (P62, 64, 21, 1),
    (P62G, 64, 13, 5), (P62G, 64, 15, 3), (P62, 64, 25, 1),
])
def test_forward_inverse_stay_in_bounds(ntt, p, bits, ell, batch):
    L = 1 << ell
    plan = ntt.Plan(p, root(p, L), ell, bits)
    g = Guarded(batch * L, _dt(bits))
    _fill(ntt, g.t, p, 1)
    ref = g.t.clone()
    plan.forward(g.t)
    g.check("forward")
    plan.forward(ref)
    assert torch.equal(_ival(g.t), _ival(ref)), "forward result depends on the buffer's surroundings"
    plan.inverse(g.t)
    g.check("inverse")
    plan.inverse(ref)
    assert torch.equal(_ival(g.t), _ival(ref))


@pytest.mark.parametrize("p,bits,ell,batch", [(P30, 32, 16, 3), (P30, 32, 10, 37), (P62, 64, 12, 5),
                                               (P62, 64, 15, 3), (P30, 32, 18, 1)])
def test_pointwise_and_convolution_stay_in_bounds(ntt, p, bits, ell, batch):
    L = 1 << ell
    plan = ntt.Plan(p, root(p, L), ell, bits)
    dt = _dt(bits)
    a, b, c = Guarded(batch * L, dt), Guarded(batch * L, dt), Guarded(batch * L, dt)
    _fill(ntt, a.t, p, 2)
    _fill(ntt, b.t, p, 3)
    a0, b0 = a.t.clone(), b.t.clone()
    plan.pointwise_mul(c.t, a.t, b.t, scale_inv_L=True)
    for gb, w in ((a, "a"), (b, "b"), (c, "c")):
        gb.check(f"pointwise ({w})")
    ref = torch.empty_like(a0)
    plan.pointwise_mul(ref, a0, b0, scale_inv_L=True)
    assert torch.equal(_ival(c.t), _ival(ref))
    plan.cyclic_convolve(a.t, b.t)
    a.check("cyclic_convolve (a)")
    b.check("cyclic_convolve (b)")
    plan.cyclic_convolve(a0, b0)
    assert torch.equal(_ival(a.t), _ival(a0))


def test_crt3_and_block_transpose_stay_in_bounds(ntt):
    n = 3 * 4096 + 17
    rs = []
    for i, q in enumerate(RNS):
        r = torch.empty(n, dtype=torch.uint32, device="cuda")
        ntt.synth_uniform(r, 9, i, bound=q)
        rs.append(r)
    out = Guarded(2 * n, torch.uint64)
    ntt.crt3(out.t, *rs, RNS)
    out.check("crt3")
    ref = torch.empty(2 * n, dtype=torch.uint64, device="cuda")
    ntt.crt3(ref, *rs, RNS)
    assert torch.equal(_ival(out.t), _ival(ref))
    for wb, dt in ((4, torch.uint32), (8, torch.uint64)):
        n0, n1, n2 = 6, 5, 96
        src = torch.empty(n0 * n1 * n2, dtype=dt, device="cuda")
        ntt.synth_uniform(src, 9, 7, bits=8 * wb)
        dst = Guarded(src.numel(), dt)
        ntt.block_transpose(dst.t, src, n0, n1, n2)
        dst.check(f"block_transpose u{8 * wb}")
        want = src.view(n0, n1, n2).transpose(0, 1).contiguous().view(-1)
        assert torch.equal(_ival(dst.t), _ival(want))


@pytest.mark.parametrize("p,bits,ell,ell1,G", [(P62, 64, 16, 8, 2), (P30, 32, 16, 8, 2), (P62, 64, 20, 10, 4)])
def test_fourstep_halves_stay_in_bounds(ntt, p, bits, ell, ell1, G):
    """ntt_fourstep_cols / _rows (forward) and _rows_inv / _cols_inv on guarded shards."""
    from paper_1205_2926_b200.dist import FourStepLayout
    lay = FourStepLayout(ell, ell1, G)
    L, N1, N2, Wl, R = lay.L, lay.N1, lay.N2, lay.local_width, lay.rows_per_rank
    plan = ntt.Plan(p, root(p, L), ell, bits)
    dt = _dt(bits)
    x = torch.empty(L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(5), 6, bound=p)
    ref = x.clone()
    plan.forward(ref)
    shards = []
    for g in range(G):
        s = Guarded(lay.shard_words, dt)
        s.t.copy_(x.view(N1, N2)[:, g * Wl:(g + 1) * Wl].reshape(-1))
        plan.fourstep_cols(ell1, s.t, g, G)
        s.check("fourstep_cols")
        shards.append(s)
    outs = []
    for h in range(G):
        recv = Guarded(lay.shard_words, dt)
        recv.t.copy_(torch.cat([shards[g].t.view(N1, Wl)[h * R:(h + 1) * R].reshape(-1) for g in range(G)]))
        out = Guarded(lay.shard_words, dt)
        plan.fourstep_rows(ell1, recv.t, out.t, h, G)
        recv.check("fourstep_rows (recv)")
        out.check("fourstep_rows (out)")
        outs.append(out)
    assert torch.equal(_ival(torch.cat([o.t for o in outs])), _ival(ref))
    # inverse halves on the row shards
    sends = []
    for h in range(G):
        send = Guarded(lay.shard_words, dt)
        plan.fourstep_rows_inv(ell1, outs[h].t, send.t, h, G)
        outs[h].check("fourstep_rows_inv (rows)")
        send.check("fourstep_rows_inv (send)")
        sends.append(send)
    n = lay.shard_words // G
    for g in range(G):
        recv = Guarded(lay.shard_words, dt)
        recv.t.copy_(torch.cat([sends[h].t[g * n:(g + 1) * n] for h in range(G)]))
        plan.fourstep_cols_inv(ell1, recv.t, g, G)
        recv.check("fourstep_cols_inv")
        want = (x.view(N1, N2)[:, g * Wl:(g + 1) * Wl].reshape(-1).cpu().numpy().astype(object) * L) % p
        assert np.array_equal(recv.t.cpu().numpy().astype(object), want)


def test_execute_host_stays_in_bounds(ntt):
    p, bits, ell, batch = P62, 64, 12, 37
    L = 1 << ell
    plan = ntt.Plan(p, root(p, L), ell, bits)
    x = torch.empty(batch * L, dtype=torch.uint64, device="cuda")
    ntt.synth_uniform(x, 3, 3, bound=p)
    host_in = x.cpu().pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    scratch = Guarded(8 * L + 3, torch.uint64)  # room for a few transforms, ragged
    plan.execute_host(ntt.NTT_OP_FORWARD | ntt.NTT_OP_INVERSE, host_in, host_out, scratch.t)
    scratch.check("execute_host scratch")
    ref = x.clone()
    plan.forward(ref)
    plan.inverse(ref)
    assert torch.equal(_ival(host_out.cuda()), _ival(ref))
