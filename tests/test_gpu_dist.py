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


def _a2a(sends, G):
    """all_to_all_single emulation: rank h receives chunk h of every rank g, in rank order."""
    n = sends[0].numel() // G
    return [torch.cat([sends[g][h * n:(h + 1) * n] for g in range(G)]) for h in range(G)]


def _ieq(a, b, bits):
    dt = torch.int64 if bits == 64 else torch.int32
    return torch.equal(a.view(dt), b.view(dt))


@pytest.mark.parametrize("p,bits,ell,ell1,G", [
    (P62, 64, 12, 6, 2), (P62, 64, 16, 8, 4), (P30, 32, 16, 8, 2), (P62, 64, 20, 10, 8), (P62, 64, 28, 14, 8),
])
def test_fourstep_inverse_virtual_ranks(ntt, p, bits, ell, ell1, G):
    """F4: distributed inverse (rows_inv -> all-to-all -> cols_inv) of the single-GPU forward output
    gives the column shards of L*x, i.e. exactly ntt_inverse(ntt_forward(x)) resharded."""
    from paper_1205_2926_b200.dist import FourStepLayout
    import synth
    lay = FourStepLayout(ell, ell1, G)
    L, N1, N2, Wl = lay.L, lay.N1, lay.N2, lay.local_width
    w = pow(3, (p - 1) // L, p)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(5), 1, bound=p)
    spec = x.clone()
    plan.forward(spec)
    ref = spec.clone()
    plan.inverse(ref)  # = L*x, natural order (itself pinned vs the oracle in test_gpu_parity)
    rows = [spec[g * lay.shard_words:(g + 1) * lay.shard_words].clone() for g in range(G)]
    del spec
    sends = []
    for g in range(G):
        send = torch.empty(lay.shard_words, dtype=dt, device="cuda")
        keep = rows[g].clone()
        plan.fourstep_rows_inv(ell1, rows[g], send, g, G)
        assert _ieq(rows[g], keep, bits), "rows_inv must not modify its input"
        sends.append(send)
    del rows
    recvs = _a2a(sends, G)
    del sends
    for h in range(G):
        plan.fourstep_cols_inv(ell1, recvs[h], h, G)
        want = ref.view(N1, N2)[:, h * Wl:(h + 1) * Wl].contiguous().view(-1)
        assert _ieq(recvs[h], want, bits), h


@pytest.mark.parametrize("p,bits,ell,ell1,G", [(P62, 64, 16, 8, 4), (P30, 32, 16, 8, 2), (P62, 64, 24, 12, 8)])
def test_fourstep_contig_roundtrip_virtual_ranks(ntt, p, bits, ell, ell1, G):
    """F4: contiguous natural shards -> (pack, all-to-all, cols, all-to-all, rows) -> contiguous shards of
    Alg. 1's output, bit-exact vs ntt_forward; then back with the contiguous inverse to L*x."""
    from paper_1205_2926_b200.dist import FourStepLayout
    import synth
    lay = FourStepLayout(ell, ell1, G)
    L, R, Wl, S = lay.L, lay.rows_per_rank, lay.local_width, lay.shard_words
    w = pow(3, (p - 1) // L, p)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(5), 2, bound=p)
    spec_ref = x.clone()
    plan.forward(spec_ref)
    # forward, contiguous input: pack each rank's rows into send blocks
    bufs = [torch.empty(S, dtype=dt, device="cuda") for _ in range(G)]
    for g in range(G):
        ntt.block_transpose(bufs[g], x[g * S:(g + 1) * S], R, G, Wl)
    cols = _a2a(bufs, G)
    for g in range(G):
        plan.fourstep_cols(ell1, cols[g], g, G)
    recv = _a2a(cols, G)
    outs = []
    for g in range(G):
        o = torch.empty(S, dtype=dt, device="cuda")
        plan.fourstep_rows(ell1, recv[g], o, g, G)
        outs.append(o)
    assert _ieq(torch.cat(outs), spec_ref, bits)
    # inverse, contiguous output
    sends = []
    for g in range(G):
        s_ = torch.empty(S, dtype=dt, device="cuda")
        plan.fourstep_rows_inv(ell1, outs[g], s_, g, G)
        sends.append(s_)
    colsh = _a2a(sends, G)
    for g in range(G):
        plan.fourstep_cols_inv(ell1, colsh[g], g, G)
    back = _a2a(colsh, G)
    res = []
    for g in range(G):
        o = torch.empty(S, dtype=dt, device="cuda")
        ntt.block_transpose(o, back[g], G, R, Wl)
        res.append(o)
    got = torch.cat(res).cpu().numpy().astype(object)
    want = (x.cpu().numpy().astype(object) * L) % p
    assert (got == want).all()


def test_block_transpose(ntt):
    for dt, n0, n1, n2 in ((torch.uint64, 3, 5, 16), (torch.uint32, 4, 8, 32), (torch.uint64, 2, 3, 7),
                           (torch.uint32, 1, 1, 1)):
        src = torch.arange(n0 * n1 * n2, dtype=torch.int64, device="cuda").to(
            torch.int64 if dt == torch.uint64 else torch.int32)
        dst = torch.empty_like(src)
        ntt.block_transpose(dst, src, n0, n1, n2)
        assert torch.equal(dst.view(n1, n0, n2), src.view(n0, n1, n2).transpose(0, 1))


@pytest.mark.parametrize("p,bits,ell,ell1,G", [
    (P62, 64, 12, 6, 2), (P62, 64, 16, 8, 4), (P30, 32, 16, 8, 2), (P62, 64, 20, 10, 8), (P62, 64, 28, 14, 8),
    # one-round column passes (R == 1: u64 2^4, u32 2^4 / 2^5), whose prefetch is not behind a round barrier
    (P62, 64, 10, 4, 2), (P30, 32, 10, 4, 2), (P30, 32, 12, 5, 2),
])
def test_fourstep_p2p_virtual_ranks(ntt, p, bits, ell, ell1, G):
    """Fused column pass + all-to-all (ntt_fourstep_cols_p2p): G virtual ranks on one GPU whose 'peer'
    receive buffers are local; after all ranks' column passes, the row pass output equals ntt_forward."""
    from paper_1205_2926_b200.dist import FourStepForwardP2P, FourStepLayout
    import synth
    lay = FourStepLayout(ell, ell1, G)
    L, N1, N2, Wl = lay.L, lay.N1, lay.N2, lay.local_width
    w = pow(3, (p - 1) // L, p)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(5), 3, bound=p)
    ref = x.clone()
    plan.forward(ref)
    shards = [x.view(N1, N2)[:, g * Wl:(g + 1) * Wl].contiguous().view(-1) for g in range(G)]
    del x
    recvs = [torch.full((lay.shard_words,), 7, dtype=dt, device="cuda") for _ in range(G)]
    ptrs = [r.data_ptr() for r in recvs]
    ranks = [FourStepForwardP2P(plan, lay, g, recv=recvs[g], peer_ptrs=ptrs) for g in range(G)]
    for g in range(G):
        ranks[g].cols_exchange(shards[g])
    outs = []
    for g in range(G):
        o = torch.empty(lay.shard_words, dtype=dt, device="cuda")
        ranks[g].rows(o)
        outs.append(o)
    assert _ieq(torch.cat(outs), ref, bits)


def test_fourstep_p2p_symmetric_memory_world1(ntt):
    """The product's P2P plumbing (torch symmetric memory rendezvous, peer pointers, stream-ordered barrier)
    on a one-rank NCCL group: FourStepForwardP2P equals ntt_forward."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1205_2926_b200.dist import FourStepForwardP2P, FourStepLayout
    import synth
    if not dist.is_initialized():
        sck = socket.socket()
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
        sck.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        p, ell, ell1 = P62, 16, 8
        lay = FourStepLayout(ell, ell1, 1)
        plan = ntt.Plan(p, pow(3, (p - 1) >> ell, p), ell, 64)
        x = torch.empty(lay.L, dtype=torch.uint64, device="cuda")
        ntt.synth_uniform(x, synth.config_seed(5), 4, bound=p)
        ref = x.clone()
        plan.forward(ref)
        fs = FourStepForwardP2P(plan, lay, 0)
        out = torch.empty_like(x)
        fs(x.clone(), out)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int64), ref.view(torch.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p,bits,ell,ell1,G", [(P62, 64, 16, 8, 4), (P30, 32, 16, 8, 2), (P62, 64, 28, 14, 8)])
def test_fourstep_inverse_p2p_virtual_ranks(ntt, p, bits, ell, ell1, G):
    """Fused row inverse + all-to-all (ntt_fourstep_rows_inv_p2p) then cols_inv: column shards of L*x."""
    from paper_1205_2926_b200.dist import FourStepInverseP2P, FourStepLayout
    import synth
    lay = FourStepLayout(ell, ell1, G)
    L, N1, N2, Wl = lay.L, lay.N1, lay.N2, lay.local_width
    w = pow(3, (p - 1) // L, p)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(5), 5, bound=p)
    spec = x.clone()
    plan.forward(spec)
    ref = spec.clone()
    plan.inverse(ref)
    recvs = [torch.full((lay.shard_words,), 9, dtype=dt, device="cuda") for _ in range(G)]
    ptrs = [r.data_ptr() for r in recvs]
    ranks = [FourStepInverseP2P(plan, lay, g, recv=recvs[g], peer_ptrs=ptrs) for g in range(G)]
    for g in range(G):
        ranks[g].rows_exchange(spec[g * lay.shard_words:(g + 1) * lay.shard_words])
    for g in range(G):
        ranks[g].cols_inv()
        want = ref.view(N1, N2)[:, g * Wl:(g + 1) * Wl].contiguous().view(-1)
        assert _ieq(recvs[g], want, bits), g


@pytest.mark.parametrize("p,bits,ell,ell1,G", [(P62, 64, 16, 8, 2), (P30, 32, 16, 8, 4)])
def test_fourstep_p2p_calls_overlap_across_ranks(ntt, p, bits, ell, ell1, G):
    """Write-after-read across calls: rank 0's call k+1 (its stores into every peer's receive buffer) is
    enqueued before rank 1..G-1 read call k's data.  The double-buffered receive side (_P2PRecv) keeps
    both calls' results equal to ntt_forward; single-buffered, call k+1 would overwrite call k."""
    from paper_1205_2926_b200.dist import FourStepForwardP2P, FourStepLayout
    import synth
    lay = FourStepLayout(ell, ell1, G)
    L, N1, N2, Wl = lay.L, lay.N1, lay.N2, lay.local_width
    w = pow(3, (p - 1) // L, p)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    xs, refs = [], []
    for k in range(2):
        x = torch.empty(L, dtype=dt, device="cuda")
        ntt.synth_uniform(x, synth.config_seed(5), 10 + k, bound=p)
        r = x.clone()
        plan.forward(r)
        xs.append([x.view(N1, N2)[:, g * Wl:(g + 1) * Wl].contiguous().view(-1) for g in range(G)])
        refs.append(r)
    recvs = [[torch.full((lay.shard_words,), 7, dtype=dt, device="cuda") for _ in range(2)] for _ in range(G)]
    ptrs = [[recvs[g][i].data_ptr() for g in range(G)] for i in range(2)]
    ranks = [FourStepForwardP2P(plan, lay, g, recv=recvs[g], peer_ptrs=ptrs) for g in range(G)]
    outs = [[torch.empty(lay.shard_words, dtype=dt, device="cuda") for _ in range(G)] for _ in range(2)]
    for g in range(G):
        ranks[g].cols_exchange(xs[0][g])           # call 0, every rank
    ranks[0].rows(outs[0][0])
    ranks[0].cols_exchange(xs[1][0])               # rank 0 races ahead into call 1 ...
    for g in range(1, G):
        ranks[g].rows(outs[0][g])                  # ... before its peers read call 0
    for g in range(1, G):
        ranks[g].cols_exchange(xs[1][g])
    for g in range(G):
        ranks[g].rows(outs[1][g])
    for k in range(2):
        assert _ieq(torch.cat(outs[k]), refs[k], bits), k
