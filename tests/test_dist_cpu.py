"""Multi-process (gloo, world size 2, CPU) tests of the multi-GPU host logic.

The distributed four-step's layout and its collective (`paper_1205_2926_b200.dist`) run for real over
gloo; the two pass kernels are emulated here on the CPU from their documented semantics
(include/ntt_b200.h) with the oracle, and the assembled output shards must equal the oracle's single
transform.  Batch sharding must cover every transform exactly once.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

P62 = 29 * 2**57 + 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _bitrev(j, n):
    return int(format(j, f"0{n}b")[::-1], 2) if n else 0


def _emulated_cols(shard, layout, rank, p, w):
    """ntt_fourstep_cols semantics: length-N1 NTT (root w^N2) down each local column, then
    element (r, c) *= w^{c rev_ell1(r)} with c the global column."""
    import oracle
    N1, Wl = layout.N1, layout.local_width
    m = shard.reshape(N1, Wl).copy()
    wc = pow(w, layout.N2, p)
    c0, _ = layout.columns(rank)
    for cl in range(Wl):
        col = oracle.ntt_forward(p, wc, m[:, cl])
        for r in range(N1):
            col[r] = int(col[r]) * pow(w, (c0 + cl) * _bitrev(r, layout.ell1), p) % p
        m[:, cl] = col
    return m.reshape(-1)


def _emulated_rows(recv, layout, p, w):
    """ntt_fourstep_rows semantics: row r (local) = concat over h of block_h[r]; length-N2 NTT."""
    import oracle
    G, R, Wl = layout.world, layout.rows_per_rank, layout.local_width
    blocks = recv.reshape(G, R, Wl)
    rows = np.concatenate([blocks[h] for h in range(G)], axis=1)  # R x N2
    wr = pow(w, layout.N1, p)
    return oracle.ntt_forward(p, wr, rows).reshape(-1)


def _worker(rank, world, port, ell, ell1, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_1205_2926_b200.dist import FourStepForward, FourStepLayout, batch_shard, scatter_columns
    layout = FourStepLayout(ell, ell1, world)
    p = P62
    w = pow(3, (p - 1) // layout.L, p)
    x = synth.uniform_mod(synth.config_seed(5), 0, 0, layout.L, p)
    shard = scatter_columns(x, layout, rank)
    shard = _emulated_cols(shard, layout, rank, p, w)
    send = torch.from_numpy(shard.view(np.int64).copy())
    recv = torch.empty_like(send)
    FourStepForward(plan=None, layout=layout, rank=rank).exchange(send, recv)  # the product's collective
    out = _emulated_rows(recv.numpy().view(np.uint64), layout, p, w)
    np.save(os.path.join(out_dir, f"out{rank}.npy"), out)
    # batch sharding: every transform exactly once
    covered = torch.zeros(1000, dtype=torch.int64)
    s, n = batch_shard(1000, rank, world)
    covered[s:s + n] += 1
    dist.all_reduce(covered)
    np.save(os.path.join(out_dir, f"cov{rank}.npy"), covered.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("ell,ell1", [(10, 5), (11, 5)])
def test_fourstep_world2_gloo(tmp_path, ell, ell1):
    import oracle
    import synth
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), ell, ell1, str(tmp_path)), nprocs=world, join=True)
    L = 1 << ell
    p = P62
    w = pow(3, (p - 1) // L, p)
    x = synth.uniform_mod(synth.config_seed(5), 0, 0, L, p)
    ref = oracle.ntt_forward(p, w, x)
    from paper_1205_2926_b200.dist import FourStepLayout
    layout = FourStepLayout(ell, ell1, world)
    for g in range(world):
        a, b = layout.output_range(g)
        assert np.array_equal(np.load(tmp_path / f"out{g}.npy"), ref[a:b]), g
        assert (np.load(tmp_path / f"cov{g}.npy") == 1).all()


def _emulated_rows_inv(rows, layout, p, w):
    """ntt_fourstep_rows_inv semantics: inverse NTT (root w^{-N1}, unscaled) of each of the rank's rows,
    row r's column block h -> block h of the send buffer."""
    import oracle
    G, R, Wl, N2 = layout.world, layout.rows_per_rank, layout.local_width, layout.N2
    nat = oracle.ntt_inverse(p, pow(w, layout.N1, p), rows.reshape(R, N2))  # R x N2 natural
    return np.concatenate([nat[:, h * Wl:(h + 1) * Wl].reshape(-1) for h in range(G)])


def _emulated_cols_inv(shard, layout, rank, p, w):
    """ntt_fourstep_cols_inv semantics: (r, c) *= w^{-c rev(r)}, then inverse length-N1 NTTs down columns."""
    import oracle
    N1, Wl = layout.N1, layout.local_width
    m = shard.reshape(N1, Wl).copy()
    wi = pow(w, p - 2, p)
    c0, _ = layout.columns(rank)
    for cl in range(Wl):
        col = [int(m[r, cl]) * pow(wi, (c0 + cl) * _bitrev(r, layout.ell1), p) % p for r in range(N1)]
        m[:, cl] = oracle.ntt_inverse(p, pow(w, layout.N2, p), np.array(col, dtype=np.uint64))
    return m.reshape(-1)


def _worker_inv(rank, world, port, ell, ell1, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_1205_2926_b200.dist import FourStepInverse, FourStepLayout
    layout = FourStepLayout(ell, ell1, world)
    p = P62
    w = pow(3, (p - 1) // layout.L, p)
    x = synth.uniform_mod(synth.config_seed(5), 1, 0, layout.L, p)
    spec = oracle.ntt_forward(p, w, x)
    a, b = layout.output_range(rank)
    send = _emulated_rows_inv(spec[a:b], layout, p, w)
    st = torch.from_numpy(send.view(np.int64).copy())
    recv = torch.empty_like(st)
    FourStepInverse(plan=None, layout=layout, rank=rank).exchange(st, recv)  # the product's collective
    out = _emulated_cols_inv(recv.numpy().view(np.uint64), layout, rank, p, w)
    np.save(os.path.join(out_dir, f"inv{rank}.npy"), out)
    dist.destroy_process_group()


@pytest.mark.parametrize("ell,ell1", [(10, 5), (9, 4)])
def test_fourstep_inverse_world2_gloo(tmp_path, ell, ell1):
    """F4 layout: rows_inv -> all_to_all_single (gloo) -> cols_inv returns the column shards of L*x."""
    import synth
    from paper_1205_2926_b200.dist import FourStepLayout, scatter_columns
    world = 2
    mp.spawn(_worker_inv, args=(world, _free_port(), ell, ell1, str(tmp_path)), nprocs=world, join=True)
    layout = FourStepLayout(ell, ell1, world)
    p = P62
    x = synth.uniform_mod(synth.config_seed(5), 1, 0, layout.L, p)
    Lx = np.array([(int(v) * layout.L) % p for v in x], dtype=np.uint64)
    for g in range(world):
        assert np.array_equal(np.load(tmp_path / f"inv{g}.npy"), scatter_columns(Lx, layout, g)), g


def test_layout_helpers():
    from paper_1205_2926_b200.dist import FourStepLayout, batch_shard
    lay = FourStepLayout(28, 14, 8)
    assert lay.local_width == 2048 and lay.rows_per_rank == 2048 and lay.block_words == 2048 * 2048
    assert lay.shard_words * 8 == 1 << 28
    assert lay.columns(3) == (6144, 8192)
    assert lay.input_index(1, 2, 5) == 2 * 16384 + 2048 + 5
    assert [batch_shard(10, r, 4) for r in range(4)] == [(0, 3), (3, 3), (6, 2), (8, 2)]
    with pytest.raises(ValueError):
        FourStepLayout(10, 5, 3)
