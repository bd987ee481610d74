"""Multi-GPU partitioning of the NTT hot path.

* Batched configs (C2-C4): independent transforms shard over ranks with no data-path collective
  (`batch_shard`).
* One oversized transform (C5): a four-step split.  View the length-L transform as an N1 x N2 row-major
  matrix (N1 = 2^ell1).  Rank g of G holds the column shard c in [g N2/G, (g+1) N2/G) as an N1 x (N2/G)
  row-major matrix and runs
      ntt_fourstep_cols  (column NTTs of length N1 + twiddle omega^{c rev(r)}; stages 1..ell1 of Alg. 1,
                          P:27-46, re-associated)
      one all-to-all     (rank g sends rows [h N1/G, (h+1) N1/G) of its shard -- contiguous, no pack --
                          to rank h)
      ntt_fourstep_rows  (row NTTs of length N2 over the G received blocks, normalised)
  and ends with flat positions [g L/G, (g+1) L/G) of Algorithm 1's bit-reversed output.

The same split runs backwards (`FourStepInverse`): row inverse NTTs on the
rank's rows of the bit-reversed spectrum, scattered straight into the all-to-all send blocks
(`ntt_fourstep_rows_inv`), the all-to-all, then the inverse twiddle and column inverse NTTs
(`ntt_fourstep_cols_inv`), leaving the natural-order column shard of L*a.  `FourStepForwardContig` /
`FourStepInverseContig` take / return contiguous natural-order shards (rank g holds x[g L/G, (g+1) L/G))
at the cost of a second all-to-all and one block transpose (`ntt_block_transpose`).

`FourStepForwardP2P` fuses the all-to-all into the column pass (`ntt_fourstep_cols_p2p`): the last column
pass stores each row straight into the owning rank's receive buffer over NVLink (torch symmetric memory gives
the peer addresses and a stream-ordered cross-rank barrier), so no separate collective runs at all.

The collective is `torch.distributed.all_to_all_single` on the NCCL process group (gloo in CPU tests);
the compute steps are the CUDA kernels behind the C ABI (`Plan.fourstep_cols/rows`).  The layout
helpers below are pure host logic, shared by the product path and the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass


def batch_shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [start, start+count) of `total` independent transforms for `rank`."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class FourStepLayout:
    """Shapes of the distributed four-step split of a length-2^ell transform over `world` ranks."""
    ell: int
    ell1: int
    world: int

    def __post_init__(self):
        if self.world & (self.world - 1) or self.world < 1:
            raise ValueError("world must be a power of two")
        if not (0 < self.ell1 < self.ell):
            raise ValueError("need 0 < ell1 < ell")
        if self.N1 % self.world or self.N2 % self.world:
            raise ValueError("world must divide N1 and N2")

    @property
    def N1(self) -> int:
        return 1 << self.ell1

    @property
    def N2(self) -> int:
        return 1 << (self.ell - self.ell1)

    @property
    def L(self) -> int:
        return 1 << self.ell

    @property
    def local_width(self) -> int:          # columns per rank
        return self.N2 // self.world

    @property
    def rows_per_rank(self) -> int:        # rows owned after the exchange
        return self.N1 // self.world

    @property
    def shard_words(self) -> int:          # words per rank, before and after
        return self.L // self.world

    @property
    def block_words(self) -> int:          # words per all-to-all block
        return self.rows_per_rank * self.local_width

    def columns(self, rank: int) -> tuple[int, int]:
        """Global column range [c0, c1) held by `rank` before the exchange."""
        return rank * self.local_width, (rank + 1) * self.local_width

    def input_index(self, rank: int, r: int, c_local: int) -> int:
        """Global (natural-order) input index of local element (r, c_local) of `rank`'s shard."""
        return self.N2 * r + rank * self.local_width + c_local

    def output_range(self, rank: int) -> tuple[int, int]:
        """Flat positions of Algorithm 1's bit-reversed output held by `rank` after the rows pass."""
        return rank * self.shard_words, (rank + 1) * self.shard_words


def scatter_columns(x_flat, layout: FourStepLayout, rank: int):
    """Host helper: `rank`'s column shard (N1 x N2/G, row-major) of a full natural-order input."""
    c0, c1 = layout.columns(rank)
    return x_flat.reshape(layout.N1, layout.N2)[:, c0:c1].reshape(-1)


class FourStepForward:
    """Distributed forward NTT of one length-2^ell transform (config C5) on the calling rank.

    x_shard, recv, out: device tensors of layout.shard_words words each (recv/out may not alias x_shard).
    """

    def __init__(self, plan, layout: FourStepLayout, rank: int, group=None):
        self.plan, self.layout, self.rank, self.group = plan, layout, rank, group

    def cols(self, x_shard, stream=None):
        self.plan.fourstep_cols(self.layout.ell1, x_shard, self.rank, self.layout.world, stream=stream)

    def exchange(self, x_shard, recv):
        import torch.distributed as dist
        if self.layout.world == 1:
            recv.copy_(x_shard)
        else:
            dist.all_to_all_single(recv, x_shard, group=self.group)

    def rows(self, recv, out, stream=None):
        self.plan.fourstep_rows(self.layout.ell1, recv, out, self.rank, self.layout.world, stream=stream)

    def __call__(self, x_shard, recv, out, stream=None):
        self.cols(x_shard, stream)
        self.exchange(x_shard, recv)
        self.rows(recv, out, stream)
        return out


def _exchange(send, recv, world, group):
    import torch.distributed as dist
    if world == 1:
        recv.copy_(send)
    else:
        dist.all_to_all_single(recv, send, group=group)


class FourStepInverse:
    """Distributed inverse of FourStepForward: `rows` (this rank's N1/G rows of the bit-reversed spectrum,
    layout.shard_words words, left unmodified) -> `out` = natural-order column shard of L*a
    (N1 x N2/G row-major).  send: scratch of shard_words words."""

    def __init__(self, plan, layout: FourStepLayout, rank: int, group=None):
        self.plan, self.layout, self.rank, self.group = plan, layout, rank, group

    def rows_inv(self, rows, send, stream=None):
        self.plan.fourstep_rows_inv(self.layout.ell1, rows, send, self.rank, self.layout.world, stream=stream)

    def exchange(self, send, out):
        _exchange(send, out, self.layout.world, self.group)

    def cols_inv(self, out, stream=None):
        self.plan.fourstep_cols_inv(self.layout.ell1, out, self.rank, self.layout.world, stream=stream)

    def __call__(self, rows, send, out, stream=None):
        self.rows_inv(rows, send, stream)
        self.exchange(send, out)
        self.cols_inv(out, stream)
        return out


class FourStepForwardContig:
    """Forward NTT of one transform from a contiguous natural-order shard (rank g holds x[g L/G, (g+1) L/G),
    i.e. rows [g N1/G, (g+1) N1/G) of the N1 x N2 view) to the contiguous bit-reversed output shard:
    block-transpose pack, all-to-all (-> column shard), FourStepForward.  x is clobbered; buf: scratch."""

    def __init__(self, plan, layout: FourStepLayout, rank: int, group=None):
        self.fwd = FourStepForward(plan, layout, rank, group)
        self.layout = layout

    def __call__(self, x, buf, out, stream=None):
        from . import block_transpose
        lay = self.layout
        # rows x (G blocks of local_width) -> G blocks of (rows x local_width)
        block_transpose(buf, x, lay.rows_per_rank, lay.world, lay.local_width, stream=stream)
        _exchange(buf, x, lay.world, self.fwd.group)          # x <- column shard
        return self.fwd(x, buf, out, stream)


class FourStepInverseContig:
    """Inverse of FourStepForwardContig: contiguous bit-reversed shard in (unmodified) -> contiguous
    natural-order shard of L*a in `out`.  send, buf: scratch."""

    def __init__(self, plan, layout: FourStepLayout, rank: int, group=None):
        self.inv = FourStepInverse(plan, layout, rank, group)
        self.layout = layout

    def __call__(self, rows, send, buf, out, stream=None):
        from . import block_transpose
        lay = self.layout
        self.inv(rows, send, buf, stream)                      # buf <- natural column shard (N1 x Wl)
        _exchange(buf, send, lay.world, self.inv.group)        # block g = rows [rank R, ...) x cols of rank g
        # G blocks of (rows x local_width) -> rows x (G blocks of local_width)
        block_transpose(out, send, lay.world, lay.rows_per_rank, lay.local_width, stream=stream)
        return out


class _P2PRecv:
    """Receive buffers of a fused (peer-memory) exchange, double-buffered across calls.

    Call k stores into buffer k mod 2 of every peer.  A rank can only reach the stores of call k+2
    after the stream-ordered barrier of call k+1, which every peer enters after enqueueing its own
    consumer of call k (rows / cols_inv) on the same stream, so a fast rank never overwrites a buffer
    a slow peer is still reading (write-after-read across calls).  With a symmetric-memory handle the
    two buffers are the halves of one rendezvoused allocation.  Virtual-rank tests pass `recv` (one
    tensor, or a pair) and `peer_ptrs` (one list of addresses, or a pair of lists) directly."""

    def __init__(self, plan, layout, group, recv, peer_ptrs, dtype):
        self.hdl = None
        if recv is None:
            import torch
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm
            dt = dtype or (torch.uint64 if plan.word_bytes == 8 else torch.uint32)
            n = layout.shard_words
            buf = symm.empty(2 * n, dtype=dt, device=torch.device("cuda", torch.cuda.current_device()))
            self.hdl = symm.rendezvous(buf, group or dist.group.WORLD)
            base = list(self.hdl.buffer_ptrs)
            self.bufs = [buf[:n], buf[n:]]
            self.ptr_sets = [base, [b + n * plan.word_bytes for b in base]]
        elif isinstance(recv, (list, tuple)):
            self.bufs = list(recv)
            self.ptr_sets = [list(pp) for pp in peer_ptrs]
        else:
            self.bufs = [recv]
            self.ptr_sets = [list(peer_ptrs)]
        assert len(self.bufs) == len(self.ptr_sets)
        self.calls = 0
        self.cur = 0

    def next(self):
        """Buffer index of the next call (the producer side of the exchange)."""
        self.cur = self.calls % len(self.bufs)
        self.calls += 1
        return self.cur

    def barrier(self, stream):
        """Cross-rank barrier, enqueued on `stream` (the kernels' stream), after this rank's stores."""
        if self.hdl is None:
            return
        import torch
        if stream is None:
            self.hdl.barrier(channel=0)
        else:
            s = torch.cuda.ExternalStream(stream) if isinstance(stream, int) else stream
            with torch.cuda.stream(s):
                self.hdl.barrier(channel=0)


class FourStepForwardP2P:
    """FourStepForward with the all-to-all fused into the column pass over peer memory.

    The receive buffers are a symmetric-memory allocation (torch.distributed._symmetric_memory) rendezvoused
    on `group`, double-buffered across calls (_P2PRecv).  One call: ntt_fourstep_cols_p2p (column NTTs +
    twiddle, rows stored into the peers' current buffer), a symmetric-memory barrier on the same stream,
    ntt_fourstep_rows.  `recv`/`peer_ptrs` may be passed in directly (tests run G virtual ranks on one GPU
    with ordinary buffers and no barrier)."""

    def __init__(self, plan, layout: FourStepLayout, rank: int, group=None, recv=None, peer_ptrs=None, dtype=None):
        self.plan, self.layout, self.rank, self.group = plan, layout, rank, group
        self._rx = _P2PRecv(plan, layout, group, recv, peer_ptrs, dtype)
        self.hdl = self._rx.hdl

    @property
    def recv(self):
        return self._rx.bufs[self._rx.cur]

    @property
    def peer_ptrs(self):
        return self._rx.ptr_sets[self._rx.cur]

    def cols_exchange(self, x_shard, stream=None):
        i = self._rx.next()
        self.plan.fourstep_cols_p2p(self.layout.ell1, x_shard, self._rx.ptr_sets[i], self.rank, self.layout.world,
                                    stream=stream)
        self._rx.barrier(stream)  # every rank's stores into this buffer are visible

    def rows(self, out, stream=None):
        self.plan.fourstep_rows(self.layout.ell1, self.recv, out, self.rank, self.layout.world, stream=stream)

    def __call__(self, x_shard, out, stream=None):
        self.cols_exchange(x_shard, stream)
        self.rows(out, stream)
        return out


class FourStepInverseP2P:
    """FourStepInverse with the all-to-all fused into the row pass (ntt_fourstep_rows_inv_p2p): each row's
    natural-order inverse is scattered straight into the owning ranks' current receive buffer over NVLink
    (double-buffered across calls, _P2PRecv), a symmetric-memory barrier on the same stream, then
    ntt_fourstep_cols_inv on this rank's buffer, which ends as the natural-order column shard of L*a.
    The returned buffer stays valid until the call after next.  `recv`/`peer_ptrs` may be passed in
    (virtual-rank tests)."""

    def __init__(self, plan, layout: FourStepLayout, rank: int, group=None, recv=None, peer_ptrs=None, dtype=None):
        self.plan, self.layout, self.rank = plan, layout, rank
        self._rx = _P2PRecv(plan, layout, group, recv, peer_ptrs, dtype)
        self.hdl = self._rx.hdl

    @property
    def recv(self):
        return self._rx.bufs[self._rx.cur]

    @property
    def peer_ptrs(self):
        return self._rx.ptr_sets[self._rx.cur]

    def rows_exchange(self, rows, stream=None):
        i = self._rx.next()
        self.plan.fourstep_rows_inv_p2p(self.layout.ell1, rows, self._rx.ptr_sets[i], self.rank, self.layout.world,
                                        stream=stream)
        self._rx.barrier(stream)

    def cols_inv(self, stream=None):
        self.plan.fourstep_cols_inv(self.layout.ell1, self.recv, self.rank, self.layout.world, stream=stream)

    def __call__(self, rows, stream=None):
        """Returns the current receive buffer, which then holds the natural-order column shard of L*a."""
        self.rows_exchange(rows, stream)
        self.cols_inv(stream)
        return self.recv
