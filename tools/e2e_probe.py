"""PCIe / end-to-end probe for config C2: pinned H2D and D2H bandwidth alone and concurrent, and
ntt_execute_host (fwd+inv) at several device-buffer sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1205_2926_b200 as ntt  # noqa: E402

p, ell, batch = 29 * 2**57 + 1, 12, 4096
L = 1 << ell
n = batch * L
plan = ntt.Plan(p, pow(3, (p - 1) >> ell, p), ell, 64)
h_in = torch.empty(n, dtype=torch.uint64, pin_memory=True)
h_in.view(torch.int64).random_(0, p)
h_out = torch.empty_like(h_in).pin_memory()
d = torch.empty(n, dtype=torch.uint64, device="cuda")
s = torch.cuda.current_stream()
s2 = torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


nb = n * 8
res = {}
res["h2d_GBps"] = nb / timed(lambda: d.copy_(h_in, non_blocking=True)) / 1e6
res["d2h_GBps"] = nb / timed(lambda: h_out.copy_(d, non_blocking=True)) / 1e6
d2 = torch.empty_like(d)


def both():
    ev = torch.cuda.Event()
    ev.record(s)
    s2.wait_event(ev)
    d.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d2, non_blocking=True)
    ev2 = torch.cuda.Event()
    ev2.record(s2)
    s.wait_event(ev2)


res["concurrent_each_GBps"] = nb / timed(both) / 1e6
for mb in (32, 64, 128, 256):
    buf = torch.empty(mb << 17, dtype=torch.uint64, device="cuda")
    ms = timed(lambda: plan.execute_host(ntt.NTT_OP_FORWARD | ntt.NTT_OP_INVERSE, h_in, h_out, buf))
    res[f"execute_host_{mb}MiB_ms"] = round(ms, 3)
print({k: round(v, 2) for k, v in res.items()})

# pure-copy pipeline with the same chunking as ntt_execute_host (3 streams, 12 chunks): the PCIe floor
streams = [torch.cuda.Stream() for _ in range(3)]
chunks = 12
cw = n // chunks
bufs = [torch.empty(cw, dtype=torch.uint64, device="cuda") for _ in range(3)]


def pipe():
    ev = torch.cuda.Event()
    ev.record(s)
    for st in streams:
        st.wait_event(ev)
    for k in range(chunks):
        st = streams[k % 3]
        with torch.cuda.stream(st):
            bufs[k % 3].copy_(h_in[k * cw:(k + 1) * cw], non_blocking=True)
            h_out[k * cw:(k + 1) * cw].copy_(bufs[k % 3], non_blocking=True)
    for st in streams:
        e = torch.cuda.Event()
        e.record(st)
        s.wait_event(e)


print({"copy_only_pipeline_ms": round(timed(pipe), 3)})

# role-split pipeline: one H2D stream, one D2H stream, a ring of NB buffers (copies only)
def role_pipe(nb, chunks):
    cw = n // chunks
    ring = [torch.empty(cw, dtype=torch.uint64, device="cuda") for _ in range(nb)]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    freed = [None] * nb

    def run():
        ev = torch.cuda.Event()
        ev.record(s)
        h2d_s.wait_event(ev)
        d2h_s.wait_event(ev)
        for k in range(chunks):
            b = k % nb
            if freed[b] is not None:
                h2d_s.wait_event(freed[b])
            with torch.cuda.stream(h2d_s):
                ring[b].copy_(h_in[k * cw:(k + 1) * cw], non_blocking=True)
            loaded = torch.cuda.Event()
            loaded.record(h2d_s)
            d2h_s.wait_event(loaded)
            with torch.cuda.stream(d2h_s):
                h_out[k * cw:(k + 1) * cw].copy_(ring[b], non_blocking=True)
            fe = torch.cuda.Event()
            fe.record(d2h_s)
            freed[b] = fe
        e = torch.cuda.Event()
        e.record(d2h_s)
        s.wait_event(e)
    return run


for nb, ch in ((4, 16),):
    print({f"role_pipe_nb{nb}_ch{ch}_ms": round(timed(role_pipe(nb, ch)), 3)})
