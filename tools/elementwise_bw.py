"""HBM roofline of the elementwise kernels (F3 CRT lift, A7 pointwise product): algorithmic bytes per
launch / CUDA-event time, against MEASURED_PEAKS.json's copy bandwidth.  Inputs larger than L2.
    python tools/elementwise_bw.py  -> one JSON object"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1205_2926_b200 as ntt  # noqa: E402

RNS = (469762049, 167772161, 998244353)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    return ms[len(ms) // 2]


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = float(peaks.get("hbm_gbs", 6550.0))
    out = {"peak_GBps": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    n = 1024 << 16  # C3's output: 1024 products of length 2^16
    rs = []
    for i, q in enumerate(RNS):
        r = torch.empty(n, dtype=torch.uint32, device="cuda")
        ntt.synth_uniform(r, 7, i, bound=q)
        rs.append(r)
    o = torch.empty(2 * n, dtype=torch.uint64, device="cuda")
    ms = timed(lambda: ntt.crt3(o, *rs, RNS))
    b = 3 * 4 * n + 16 * n
    out["crt3 (C3 output, 3 x u32 in, 128-bit out)"] = {"ms": ms, "bytes": b, "GBps": b / ms / 1e6,
                                                       "frac": b / ms / 1e6 / peak}
    for bits, p, ell, batch in ((64, 29 * 2**57 + 1, 12, 4096), (32, 998244353, 16, 1024)):
        L = 1 << ell
        plan = ntt.Plan(p, pow(3, (p - 1) >> ell, p), ell, bits)
        dt = torch.uint64 if bits == 64 else torch.uint32
        a = torch.empty(batch * L, dtype=dt, device="cuda")
        b_ = torch.empty_like(a)
        c = torch.empty_like(a)
        ntt.synth_uniform(a, 7, 5, bound=p)
        ntt.synth_uniform(b_, 7, 6, bound=p)
        ms = timed(lambda: plan.pointwise_mul(c, a, b_, scale_inv_L=True))
        nb = 3 * a.numel() * a.element_size()
        out[f"pointwise u{bits} {batch} x 2^{ell} (2 in, 1 out)"] = {"ms": ms, "bytes": nb, "GBps": nb / ms / 1e6,
                                                                      "frac": nb / ms / 1e6 / peak}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
