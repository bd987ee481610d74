"""Break down the latency of a single small transform (config C1): event overhead, an empty torch
kernel, the C1 forward with and without an L2 flush before it."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1205_2926_b200 as ntt  # noqa: E402

p, ell = 998244353, 10
plan = ntt.Plan(p, pow(3, (p - 1) >> ell, p), ell, 32)
x = torch.empty(1 << ell, dtype=torch.uint32, device="cuda")
ntt.synth_uniform(x, 1, 0, bound=p)
y = torch.empty(1, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def t(fn, pre=None, reps=50):
    out = []
    for _ in range(reps + 3):
        if pre:
            pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3)
    return round(statistics.median(out[3:]), 2)


print({"events_only_us": t(lambda: None), "empty_torch_kernel_us": t(lambda: y.add_(1)),
       "c1_fwd_warm_us": t(lambda: plan.forward(x)), "c1_fwd_after_l2_flush_us": t(lambda: plan.forward(x), flush.zero_),
       "c1_fwd_x10_warm_us_each": t(lambda: [plan.forward(x) for _ in range(10)]) / 10})
