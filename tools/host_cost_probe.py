"""Host-side cost per call of the C1 path (one 2^10 u32 forward): the Python binding, the raw C-ABI
call through ctypes, and a no-op ctypes call.  python tools/host_cost_probe.py"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1205_2926_b200 as ntt  # noqa: E402


def per_call(fn, n=3000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t) / n * 1e6, (t2 - t) / n * 1e6


def main():
    p, ell = 998244353, 10
    plan = ntt.Plan(p, pow(3, (p - 1) >> ell, p), ell, 32)
    x = torch.empty(1 << ell, dtype=torch.uint32, device="cuda")
    ntt.synth_uniform(x, 1, 0, bound=p)
    lib = ntt.lib()
    h, ptr = plan.handle, ctypes.c_void_p(x.data_ptr())
    res = {
        "plan.forward": per_call(lambda: plan.forward(x)),
        "lib.ntt_forward (raw ctypes, default stream)": per_call(lambda: lib.ntt_forward(h, ptr, 1, None)),
        "lib.ntt_abi_version (ctypes no-op)": per_call(lambda: lib.ntt_abi_version()),
    }
    for k, (host, tot) in res.items():
        print(f"{k:48s} host {host:6.2f} us/call   incl. GPU {tot:6.2f} us/call")


if __name__ == "__main__":
    main()
