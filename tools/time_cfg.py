"""Time the transforms of one bench config with CUDA events (median of reps, L2 flushed
between reps) through the library named by NTT_B200_LIB (default: the in-tree build).
    NTT_B200_LIB=variants/libntt_X.so python tools/time_cfg.py c2 [reps] [--check]
--check compares one forward against the default library's... no: against the oracle on 2 transforms."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1205_2926_b200 as ntt  # noqa: E402
from bench import CONFIGS, butterflies, root  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 20
    if key.startswith("x:"):  # x:p:bits:ell:batch[:ops]  custom shape, e.g. x:998244353:32:14:4096:fwd
        f = key.split(":")
        cfg = dict(primes=(int(f[1]),), bits=int(f[2]), ell=int(f[3]), batch=int(f[4]),
                   ops=tuple((f[5] if len(f) > 5 else "fwd,inv").split(",")), key=key)
    else:
        cfg = dict(CONFIGS[key], key=key)
    L = 1 << cfg["ell"]
    dt = torch.uint64 if cfg["bits"] == 64 else torch.uint32
    plans = [ntt.Plan(p, root(p, L), cfg["ell"], cfg["bits"]) for p in cfg["primes"]]
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {"lib": os.path.basename(ntt.LIB_PATH), "config": key}
    if cfg["ops"] == ("conv",):
        a = torch.zeros(cfg["batch"], L, dtype=dt, device="cuda")
        b = torch.zeros_like(a)
        ntt.synth_uniform(a[:, : L // 2].contiguous(), 1, 0, bits=20)
        work = [(a.clone(), b.clone()) for _ in plans]
        fns = {"conv": lambda: [pl.cyclic_convolve(x, y) for pl, (x, y) in zip(plans, work)]}
    else:
        x = torch.empty(cfg["batch"] * L, dtype=dt, device="cuda")
        ntt.synth_uniform(x, 1, 0, bound=cfg["primes"][0])
        fns = {op: (lambda op=op: (plans[0].forward if op == "fwd" else plans[0].inverse)(x)) for op in cfg["ops"]}
    for name, fn in fns.items():
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        n_ops = len(cfg["ops"]) if cfg["ops"] != ("conv",) else 1
        res[name] = {"ms": round(ms, 4), "Gbfly_s": round(butterflies(cfg, cfg["batch"]) / n_ops / (ms * 1e-3) / 1e9, 1)}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
