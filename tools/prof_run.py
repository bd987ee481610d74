"""Minimal driver for ncu captures: runs `reps` steps of one bench config's hot path.
    python tools/prof_run.py c2 [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1205_2926_b200 as ntt  # noqa: E402
from bench import CONFIGS, root  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = CONFIGS[key]
    L = 1 << cfg["ell"]
    dt = torch.uint64 if cfg["bits"] == 64 else torch.uint32
    plans = [ntt.Plan(p, root(p, L), cfg["ell"], cfg["bits"]) for p in cfg["primes"]]
    if cfg["ops"] == ("conv",):
        a = torch.zeros(cfg["batch"], L, dtype=dt, device="cuda")
        b = torch.zeros_like(a)
        ntt.synth_uniform(a, 1, 0, bits=20)
        ntt.synth_uniform(b, 1, 1, bits=20)
        a[:, L // 2:] = 0
        b[:, L // 2:] = 0
        for _ in range(reps):
            for pl in plans:
                pl.cyclic_convolve(a.clone(), b.clone())
    else:
        x = torch.empty(cfg["batch"] * L, dtype=dt, device="cuda")
        ntt.synth_uniform(x, 1, 0, bound=cfg["primes"][0])
        for _ in range(reps):
            for op in cfg["ops"]:
                (plans[0].forward if op == "fwd" else plans[0].inverse)(x)
    torch.cuda.synchronize()
    print("ok", key, reps)


if __name__ == "__main__":
    main()
