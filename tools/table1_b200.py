"""The paper's Table 1 comparison (Algorithm 2 vs Algorithm 3, cycles per butterfly,
L = 2^11, 62-bit prime) re-run on B200 with batched transforms; Algorithm 5 added (F2).  Besides the
paper's shape, one line per BASELINE config (C1-C5 forward), each running the config's own kernels
(on-chip, 2-CTA cluster, four-step column passes) with the selected butterfly.

    python tools/table1_b200.py [--batch 8192]

Prints one JSON object: butterflies/s and ns per butterfly per SM for each butterfly, per shape.
Forward transforms only (Alg. 2 and Alg. 5 are forward butterflies), canonical inputs.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1205_2926_b200 as ntt  # noqa: E402

P62 = 29 * 2**57 + 1
P62G = 2305843009146585089
P30 = 998244353


def run(p, bits, ell, batch, alg, reps=20):
    L = 1 << ell
    w = pow(3, (p - 1) // L, p)
    plan = ntt.Plan(p, w, ell, bits, butterfly=alg)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x0 = torch.empty(batch * L, dtype=dt, device="cuda")
    ntt.synth_uniform(x0, 0x12052926, alg, bound=p)
    x = x0.clone()
    s = torch.cuda.current_stream()
    for _ in range(3):
        plan.forward(x)
    ms = []
    for _ in range(reps):
        x.copy_(x0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        plan.forward(x)
        e1.record(s)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    t = ms[len(ms) // 2] * 1e-3
    bfly = batch * (L // 2) * ell
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    return {"bfly_per_s": bfly / t, "ms": t * 1e3, "ns_per_bfly_per_SM": t * 1e9 * sms / bfly}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8192)
    a = ap.parse_args()
    out = {"paper_table1_cycles_per_bfly": {"Westmere": {"alg2": 10.1, "alg3": 6.9}, "SandyBridge": {"alg2": 9.1, "alg3": 5.9},
                                            "Piledriver": {"alg2": 13.9, "alg3": 12.0}},
           "shapes": {}}
    shapes = (("paper L=2^11 62-bit p (p=1 mod 2^32)", P62, 64, 11, a.batch),
              ("paper L=2^11 62-bit p (generic p)", P62G, 64, 11, a.batch),
              ("u32 L=2^11, p=998244353", P30, 32, 11, a.batch),
              ("C1 1 x 2^10 u32 (latency)", P30, 32, 10, 1),
              ("C2 4096 x 2^12 u64 (forward)", P62, 64, 12, 4096),
              ("C3 1024 x 2^16 u32 p=998244353 (forward, 2-CTA cluster kernel)", P30, 32, 16, 1024),
              ("C4 64 x 2^24 u64 (column pass with twiddle matrix + 2^15 cluster row pass)", P62, 64, 24, 64),
              ("C5 1 x 2^28 u64 (two factored column passes + 2^12 row pass)", P62, 64, 28, 1))
    for name, p, bits, ell, batch in shapes:
        r = {f"alg{alg}": run(p, bits, ell, batch, alg) for alg in (2, 3, 5)}
        r["alg2_over_alg3_time"] = r["alg2"]["ms"] / r["alg3"]["ms"]
        r["alg5_over_alg3_time"] = r["alg5"]["ms"] / r["alg3"]["ms"]
        out["shapes"][name] = r
    print(json.dumps(out))


if __name__ == "__main__":
    main()
