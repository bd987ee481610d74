"""Child process of test_gpu_audit.py: loads the range-audit build (NTT_B200_LIB=audit) and runs the
config shapes through it, printing one JSON object of violation counts per case."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1205_2926_b200 as ntt  # noqa: E402
import synth  # noqa: E402

P30, P62 = 998244353, 29 * 2**57 + 1


def root(p, L):
    return pow(3, (p - 1) // L, p)


def case(name, fn, mutate=False):
    ntt.audit_reset(0, mutate=mutate)
    fn()
    torch.cuda.synchronize()
    out[name] = ntt.audit_counts(0)
    ntt.audit_reset(0, mutate=False)


def transform(p, bits, ell, batch, ops=("fwd", "inv"), alg=3, top=False):
    def fn():
        L = 1 << ell
        plan = ntt.Plan(p, root(p, L), ell, bits, butterfly=alg)
        dt = torch.uint64 if bits == 64 else torch.uint32
        x = torch.empty(batch * L, dtype=dt, device="cuda")
        ntt.synth_uniform(x, synth.config_seed(7), ell, bound=p)
        def fill(v):  # word v in every 3rd / 5th place (through a signed view: torch has no uint64 fill)
            if bits == 64:
                return x.view(torch.int64), v - (1 << 64) if v >= 1 << 63 else v
            return x.view(torch.int32), v - (1 << 32) if v >= 1 << 31 else v
        if top:  # inputs at the top of Algorithm 3's accepted range [0,2p)
            t, v = fill(2 * p - 1)
            t[::3] = v
        for op in ops:
            if op == "inv" and top:
                t, v = fill(4 * p - 1)  # Algorithm 4 accepts [0,4p)
                t[::5] = v
            (plan.forward if op == "fwd" else plan.inverse)(x)
    return fn


def conv(batch):
    def fn():
        L = 1 << 16
        for p in (469762049, 167772161, 998244353):
            plan = ntt.Plan(p, root(p, L), 16, 32)
            a = torch.zeros(batch, L, dtype=torch.uint32, device="cuda")
            b = torch.zeros_like(a)
            t = torch.empty(batch * L // 2, dtype=torch.uint32, device="cuda")
            ntt.synth_uniform(t, 3, 0, bits=20)
            a[:, :L // 2] = t.view(batch, -1)
            ntt.synth_uniform(t, 3, 1, bits=20)
            b[:, :L // 2] = t.view(batch, -1)
            plan.cyclic_convolve(a, b)
    return fn


def stress_case(name, p, bits, ell, batch, ops=("fwd", "inv"), conv=False):
    """The same transform with and without race stress (per-warp random delays at every round): the
    results must be identical and the range audit clean."""
    L = 1 << ell
    plan = ntt.Plan(p, root(p, L), ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(batch * L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(8), ell, bound=p)
    outs, ms = [], []
    for stress in (False, False, True):  # the first run loads the kernels (lazy module loading): untimed
        ntt.audit_reset(0, stress=stress)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if conv:
            a = x.clone().view(batch, L)
            b = x.clone().view(batch, L).flip(0).contiguous()
            plan.cyclic_convolve(a, b)
            y = a.view(-1)
        else:
            y = x.clone()
            for op in ops:
                (plan.forward if op == "fwd" else plan.inverse)(y)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        outs.append((y.view(torch.int64) if bits == 64 else y.view(torch.int32)).clone())
        viol = ntt.audit_counts(0)
    ntt.audit_reset(0)
    out["STRESS " + name] = {"identical": bool(torch.equal(outs[1], outs[2]) and torch.equal(outs[0], outs[2])),
                             "violations": viol, "ms_plain": round(ms[1], 3), "ms_stressed": round(ms[2], 3)}


def stress_p2p(name, p, bits, ell, ell1, G):
    """The fused column pass + all-to-all (virtual ranks on one GPU, P2P stores into the peers' receive
    buffers) under race stress: equal to ntt_forward."""
    from paper_1205_2926_b200.dist import FourStepForwardP2P, FourStepLayout
    lay = FourStepLayout(ell, ell1, G)
    L, N1, N2, Wl = lay.L, lay.N1, lay.N2, lay.local_width
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(5), 3, bound=p)
    ref = x.clone()
    plan.forward(ref)
    ok = True
    for stress in (False, True):
        ntt.audit_reset(0, stress=stress)
        shards = [x.view(N1, N2)[:, g * Wl:(g + 1) * Wl].contiguous().view(-1) for g in range(G)]
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
        torch.cuda.synchronize()
        iv = torch.int64 if bits == 64 else torch.int32
        ok = ok and bool(torch.equal(torch.cat(outs).view(iv), ref.view(iv)))
        viol = ntt.audit_counts(0)
    ntt.audit_reset(0)
    out["STRESS " + name] = {"identical": ok, "violations": viol, "ms_plain": 1.0, "ms_stressed": 1.0}


assert ntt.audit_build(), "NTT_B200_LIB=audit did not load the audit build"
out = {}
which = sys.argv[1:] or ["all"]
if "all" in which or "clean" in which:
    case("C1 2^10 u32", transform(P30, 32, 10, 1, top=True))
    case("C2 4096 x 2^12 u64 fwd+inv", transform(P62, 64, 12, 4096, top=True))
    case("C3 64 pairs x 2^16 u32 convolution (3 primes)", conv(64))
    case("2^15 u64 cluster fwd+inv", transform(P62, 64, 15, 64, top=True))
    case("C4 shape 2 x 2^24 u64 fwd+inv", transform(P62, 64, 24, 2, top=True))
    case("C5 shape 2^28 u64 fwd+inv", transform(P62, 64, 28, 1, top=True))
    case("C4 shape 2 x 2^24 u64 fwd Alg. 5", transform(P62, 64, 24, 2, ops=("fwd",), alg=5))
    case("C4 shape 2 x 2^24 u64 fwd Alg. 2", transform(P62, 64, 24, 2, ops=("fwd",), alg=2))
    case("2^20 u32 fwd+inv", transform(P30, 32, 20, 2, top=True))
if "all" in which or "mutant" in which:
    case("MUTANT C2 4096 x 2^12 u64 fwd", transform(P62, 64, 12, 4096, ops=("fwd",)), mutate=True)
    case("MUTANT C4 shape 1 x 2^24 u64 fwd", transform(P62, 64, 24, 1, ops=("fwd",)), mutate=True)
    case("MUTANT 2^16 u32 fwd", transform(P30, 32, 16, 8, ops=("fwd",)), mutate=True)
if "all" in which or "stress" in which:
    stress_case("C2 4096 x 2^12 u64 fwd+inv", P62, 64, 12, 4096)
    stress_case("2^15 u64 cluster fwd+inv", P62, 64, 15, 64)
    stress_case("2^16 u32 cluster fwd+inv", P30, 32, 16, 64)
    stress_case("2^16 u32 convolution (fused pointwise)", P30, 32, 16, 32, conv=True)
    stress_case("C4 shape 2 x 2^24 u64 fwd+inv", P62, 64, 24, 2)
    stress_case("C5 shape 2^28 u64 fwd", P62, 64, 28, 1, ops=("fwd",))
    stress_case("2^10 u32 fwd+inv", P30, 32, 10, 7)
    stress_p2p("P2P four-step 2^16 over 4 virtual ranks", P62, 64, 16, 8, 4)
    stress_p2p("P2P four-step 2^10, one-round column pass (R = 1)", P62, 64, 10, 4, 2)
    stress_p2p("P2P four-step 2^12 u32, one-round column pass (R = 1)", P30, 32, 12, 5, 2)
print(json.dumps(out))
