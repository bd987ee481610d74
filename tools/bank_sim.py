"""Shared-memory bank-conflict simulator for the round/exchange access patterns of the
contiguous NTT kernel.  Model: 32 banks x 4 B; an access of width
w bytes is served in phases of 128/w lanes; a phase costs max over banks of the number of
distinct 4-byte words it touches.  Ideal = one wavefront per phase.

    python tools/bank_sim.py          # report every (word, N, round) pattern
"""
import sys


def swz_tma128(i, wb):
    """Element index -> physical element index under TMA SWIZZLE_128B (16-B chunk ^= row % 8)."""
    o = i * wb
    o ^= ((o >> 7) & 7) << 4
    return o // wb


def swz_xor(i, wb):
    s = 4 if wb == 8 else 5
    return i ^ ((i >> s) & ((1 << s) - 1))


def wavefronts(addrs, w):
    """addrs: 32 byte addresses (None = inactive lane), access width w."""
    per_phase = 128 // w if w >= 4 else 32
    total = 0
    for ph in range(0, 32, per_phase):
        banks = {}
        for a in addrs[ph:ph + per_phase]:
            if a is None:
                continue
            for b4 in range(a // 4, (a + w) // 4):
                banks.setdefault(b4 % 32, set()).add(b4)
        total += max((len(v) for v in banks.values()), default=0)
    return total


def rounds(logn, le):
    R = (logn + le - 1) // le
    sr = [logn // R + (1 if r < logn % R else 0) for r in range(R)]
    lv = [sum(sr[:r]) for r in range(R)]
    return sr, lv


def check(wb, logn, le, swz, vec_runs=True):
    """Worst-case wavefront ratio (actual / ideal) over all rounds and warps of one CTA slot."""
    N = 1 << logn
    E = 1 << le
    T = N // E
    sr, lv = rounds(logn, le)
    worst = 1.0
    report = []
    for r, (SR, LEVEL) in enumerate(zip(sr, lv)):
        S, G = 1 << SR, E >> SR
        D, B = N >> (LEVEL + SR), N >> LEVEL
        ratio_r = 1.0
        for warp0 in range(0, T, 32):
            lanes = range(warp0, min(warp0 + 32, T))
            for q in range(G):
                if D == 1 and vec_runs and S * wb >= 16:
                    per = 16 // wb
                    for h0 in range(0, S, per):
                        addrs = []
                        for t in lanes:
                            g = t + T * q
                            i = (g // D) * B + h0 * D + (g % D)
                            addrs.append(swz(i, wb) * wb)
                        addrs += [None] * (32 - len(addrs))
                        # a 16-B vector needs its elements adjacent after swizzling
                        ok = all(swz((a // wb) + 0, wb) is not None for a in addrs if a is not None)
                        n_act = sum(a is not None for a in addrs)
                        ideal = -(-n_act * 16 // 128)
                        ratio_r = max(ratio_r, wavefronts(addrs, 16) / max(ideal, 1))
                else:
                    for h in range(S):
                        addrs = []
                        for t in lanes:
                            g = t + T * q
                            i = (g // D) * B + h * D + (g % D)
                            addrs.append(swz(i, wb) * wb)
                        addrs += [None] * (32 - len(addrs))
                        n_act = sum(a is not None for a in addrs)
                        ideal = -(-n_act * wb // 128)
                        ratio_r = max(ratio_r, wavefronts(addrs, wb) / max(ideal, 1))
        report.append((r, SR, LEVEL, D, ratio_r))
        worst = max(worst, ratio_r)
    return worst, report


def vec_pairs_adjacent(swz, wb, N):
    """16-B vectors of consecutive elements stay adjacent and 16-B aligned after swizzling."""
    per = 16 // wb
    for i in range(0, N, per):
        base = swz(i, wb)
        if base % per or any(swz(i + k, wb) != base + k for k in range(per)):
            return False
    return True


if __name__ == "__main__":
    for name, swz in (("tma128", swz_tma128), ("xor_elem", swz_xor)):
        print(f"== {name}")
        for wb, rng, le_of in ((8, range(5, 15), lambda n: 4 if n <= 13 else 5), (4, range(6, 16), lambda n: 5)):
            for logn in rng:
                le = le_of(logn)
                w, rep = check(wb, logn, le, swz)
                vp = vec_pairs_adjacent(swz, wb, 1 << logn)
                print(f"  u{wb*8} N=2^{logn:<2d} LE={le} worst={w:.2f} vec_ok={vp} rounds=" +
                      " ".join(f"[r{r} SR{s} D{d}:{x:.2f}]" for r, s, l, d, x in rep))
