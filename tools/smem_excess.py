"""Shared-memory excess wavefronts per SASS instruction from an ncu source-page export
(`ncu -i rep --page source --csv --print-source sass`): every kernel in the file, its total excess and
the instructions carrying it.
    python tools/smem_excess.py <sass.csv> [top]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    blocks, cur, seen = [], None, set()
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = None if r[1] in seen else {"name": r[1], "rows": []}
            seen.add(r[1])
            if cur:
                blocks.append(cur)
            continue
        if cur is None:
            continue
        if r and r[0] == "Address":
            cur["hdr"] = {k: i for i, k in enumerate(r)}
        elif "hdr" in cur and len(r) >= len(cur["hdr"]):
            cur["rows"].append(r)
    for b in blocks:
        h = b["hdr"]
        ex = [(int(r[h["L1 Wavefronts Shared Excessive"]] or 0), int(r[h["L1 Wavefronts Shared"]] or 0), i,
               r[h["Source"]].strip()[:64]) for i, r in enumerate(b["rows"])]
        tot, wf = sum(e[0] for e in ex), sum(e[1] for e in ex)
        print(f"{b['name'][:110]}\n  shared wavefronts {wf}, excess {tot} ({100 * tot / max(wf, 1):.1f} %)")
        for e in sorted(ex, reverse=True)[:top]:
            if e[0]:
                print(f"    {e[0]:>10} / {e[1]:>10}  #{e[2]:<5} {e[3]}")


if __name__ == "__main__":
    main()
