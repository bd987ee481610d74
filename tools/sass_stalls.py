"""Stall-reason totals and the hottest SASS lines of one kernel from an ncu source page export
(`ncu -i rep --page source --csv --print-source sass`).
    python tools/sass_stalls.py <kernel_sass.csv> [top]"""
import collections
import csv
import sys


def main():
    fn = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(open(fn)))
    # one block per kernel: a "Kernel Name" row, a header row starting with "Address", then the lines;
    # the first kernel's block is analysed (pass a file exported with -k for another)
    h0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[h0]
    idx = {h: i for i, h in enumerate(hdr)}
    data = []
    for r in rows[h0 + 1:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) >= len(hdr) and r[0] != "Address":
            data.append(r)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    for r in data:
        for h in stalls:
            tot[h] += int(r[idx[h]] or 0)
    all_s = sum(tot.values())
    print("stall reasons (share of samples):")
    for h, c in tot.most_common():
        if c:
            print(f"  {h:28s} {c / all_s * 100:5.1f}%")
    print(f"hottest {top} instructions (samples share, top reasons):")
    data.sort(key=lambda r: -int(r[idx['Warp Stall Sampling (All Samples)']] or 0))
    for r in data[:top]:
        s = int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
        reasons = sorted(((int(r[idx[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
        print(f"  {s / all_s * 100:5.2f}%  {r[idx['Address']][-5:]}  {r[idx['Source']].strip()[:60]:60s} "
              + " ".join(f"{n}:{c}" for c, n in reasons if c))


if __name__ == "__main__":
    main()
