"""Summarise ncu reports / launch lists into profiles/ (committed evidence).

    python tools/ncu_summary.py report <file.ncu-rep> <out.md> [--json out.json --config c2]
    python tools/ncu_summary.py launches <launches.csv> <out.md>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy (IMAD) pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def report(rep, out_md, out_json=None, config=None):
    hdr, units, rows = raw_rows(rep)
    lines = [f"# ncu --set full summary: `{rep.split('/')[-1]}`", ""]
    per_kernel = []
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        d = {"kernel": name}
        lines.append(f"## `{name}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {label} (`{k}`) | {r[i]} | {units[i]} |")
                d[k] = r[i]
                d[k + ".unit"] = units[i]
        st = [(h, float(r[i])) for i, h in enumerate(hdr)
              if "smsp__average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio")
              and r[i] not in ("", "n/a")]
        st.sort(key=lambda x: -x[1])
        lines.append("")
        lines.append("Top stall reasons (cycles per issued instruction): " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for h, v in st[:8]))
        lines.append("")
        per_kernel.append(d)
    open(out_md, "w").write("\n".join(lines) + "\n")
    if out_json:
        def to_bytes(v, u):
            f = float(v)
            return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        try:
            data = json.load(open(out_json))
        except Exception:
            data = {}
        traffic = []
        for d in per_kernel:
            rd = to_bytes(d["dram__bytes_read.sum"], d["dram__bytes_read.sum.unit"])
            wr = to_bytes(d["dram__bytes_write.sum"], d["dram__bytes_write.sum.unit"])
            traffic.append({"kernel": d["kernel"], "dram_bytes": rd + wr})
        data[config] = {"source": rep.split("/")[-1], "kernels": traffic,
                        "dram_bytes_per_launch": max(t["dram_bytes"] for t in traffic)}
        json.dump(data, open(out_json, "w"), indent=1)


def launches(csv_path, out_md):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[1:]:
        if len(r) <= vi or not r[vi]:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki]
        short = name.split("(")[0]
        agg[short][0] += 1
        agg[short][1] += v * scale
        total += v * scale
    lines = [f"# Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`): `{csv_path.split('/')[-1]}`",
             "", "Cold-cache, serialised per-launch times: compare shares, not absolutes.  The whole bench command is",
             "listed (ALU calibration, input generation, L2 flushes, the e2e host-pipeline chunks and the timed steps).", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / total:.1f}% |")
    # per (kernel, grid): the full-batch launches of the timed steps are the ones with the largest grid
    gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
    if gi is not None:
        byg = defaultdict(list)
        for r in rows[1:]:
            if len(r) <= vi or not r[vi]:
                continue
            v = float(r[vi].replace(",", ""))
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
            byg[(r[ki].split("(")[0], r[gi])].append(v * scale)
        lines += ["", "Per kernel and grid (mean per launch):", "", "| kernel | grid | launches | mean us |", "|---|---|---|---|"]
        for (k, g), vs in sorted(byg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k}` | {g} | {len(vs)} | {sum(vs) / len(vs):.1f} |")
    # launch sequence: consecutive launches of the same kernel and grid merged, in ID order, so the
    # timed steps (warm-up + timed fwd/inv pairs) are visible apart from the e2e pipeline's chunks
    lines += ["", "Launch sequence (consecutive identical kernels merged):", "",
              "| first ID | kernel | grid | launches | us each |", "|---|---|---|---|---|"]
    seq = []
    for r in rows[1:]:
        if len(r) <= vi or not r[vi]:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        key = (r[ki].split("(")[0].replace("void nttb::", "").replace("void ", ""), r[gi] if gi is not None else "")
        us = round(v * scale, 1)
        if seq and seq[-1][1] == key and abs(seq[-1][3][-1] - us) <= max(2.0, 0.1 * us):
            seq[-1][3].append(us)
        else:
            seq.append([r[0], key, None, [us]])
    for rid, (k, g), _, vs in seq:
        each = f"{vs[0]:.1f}" if len(vs) == 1 else f"{min(vs):.1f}-{max(vs):.1f}"
        lines.append(f"| {rid} | `{k[:70]}` | {g} | {len(vs)} | {each} |")
    open(out_md, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        args = sys.argv[2:]
        oj = cfg = None
        if "--json" in args:
            oj = args[args.index("--json") + 1]
        if "--config" in args:
            cfg = args[args.index("--config") + 1]
        report(args[0], args[1], oj, cfg)
    else:
        launches(sys.argv[2], sys.argv[3])
