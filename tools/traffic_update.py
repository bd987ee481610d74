"""Record per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of a config's kernels
from an `ncu --set full` raw-page export into profiles/ncu_traffic.json, keyed by the pass names
bench.py times (so `roofline.traffic` of the dominant kernel comes from the committed capture).
    python tools/traffic_update.py c4 <raw.csv> <source-name> "k_cols_tma=fwd pass 0 (column pass, 2^9)" ...
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    cfg, raw, source = sys.argv[1], sys.argv[2], sys.argv[3]
    maps = [a.split("=", 1) for a in sys.argv[4:]]
    rows = list(csv.reader(open(raw)))
    hdr = rows[0]
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")

        def num(k):
            v = d.get(k, "0").replace(",", "")
            unit = ""
            return float(v) if v else 0.0, unit
        rd, wr = num("dram__bytes_read.sum")[0], num("dram__bytes_write.sum")[0]
        # raw pages report bytes in the unit row (rows[1]); scale Gbyte/Mbyte/Kbyte to bytes
        units = dict(zip(hdr, rows[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
        wr *= scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
        for key, pname in maps:
            if key in name and pname not in out:
                out[pname] = {"kernel": name, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                              "duration_ms": float(d.get("gpu__time_duration.sum", "0") or 0)}
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    prof = json.load(open(path)) if os.path.exists(path) else {}
    prof[cfg] = {"source": source, "per_pass": out}
    json.dump(prof, open(path, "w"), indent=1)
    print(json.dumps(prof[cfg], indent=1))


if __name__ == "__main__":
    main()
