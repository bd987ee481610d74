import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def read_golden(name):
    """Parse a tests/golden/*.txt fixture: '#' comments, 'key v1 v2 ...' lines."""
    out, rows = {}, []
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if parts[0].lstrip("-").isdigit():
                rows.append([int(v) for v in parts])
            else:
                vals = [int(v) for v in parts[1:]]
                out[parts[0]] = vals[0] if len(vals) == 1 else vals
    out["rows"] = rows
    return out
