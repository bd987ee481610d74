"""Range audit (debug build libntt_b200_audit.so, -DNTT_RANGE_AUDIT): the theorems' intervals
(Theorem 2; Theorem 3; Theorem 4) hold inside every kernel at the
config shapes, including inputs at the tops of the accepted ranges, and a butterfly with Algorithm 3's
"+2p" dropped (the mutation control) is reported."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
AUDIT_LIB = os.path.join(os.path.dirname(HERE), "paper_1205_2926_b200", "libntt_b200_audit.so")


def _run(which):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert os.path.exists(AUDIT_LIB), "the audit build is missing (__graft_entry__.build() makes it)"
    env = dict(os.environ, NTT_B200_LIB="audit")
    r = subprocess.run([sys.executable, os.path.join(HERE, "audit_child.py"), which], capture_output=True,
                       text=True, env=env, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_no_range_violations_at_config_shapes():
    counts = _run("clean")
    counts = {k: v for k, v in counts.items() if not k.startswith("STRESS")}
    assert len(counts) >= 8
    assert all(v == 0 for v in counts.values()), counts


def test_race_stress_changes_nothing():
    """Per-warp random delays at every round of every kernel (audit build's race stress; compute-sanitizer's
    racecheck is closed on the pool): results bit-identical to the unstressed run, audit clean."""
    counts = _run("stress")
    assert len(counts) >= 6
    for name, r in counts.items():
        assert r["identical"] and r["violations"] == 0, (name, r)
    # the delays really ran: the stressed runs together are slower (summed over the timed cases, so one
    # case's cold first run or a kernel whose warps absorb the delays cannot hide it)
    timed = [r for name, r in counts.items() if "P2P" not in name]
    plain, stressed = sum(r["ms_plain"] for r in timed), sum(r["ms_stressed"] for r in timed)
    assert stressed > 1.1 * plain, counts


def test_mutated_butterfly_is_reported():
    counts = _run("mutant")
    assert all(v > 0 for v in counts.values()), counts
