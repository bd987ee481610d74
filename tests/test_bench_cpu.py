"""Host logic of bench.py (no GPU): the roofline's per-pass nontrivial-product count, the shared
config object of both arms, and --gpus N failing loudly when N GPUs are not there."""
import os
import subprocess
import sys

import pytest

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def brute_nontrivial(ell):
    """Count Algorithm 1's butterflies with twiddle != 1 directly: stage i has
    m = L >> i and twiddle zeta_i^k, k < m, which is 1 only for k = 0."""
    L = 1 << ell
    return sum((L // (2 * (L >> i))) * ((L >> i) - 1) for i in range(1, ell + 1))


@pytest.mark.parametrize("ell", range(0, 13))
def test_nontrivial_formula(ell):
    assert bench.nontrivial(ell) == brute_nontrivial(ell)


@pytest.mark.parametrize("ell,passes", [(24, [9, 15]), (28, [8, 8, 12]), (20, [9, 11]), (12, [12]),
                                        (17, [4, 13]), (26, [9, 9, 8])])
def test_pass_products_sum_to_the_transform(ell, passes):
    """Sub-NTTs plus the (N-1)(S-1) non-unit four-step twiddles of every pass add up to exactly
    (L/2) ell - (L-1) per transform (the four-step keeps Algorithm 1's count)."""
    for batch in (1, 3):
        tot = sum(bench.pass_products(ell, passes, j, batch) for j in range(len(passes)))
        assert tot == batch * bench.nontrivial(ell)


def test_config_dict_is_arm_independent():
    cfg = dict(bench.CONFIGS["c4"], key="c4")
    c1 = bench.config_dict(cfg, 1)
    assert c1["workload"].startswith("C4") and c1["transforms_per_gpu"] == 64
    assert c1["butterflies_per_step_per_gpu"] == 64 * (1 << 23) * 24
    c2 = bench.config_dict(cfg, 2)
    assert c2["transforms_per_gpu"] == 32
    c5 = bench.config_dict(dict(bench.CONFIGS["c5"], key="c5"), 4)
    assert "four-step" in c5["parallelism"] and c5["butterflies_per_step_per_gpu"] == (1 << 27) * 28 // 4


def test_default_config_is_c4():
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'ap.add_argument("--config", default="c4"' in src


def test_gpus_flag_fails_loudly_without_gpus():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "only 0 CUDA device" in r.stderr


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="4", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "does not match WORLD_SIZE" in r.stderr
