#!/usr/bin/env python
"""Benchmark of the batched NTT hot path (BASELINE.json metric: NTT butterflies/s and
achieved HBM GB/s) on B200.

Default workload = BASELINE.json configs[3] (config C4), the largest configuration that fits one
GPU: 64 transforms of L = 2^24 over p = 29*2^57+1 (beta = 2^64), one step = the forward
transform of the whole batch (two kernel passes: a four-step column pass and the row pass).
Other configs (--config c1..c5) are available for measurement; the driver runs the default.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl native|reference]

N > 1: launched by torchrun (or, when WORLD_SIZE is unset, bench.py re-launches itself through
torch.distributed.run with N ranks; it exits non-zero if the box has fewer than N GPUs), one rank
per GPU over NCCL.  C4's 64 transforms are split over the ranks (strong scaling, no data-path
collective), time = max over ranks.  Prints ONE JSON line on rank 0.

Roofline: for the dominant kernel, T_MUL = its nontrivial Shoup products
((L/2) ell - (L-1) per transform over all passes, split per pass incl. the four-step twiddle
multiplies) / the derived integer-pipe peak, T_HBM = its algorithmic bytes (one read + one
write of the data per pass) / MEASURED_PEAKS.json hbm_gbs; frac = max(T_MUL, T_HBM) / measured.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P30 = 998244353
P62 = 29 * 2**57 + 1
RNS = (469762049, 167772161, 998244353)
METRIC = "NTT butterflies/s"

CONFIGS = {
    "c1": dict(workload="C1: 1 x 2^10 forward, beta=2^32, p=998244353", primes=(P30,), bits=32, ell=10, batch=1,
               ops=("fwd",), scaling="weak", seed_cfg=1),
    "c2": dict(workload="C2: 4096 x 2^12 forward+inverse, beta=2^64, p=29*2^57+1", primes=(P62,), bits=64, ell=12,
               batch=4096, ops=("fwd", "inv"), scaling="weak", seed_cfg=2),
    "c3": dict(workload="C3: 3 primes x 1024 pairs x 2^16 cyclic convolution (fwd,fwd,pointwise,inv), beta=2^32",
               primes=RNS, bits=32, ell=16, batch=1024, ops=("conv",), scaling="weak", seed_cfg=3),
    "c4": dict(workload="C4: 64 x 2^24 forward, beta=2^64, p=29*2^57+1", primes=(P62,), bits=64, ell=24, batch=64,
               ops=("fwd",), scaling="strong", seed_cfg=4),
    "c5": dict(workload="C5: 1 x 2^28 forward (single GPU four-step), beta=2^64, p=29*2^57+1", primes=(P62,), bits=64,
               ell=28, batch=1, ops=("fwd",), scaling="weak", seed_cfg=5),
}


def butterflies(cfg, batch):
    """All (L/2)*ell radix-2 butterflies of Algorithm 1, W = 1 ones included (P:226 divisor)."""
    L = 1 << cfg["ell"]
    per = (L // 2) * cfg["ell"]
    n_ntt = 3 if cfg["ops"] == ("conv",) else len(cfg["ops"])
    return per * n_ntt * batch * len(cfg["primes"])


def root(p, L):
    return pow(3, (p - 1) // L, p)


def derived_alu_peak(bits, p, sms, clock_mhz):
    """Butterflies/s bound of the fmaheavy (IMAD) pipe for Algorithm 3's multiplies (DESIGN.md
    "Roofline").  Measured opcode rates per SM per clock (tools/int_pipe_peak.cu): IMAD.WIDE.U32 and
    IMAD.HI 32, IMAD 64, i.e. 4 and 2 SMSP-cycles per warp instruction.
      beta=2^64: hi64(W'T) 4 WIDE; lo64(WT) 1 WIDE + 2 IMAD; lo64(Qp) 1 WIDE + 2 IMAD
                 -> 32 SMSP-cycles / warp-butterfly (26 when p = 1 mod 2^32: lo64(Qp) = 1 IMAD)
      beta=2^32: Q 1 IMAD.HI; W*T - Q*p 2 IMAD -> 8 SMSP-cycles / warp-butterfly."""
    if bits == 64:
        cyc = 26 if (p & 0xFFFFFFFF) == 1 else 32
    else:
        cyc = 8
    return sms * clock_mhz * 1e6 * 4 * 32 / cyc


def nontrivial(ell):
    """Nontrivial (W != 1) butterflies of one length-2^ell Algorithm 1 transform: (L/2) ell - (L-1)
    (the L-1 butterflies with W = 1 need no multiply)."""
    L = 1 << ell
    return (L // 2) * ell - (L - 1) if ell else 0


def pass_products(ell, passes, j, batch):
    """Nontrivial Shoup products of kernel pass j of the schedule `passes` (outermost first) over
    `batch` transforms.  Pass j views each block of B = 2^(ell - outer) words as N = 2^passes[j] rows
    x S columns: S column NTTs of length N plus the four-step twiddles omega_B^{c rev(r)}, of which
    (N-1)(S-1) are not 1 (r = 0 or c = 0 give W = 1); the last pass has S = 1 (row NTTs only).
    Summed over the passes this is exactly batch * nontrivial(ell) (DESIGN.md Roofline)."""
    outer = sum(passes[:j])
    n = passes[j]
    N, S = 1 << n, 1 << (ell - outer - n)
    blocks = batch << outer
    return blocks * (S * nontrivial(n) + (N - 1) * (S - 1))


def per_rank_batch(cfg, world):
    batch = cfg["batch"]
    if cfg["scaling"] == "strong" and world > 1 and cfg["key"] != "c5":
        assert batch % world == 0, "strong-scaled batch must divide over ranks"
        batch //= world
    return batch


def config_dict(cfg, world):
    """The `config` object of the JSON line; the native and the reference arm print the same one."""
    L = 1 << cfg["ell"]
    batch = per_rank_batch(cfg, world)
    dist_c5 = cfg["key"] == "c5" and world > 1
    bfly = butterflies(cfg, batch) // (world if dist_c5 else 1)
    par = (f"four-step split over {world} GPUs (one all-to-all transpose)" if dist_c5
           else f"batch-sharded x{world}, no collective")
    big = batch * L * cfg["bits"] // 8 > (256 << 20)
    return {"workload": cfg["workload"], "transforms_per_gpu": batch, "L": L, "butterflies_per_step_per_gpu": bfly,
            "parallelism": par,
            "l2": ("inputs larger than L2 (" + f"{batch * L * cfg['bits'] // 8 >> 20} MiB per GPU" + ") and "
                   if big else "") + "L2 flushed between timed steps (256 MiB zero-fill, outside the step events)"}


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


class NvmlSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every ~1 ms on a thread, so
    even a few-millisecond timed region is sampled (nvidia-smi's 100 ms period can miss it)."""
    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, torch_device):
        self.samples, self.reasons, self.h, self.nv = [], set(), None, None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            uuid = str(getattr(torch.cuda.get_device_properties(torch_device), "uuid", ""))
            try:
                self.h = nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(torch_device.index or 0)
            self.nv = nv
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, const in self.NAMES:
                    if r & getattr(nv, const, 0):
                        self.reasons.add(name)
            except Exception:
                break
            self._stop.wait(0.001)

    def start(self):
        if self.h is None:
            return
        self._stop = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self):
        if self.h is None:
            return None
        self._stop.set()
        self.t.join(timeout=2)
        if not self.samples:
            return None
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml, ~1 ms"}


# ------------------------------------------------------------------ native arm
def run_native(args, cfg, rank, world, local_rank):
    import torch
    import paper_1205_2926_b200 as ntt

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    L = 1 << cfg["ell"]
    bits = cfg["bits"]
    dt = torch.uint64 if bits == 64 else torch.uint32
    wb = bits // 8
    batch = per_rank_batch(cfg, world)
    plans = [ntt.Plan(p, root(p, L), cfg["ell"], bits, device=local_rank) for p in cfg["primes"]]
    conv = cfg["ops"] == ("conv",)
    dist_c5 = cfg["key"] == "c5" and world > 1  # one transform split four-step over the ranks
    exchange = None
    # inputs generated in HBM by the seeded counter-based generator (synth/ definition)
    seed = 0x12052926 ^ cfg["seed_cfg"]
    first = rank * batch
    with torch.cuda.stream(stream):
        if conv:
            half = L // 2
            a0 = torch.zeros(batch, L, dtype=dt, device=dev)
            b0 = torch.zeros(batch, L, dtype=dt, device=dev)
            tmp = torch.empty(batch * half, dtype=dt, device=dev)
            ntt.synth_uniform(tmp, seed, 0, start=first * half, bits=20, stream=stream)
            a0[:, :half] = tmp.view(batch, half)
            ntt.synth_uniform(tmp, seed, 1, start=first * half, bits=20, stream=stream)
            b0[:, :half] = tmp.view(batch, half)
            del tmp
            work = [(a0.clone(), b0.clone()) for _ in plans]
            src = (a0, b0)
        elif dist_c5:
            from paper_1205_2926_b200.dist import FourStepForward, FourStepLayout
            lay = FourStepLayout(cfg["ell"], cfg["ell"] // 2, world)
            full = torch.empty(L, dtype=dt, device=dev)  # the same global input on every rank
            ntt.synth_uniform(full, seed, 0, bound=cfg["primes"][0], stream=stream)
            c0, c1 = lay.columns(rank)
            x0 = full.view(lay.N1, lay.N2)[:, c0:c1].contiguous().view(-1)
            del full
            x = x0.clone()
            recv = torch.empty_like(x)
            outbuf = torch.empty_like(x)
            fs = FourStepForward(plans[0], lay, rank)
            # fused column pass + all-to-all over peer memory (ntt_fourstep_cols_p2p) when symmetric
            # memory is available and its result matches the NCCL path on this input (checked once,
            # outside the timed region); otherwise the NCCL all_to_all_single path
            exchange, fs_p2p = "nccl", None
            if os.environ.get("NTT_C5_EXCHANGE", "p2p") == "p2p":
                try:
                    from paper_1205_2926_b200.dist import FourStepForwardP2P
                    import torch.distributed as dist
                    fs_p2p = FourStepForwardP2P(plans[0], lay, rank)
                    xa, xb_ = x0.clone(), x0.clone()
                    oa, ob = torch.empty_like(x0), torch.empty_like(x0)
                    fs_p2p(xa, oa, stream)
                    fs(xb_, recv, ob, stream)
                    ok = torch.tensor([1 if torch.equal(oa.view(torch.int64 if bits == 64 else torch.int32),
                                                        ob.view(torch.int64 if bits == 64 else torch.int32)) else 0],
                                      device=dev)
                    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
                    if int(ok.item()) == 1:
                        exchange = "p2p"
                    del xa, xb_, oa, ob
                except Exception as exc:  # no symmetric memory / P2P on this system
                    print(f"[bench] p2p exchange unavailable ({exc!r}); using NCCL all_to_all", file=sys.stderr)
                    fs_p2p = None
        else:
            x0 = torch.empty(batch * L, dtype=dt, device=dev)
            ntt.synth_uniform(x0, seed, 0, start=first * L, bound=cfg["primes"][0], stream=stream)
            x = x0.clone()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream.synchronize()

    info0 = plans[0].info()
    n_pass = info0.n_passes
    sched = [info0.pass_log2[i] for i in range(n_pass)]

    def pass_name(op, j):
        if n_pass == 1:
            return f"{op} (single pass, 2^{cfg['ell']})"
        return f"{op} pass {j} ({'row' if j == n_pass - 1 else 'column'} pass, 2^{sched[j]})"

    def step(evs=None):
        """One step: the whole hot path over this rank's batch.  evs: events between launches."""
        launches = 0
        if dist_c5:
            with torch.cuda.stream(stream):
                if exchange == "p2p":
                    phases = (("cols+p2p_exchange", lambda: fs_p2p.cols_exchange(x, stream)),
                              ("rows", lambda: fs_p2p.rows(outbuf, stream)))
                else:
                    phases = (("cols", lambda: fs.cols(x, stream)), ("all_to_all", lambda: fs.exchange(x, recv)),
                              ("rows", lambda: fs.rows(recv, outbuf, stream)))
                for name, fn in phases:
                    fn()
                    launches += ntt.last_launch_count() if name != "all_to_all" else 0
                    if evs is not None:
                        evs.append((name, torch.cuda.Event(enable_timing=True)))
                        evs[-1][1].record(stream)
            return launches
        if conv:
            for pl, (a, b) in zip(plans, work):
                pl.cyclic_convolve(a, b, stream=stream)
                launches += ntt.last_launch_count()
                if evs is not None:
                    evs.append(("conv", torch.cuda.Event(enable_timing=True)))
                    evs[-1][1].record(stream)
        else:
            # the plan's kernel passes one by one (ntt_transform_pass; in this order exactly
            # ntt_forward / ntt_inverse), so each kernel is timed on its own
            for op in cfg["ops"]:
                inv = op == "inv"
                for j in (reversed(range(n_pass)) if inv else range(n_pass)):
                    plans[0].transform_pass(x, j, inverse=inv, stream=stream)
                    launches += ntt.last_launch_count()
                    if evs is not None:
                        evs.append((pass_name(op, j), torch.cuda.Event(enable_timing=True)))
                        evs[-1][1].record(stream)
        return launches

    def reset_inputs():
        with torch.cuda.stream(stream):
            if conv:
                for a, b in work:
                    a.copy_(src[0]); b.copy_(src[1])
            else:
                x.copy_(x0)

    # ---- ALU roofline peak, measured live: register-only Alg. 3 butterflies
    p0 = cfg["primes"][0]
    W0 = root(p0, 4)
    sink = torch.zeros(4, dtype=torch.int64, device=dev)
    calib = []
    for it in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n = ntt.calibrate_butterfly(bits, p0, W0, (W0 << bits) // p0, 2048 if bits == 64 else 8192, sink,
                                    stream=stream)
        e1.record(stream)
        stream.synchronize()
        if it:
            calib.append(n / (e0.elapsed_time(e1) * 1e-3))
    calib_peak = max(calib)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    # ---- warmup
    for _ in range(args.warmup):
        reset_inputs()
        step()
    stream.synchronize()

    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local_rank)
    sampler.start()
    nvml = NvmlSampler(dev)
    time.sleep(0.3)
    step_ms, kernel_ms, launches = [], {}, 0
    nvml.start()  # exactly the timed region
    for _ in range(args.steps):
        reset_inputs()
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between timed steps, on the timed stream, before the start event
        start = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        evs = []
        launches += step(evs)
        stream.synchronize()
        prev = start
        for name, ev in evs:
            kernel_ms.setdefault(name, []).append(prev.elapsed_time(ev))
            prev = ev
        step_ms.append(start.elapsed_time(evs[-1][1]))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    nv_clocks = nvml.stop()
    smi_clocks = sampler.stop()
    clocks = nv_clocks or smi_clocks
    clock_max = clocks.get("sm_max_mhz") or 1965.0
    alu_peak = derived_alu_peak(bits, p0, sms, clock_max)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    bfly_rank = butterflies(cfg, batch) // (world if dist_c5 else 1)
    value = bfly_rank * world * args.steps / (total_ms * 1e-3)

    # ---- wk of every timed launch group: nontrivial Shoup products and algorithmic HBM bytes
    # (one read + one write of the data per kernel pass)
    wk = {}
    data_bytes = batch * L * wb
    if dist_c5:
        ell1 = cfg["ell"] // 2
        ell2 = cfg["ell"] - ell1
        n1, n2 = 1 << ell1, 1 << ell2
        ncol = -(-ell1 // (9 if bits == 64 else 10))  # column passes of <= kColsMax stages
        cols_w = ((n2 // world) * nontrivial(ell1) + (n1 - 1) * (n2 // world), 2 * ncol * (L // world) * wb)
        wk = {"cols": cols_w, "cols+p2p_exchange": cols_w, "all_to_all": (0, 2 * (L // world) * wb),
                "rows": ((n1 // world) * nontrivial(ell2), 2 * (L // world) * wb)}
    elif conv:
        # forward(a), forward(b) with the pointwise product fused, inverse: 3 transforms + L products,
        # bytes: a read+write, b read + a-hat read + c-hat write, c read+write
        wk = {"conv": (3 * batch * nontrivial(cfg["ell"]) + batch * L, 7 * data_bytes)}
    else:
        for op in cfg["ops"]:
            for j in range(n_pass):
                wk[pass_name(op, j)] = (pass_products(cfg["ell"], sched, j, batch), 2 * data_bytes)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in peaks else "B200_PROFILING.md (of fallback)"

    # ---- dominant kernel (largest share of the step) and its roofline
    share = {k: sum(v) for k, v in kernel_ms.items()}
    dom = max(share, key=share.get)
    dom_ms = statistics.mean(kernel_ms[dom])
    mults, alg_bytes = wk[dom]
    t_mul = mults / alu_peak * 1e3
    t_hbm = alg_bytes / (hbm_peak * 1e9) * 1e3
    frac_int, frac_hbm = t_mul / dom_ms, t_hbm / dom_ms
    alu_bound = t_mul >= t_hbm
    # whole step: the same bounds summed over every launch group of the step
    per_step = {k: len(v) / args.steps for k, v in kernel_ms.items()}
    st_mul = sum(wk[k][0] * n for k, n in per_step.items()) / alu_peak * 1e3
    st_hbm = sum(wk[k][1] * n for k, n in per_step.items()) / (hbm_peak * 1e9) * 1e3
    step_mean = total_ms / args.steps
    # DRAM bytes per launch of the dominant kernel from the committed `ncu --set full` capture
    # (profiles/ncu_traffic.json: config -> "per_pass" -> pass name -> dram_bytes_per_launch)
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        entry = prof.get(args.config, {})
        traffic = entry.get("per_pass", {}).get(dom, {}).get("dram_bytes_per_launch")
        if traffic is None and not entry.get("per_pass"):
            traffic = entry.get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {
        "bound": "alu" if alu_bound else "hbm",
        "kernel": dom + (" [3 launches: fwd(a), fwd(b)+pointwise, inv]" if conv else ""),
        "achieved": round((mults / (dom_ms * 1e-3) / 1e9) if alu_bound else (alg_bytes / (dom_ms * 1e-3) / 1e9), 2),
        "peak": round(alu_peak / 1e9, 2) if alu_bound else hbm_peak,
        "unit": "G nontrivial Shoup products/s" if alu_bound else "GB/s",
        "frac": round(max(frac_int, frac_hbm), 4),
        "frac_int": round(frac_int, 4),
        "frac_hbm": round(frac_hbm, 4),
        "T_MUL_ms": round(t_mul, 4), "T_HBM_ms": round(t_hbm, 4), "measured_ms": round(dom_ms, 4),
        "nontrivial_products_per_launch": mults,
        "algorithmic_bytes_per_launch": alg_bytes,
        "peak_source": (f"derived fmaheavy-pipe bound of one Alg. 3 Shoup product at {sms} SMs x {clock_max:.0f} MHz "
                        f"(DESIGN.md Roofline); HBM {hbm_peak} GB/s from {hbm_src}"),
        "calibrated_register_only_Gbfly_s": round(calib_peak / 1e9, 2),
        "traffic": traffic,
        "hbm": {"achieved_GBps": round(alg_bytes / (dom_ms * 1e-3) / 1e9, 1), "peak_GBps": hbm_peak,
                "frac": round(frac_hbm, 4), "peak_source": hbm_src},
        "step": {"T_MUL_ms": round(st_mul, 4), "T_HBM_ms": round(st_hbm, 4), "measured_ms": round(step_mean, 4),
                 "frac": round(max(st_mul, st_hbm) / step_mean, 4),
                 "frac_int": round(st_mul / step_mean, 4), "frac_hbm": round(st_hbm / step_mean, 4)},
    }

    # ---- e2e: the same step through the C-ABI host-buffer call (ntt_execute_host),
    # H2D of the inputs and D2H of the results inside the timed region
    e2e = None
    if dist_c5:
        h_in = x0.cpu().pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        ms = []
        for it in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            with torch.cuda.stream(stream):
                x.copy_(h_in, non_blocking=True)
                if exchange == "p2p":
                    fs_p2p(x, outbuf, stream)
                else:
                    fs(x, recv, outbuf, stream)
                h_out.copy_(outbuf, non_blocking=True)
            e1.record(stream)
            stream.synchronize()
            if it:
                ms.append(e0.elapsed_time(e1))
        e2e_ms = sum(ms)
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": bfly_rank * world * len(ms) / (float(t.item()) * 1e-3), "unit": "butterflies/s",
               "h2d_bytes_per_step": x.numel() * wb, "d2h_bytes_per_step": x.numel() * wb,
               "api": "pinned shard copies + " + ("FourStepForwardP2P (cols with fused P2P exchange, rows)"
                                                   if exchange == "p2p" else
                                                   "FourStepForward (cols, NCCL all_to_all_single, rows)")}
    elif not conv:
        ops = 0
        for op in cfg["ops"]:
            ops |= ntt.NTT_OP_FORWARD if op == "fwd" else ntt.NTT_OP_INVERSE
        h_in = torch.empty(batch * L, dtype=dt, pin_memory=True)
        h_in.copy_(x0.cpu())
        h_out = torch.empty_like(h_in).pin_memory()
        # device scratch of the host pipeline: room for its 4-slot ring (>= 4 transforms, or >= 64 MiB), so
        # the H2D copy of one chunk, the transform of the next and the D2H of a third overlap
        dbuf_words = min(batch * L, max(4 * L, (64 << 20) // wb))
        dbuf = torch.empty(dbuf_words, dtype=dt, device=dev)
        for _ in range(2):
            plans[0].execute_host(ops, h_in, h_out, dbuf, stream=stream)
        stream.synchronize()
        ms = []
        for _ in range(max(3, min(args.steps, 10))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plans[0].execute_host(ops, h_in, h_out, dbuf, stream=stream)
            e1.record(stream)
            stream.synchronize()
            ms.append(e0.elapsed_time(e1))
        e2e_ms = sum(ms)
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": bfly_rank * world * len(ms) / (e2e_ms * 1e-3), "unit": "butterflies/s",
               "h2d_bytes_per_step": batch * L * wb, "d2h_bytes_per_step": batch * L * wb,
               "api": "ntt_execute_host (pinned host in/out, chunked H2D/compute/D2H pipeline)"}
    else:
        # C3 end to end: host a,b -> device, 3 convolutions, residues back
        h_a = src[0].cpu().pin_memory()
        h_b = src[1].cpu().pin_memory()
        h_out = torch.empty((len(plans),) + tuple(h_a.shape), dtype=dt).pin_memory()
        ms = []
        for it in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            with torch.cuda.stream(stream):
                for i, (pl, (a, b)) in enumerate(zip(plans, work)):
                    a.copy_(h_a, non_blocking=True)
                    b.copy_(h_b, non_blocking=True)
                    pl.cyclic_convolve(a, b, stream=stream)
                    h_out[i].copy_(a, non_blocking=True)
            e1.record(stream)
            stream.synchronize()
            if it:
                ms.append(e0.elapsed_time(e1))
        e2e_ms = sum(ms)
        if world > 1:  # max over ranks, like every other timing
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": bfly_rank * world * len(ms) / (e2e_ms * 1e-3), "unit": "butterflies/s",
               "h2d_bytes_per_step": 2 * batch * L * wb * len(plans),
               "d2h_bytes_per_step": batch * L * wb * len(plans),
               "api": "torch pinned copies + ntt_cyclic_convolve per prime"}

    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "butterflies/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if dist_c5 else cfg["scaling"], "vs_baseline": None,
            "dtype": "u64" if bits == 64 else "u32",
            "data": "synthetic: seeded counter-based uniform residues generated in HBM (synth/ definition)",
            "config": config_dict(cfg, world),
            "passes": sched if not dist_c5 else None,
            "exchange": (("all-to-all fused into the column pass (P2P stores over NVLink, symmetric memory)"
                          if exchange == "p2p" else "one NCCL all_to_all_single") if dist_c5 else None),
            "hbm_GBps": round(sum(wk[k][1] * len(v) for k, v in kernel_ms.items()) * world
                              / (total_ms * 1e-3) / 1e9, 1),
            "roofline": roofline,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "clocks_nvidia_smi": smi_clocks,
            "kernel_ms_mean": {k: round(statistics.mean(v), 4) for k, v in kernel_ms.items()},
        }
    return out


# ------------------------------------------------------------------ oracle (CPU) arm
def oracle_sample(cfg):
    """Bounded sample of the workload for the CPU oracle: (transforms, seconds-sized)."""
    return {"c1": 1, "c2": 4096, "c3": 1, "c4": 1, "c5": 1}[cfg["key"]]


def run_oracle_steps(cfg, steps, warmup, nthreads):
    """The oracle (oracle/, plain Alg. 1 with 128-bit %) on a bounded sample of the workload."""
    import numpy as np

    import oracle
    import synth
    L = 1 << cfg["ell"]
    seed = synth.config_seed(cfg["seed_cfg"])
    if cfg["key"] == "c5":  # a 2^28 transform is ~45 thread-seconds: use a 2^24 prefix-sized sample
        ell = 24
    else:
        ell = cfg["ell"]
    Ls = 1 << ell
    nb = oracle_sample(cfg)
    if cfg["ops"] == ("conv",):
        half = Ls // 2
        a = np.zeros((nb, Ls), dtype=np.uint64)
        b = np.zeros((nb, Ls), dtype=np.uint64)
        a[:, :half] = synth.uniform_bits(seed, 0, 0, nb * half, 20).reshape(nb, half)
        b[:, :half] = synth.uniform_bits(seed, 1, 0, nb * half, 20).reshape(nb, half)
    else:
        x = synth.uniform_mod(seed, 0, 0, nb * Ls, cfg["primes"][0]).reshape(nb, Ls)
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        for p in cfg["primes"]:
            w = root(p, Ls)
            if cfg["ops"] == ("conv",):
                fa = oracle.ntt_forward(p, w, a, nthreads=nthreads)
                fb = oracle.ntt_forward(p, w, b, nthreads=nthreads)
                oracle.ntt_inverse(p, w, oracle.pointwise(p, fa, fb, scale_L=Ls), nthreads=nthreads)
            else:
                y = x
                for op in cfg["ops"]:
                    y = (oracle.ntt_forward if op == "fwd" else oracle.ntt_inverse)(p, w, y, nthreads=nthreads)
        if it >= warmup:
            times.append(time.perf_counter() - t0)
    n_ntt = 3 if cfg["ops"] == ("conv",) else len(cfg["ops"])
    bfly = (Ls // 2) * ell * n_ntt * nb * len(cfg["primes"])
    value = bfly * len(times) / sum(times)
    sample = (f"{nb} transform(s) of 2^{ell} x {n_ntt} NTT(s) x {len(cfg['primes'])} prime(s) per step"
              + (" (2^24 stands in for the 2^28 transform)" if cfg["key"] == "c5" else ""))
    return value, sample, sum(times) / len(times)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config], key=args.config)

    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus < 1:
        sys.exit(f"bench.py: --gpus must be >= 1 (got {args.gpus})")
    if env_world is not None and int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} does not match WORLD_SIZE={env_world}")
    if env_world is None and args.gpus > 1 and args.impl == "native":
        # one process per GPU: re-launch this command under torch.distributed.run with N ranks
        import socket
        import torch
        n_dev = torch.cuda.device_count()
        if n_dev < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but only {n_dev} CUDA device(s) are visible")
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    # the reference arm (CPU oracle) runs on rank 0 alone, also when --gpus N is given without torchrun
    world = int(env_world) if env_world is not None else args.gpus
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    # plumbing test hook (not for measurements): every rank on GPU 0 over gloo, so the N > 1 code path
    # (sharding, max-over-ranks timing, the JSON line) can be exercised on a one-GPU box
    if os.environ.get("NTT_BENCH_PLUMBING_1GPU") == "1":
        local_rank = 0
    nthreads = len(os.sched_getaffinity(0))

    if args.impl == "reference":
        # The reference arm is the CPU oracle (there is no reference implementation to
        # install).  Rank 0 only; other ranks exit without work.
        if rank != 0:
            return
        value, sample, sec = run_oracle_steps(cfg, args.steps, args.warmup, nthreads)
        out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "butterflies/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
               "scaling": "strong" if (cfg["key"] == "c5" and world > 1) else cfg["scaling"], "vs_baseline": None,
               "dtype": "u64" if cfg["bits"] == 64 else "u32",
               "data": "synthetic: seeded counter-based uniform residues (synth/ definition)",
               "config": config_dict(cfg, world),
               "cpu_baseline": {"value": value, "unit": "butterflies/s", "cores": nthreads, "kind": "oracle",
                                "sample": sample, "cpu": cpu_model()},
               "e2e": {"value": value, "unit": "butterflies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if os.environ.get("NTT_BENCH_PLUMBING_1GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_native(args, cfg, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            value, sample, _ = run_oracle_steps(cfg, 1, 0, nthreads)
            out["cpu_baseline"] = {"value": value, "unit": "butterflies/s", "cores": nthreads, "kind": "oracle",
                                   "sample": sample, "cpu": cpu_model()}
        elif world > 1:
            out["cpu_baseline"] = None
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
