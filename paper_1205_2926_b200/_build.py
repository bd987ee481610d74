"""Build libntt_b200.so in-tree with nvcc for sm_100a (no JIT cache, so the .so
travels to the GPU box with the repo snapshot)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libntt_b200.so")
BUILD = os.path.join(HERE, "build")
# variants: the production library and the range-audit debug build (-DNTT_RANGE_AUDIT)
VARIANTS = {
    "": (LIB, BUILD, []),
    "audit": (os.path.join(HERE, "libntt_b200_audit.so"), os.path.join(HERE, "build_audit"),
              ["-DNTT_RANGE_AUDIT", "-Xptxas", "-O1"]),  # a checking build: ptxas -O1 keeps it quick
}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["plan.cu", "ntt_kernels.cu", "ntt_cols.cu", "ntt_contig_tma.cu", "ntt_cols_tma.cu", "ntt_split2.cu", "synth.cu"]
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"), "-I", CSRC,
]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "ntt_b200.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _build_variant(ex, name, force, deps):
    lib, bdir, extra = VARIANTS[name]
    os.makedirs(bdir, exist_ok=True)
    headers = [d for d in deps if not d.endswith(".cu")]

    def compile_one(src):
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        if not force and not _stale(obj, headers + [os.path.join(CSRC, src)]):
            return obj
        cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(bdir, src + ".log"), "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {src} ({name or 'production'} build):\n{r.stderr[-4000:]}")
        return obj

    return lib, [ex.submit(compile_one, src) for src in SOURCES]


def _link(lib, objs):
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, lib)


def build(force: bool = False, verbose: bool = False, variants=("", "audit")) -> str:
    """Compile every variant's objects in one pool and link each stale library; returns the
    production library's path."""
    deps = _deps()
    todo = [v for v in variants if force or _stale(VARIANTS[v][0], deps)]
    if todo:
        with cf.ThreadPoolExecutor(max(1, min(len(SOURCES) * len(todo), os.cpu_count() or 8))) as ex:
            jobs = [_build_variant(ex, v, force, deps) for v in todo]
            for lib, futs in jobs:
                _link(lib, [f.result() for f in futs])
                if verbose:
                    print(f"built {lib}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
