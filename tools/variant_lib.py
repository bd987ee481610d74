"""Build an experimental copy of libntt_b200.so with extra nvcc flags (e.g. -DNTT_TMA_LE64=3),
recompiling only the listed sources and linking them with the default objects.
    python tools/variant_lib.py NAME "FLAGS" [src.cu ...]  -> abvar/libntt_NAME.so (gitignored; travels to the GPU box)
Load it with NTT_B200_LIB=abvar/libntt_NAME.so (tools/time_cfg.py)."""
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_1205_2926_b200"))
import _build  # noqa: E402


def main():
    name, flags = sys.argv[1], shlex.split(sys.argv[2])
    srcs = sys.argv[3:] or ["ntt_contig_tma.cu"]
    _build.build()
    out = os.path.join(ROOT, os.environ.get("NTT_VARIANT_DIR", "abvar"))
    os.makedirs(os.path.join(out, name), exist_ok=True)
    objs = []
    for s in _build.SOURCES:
        if s in srcs:
            o = os.path.join(out, name, s.replace(".cu", ".o"))
            cmd = [_build.NVCC, *_build.FLAGS, *flags, "-c", os.path.join(_build.CSRC, s), "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            open(o + ".log", "w").write(r.stdout + r.stderr)
            if r.returncode:
                sys.exit(r.stderr[-3000:])
            objs.append(o)
        else:
            objs.append(os.path.join(_build.BUILD, s.replace(".cu", ".o")))
    lib = os.path.join(out, f"libntt_{name}.so")
    subprocess.run([_build.NVCC, "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
                    *objs, "-o", lib], check=True)
    print(lib)


if __name__ == "__main__":
    main()
