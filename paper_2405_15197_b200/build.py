"""Build liblmm.so (sm_100a) in-tree with nvcc.

    python -m paper_2405_15197_b200.build        # or __graft_entry__.build()

metamesh.cu and spill.cu are compiled with -fmad=false: its binary32 topology decisions follow the
fixed-order specification of DESIGN.md Sec. 4 (no implicitly contracted multiply-adds; the
specification's own FMAs are written explicitly).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(OUT_DIR, "liblmm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
SOURCES = {
    "lmm_api.cu": [],
    "lattice.cu": [],
    "scan.cu": [],
    "metamesh.cu": ["-fmad=false"],
    "spill.cu": ["-fmad=false"],
    "triangulate.cu": [],
}


def _stale(obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    # LMM_NVCC_EXTRA: extra nvcc flags for tuning experiments (a change forces a rebuild)
    extra_all = os.environ.get("LMM_NVCC_EXTRA", "").split()
    stamp = os.path.join(OUT_DIR, "flags.txt")
    old = open(stamp).read() if os.path.exists(stamp) else ""
    if old != " ".join(extra_all):
        force = True
        with open(stamp, "w") as f:
            f.write(" ".join(extra_all))
    headers = [os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "lmm.h"))
    objs = []
    procs = []
    for src, extra in SOURCES.items():
        s = os.path.join(SRC, src)
        o = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s, *headers, __file__]):
            cmd = [NVCC, *ARCH, *COMMON, *extra, *extra_all, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out.decode()}")
        if verbose and out:
            print(out.decode())
    if force or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs]
        r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout.decode()}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
