"""CPU-side checks of the boundary: liblmm.so builds for sm_100a, loads, and exports every
function include/lmm.h declares; the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lmm.h")).read()
    return sorted(set(re.findall(r"LMM_API\s+[\w\s\*]+?\b(lmm_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2405_15197_b200 import build as b
    return b.build()


def test_header_declares_the_problem_statement_calls():
    names = _declared()
    for must in ("lmm_create", "lmm_load_lattice", "lmm_build_metamesh", "lmm_triangulate", "lmm_write_triangles",
                 "lmm_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (lmm_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    h = ctypes.CDLL(lib)
    for n in _declared():
        getattr(h, n)


def test_library_is_sm100a_code(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _packed_adds_of_products(ptx):
    """Packed adds (add/sub .f32x2) fed -- through any chain of bit moves -- by a packed
    product (mul .f32x2): the pattern ptxas contracts into FFMA2 even under -fmad=false."""
    bad = []
    for body in re.split(r"\.(?:entry|func)\s", ptx)[1:]:
        name = body.split("(", 1)[0].strip()
        ins = []
        for line in body.splitlines():
            line = line.strip()
            m = re.match(r"(?:@!?%\w+\s+)?([a-z][\w.]*)\s+(.*);", line)
            if not m or line.startswith("//"):
                continue
            op, args = m.group(1), m.group(2)
            if op.startswith(("st.", "bra", "ret", "bar", "setp", "atom", "red.")):
                continue
            dst, _, src = args.partition(",") if not args.startswith("{") else args.partition("},")
            ins.append((op, set(re.findall(r"%\w+", dst)), set(re.findall(r"%\w+", src))))
        taint, changed = set(), True
        while changed:                                  # fixed point (loops carry values back)
            changed = False
            for op, d, sr in ins:
                if re.match(r"mul(\.rn)?\.f32x2", op):
                    new = d - taint
                elif op.startswith(("fma", "add", "sub", "mul", "div", "sqrt", "rcp")) or ".f32" in op:
                    new = set()                         # arithmetic consumes the product
                else:
                    new = d - taint if sr & taint else set()
                if new:
                    taint |= new
                    changed = True
        bad += [(name, op) for op, d, sr in ins if re.match(r"(add|sub)(\.rn)?\.f32x2", op) and sr & taint]
    return bad


def test_metamesh_has_no_contractible_packed_multiply_add(lib):
    """The meta-mesh decisions follow the binary32 specification op by op:
    scalar code is compiled -fmad=false, but ptxas contracts a packed add of a packed product
    into FFMA2 regardless.  The PTX of metamesh.cu (same flags) must hold no such pair -- the
    side function's fused multiply-adds are written as explicit fma.rn.f32x2 (Sec. 4.4)."""
    import tempfile
    from paper_2405_15197_b200 import build as b
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "mm.ptx")
        subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=compute_100a", "-O3", "-std=c++17",
                        "--expt-relaxed-constexpr", *b.SOURCES["metamesh.cu"], "-ptx",
                        os.path.join(b.SRC, "metamesh.cu"), "-o", out], check=True, capture_output=True)
        ptx = open(out).read()
    assert re.search(r"mul\.rn\.f32x2", ptx) and re.search(r"fma\.rn\.f32x2", ptx)
    # the checker itself must see the hazard: a packed add of a packed product
    probe = ".entry probe(\n\tmul.rn.f32x2 %rd1, %rd2, %rd3;\n\tmov.b64 {%r1, %r2}, %rd1;\n" \
            "\tmov.b64 %rd4, {%r1, %r2};\n\tadd.rn.f32x2 %rd5, %rd4, %rd6;\n"
    assert _packed_adds_of_products(probe)
    bad = _packed_adds_of_products(ptx)
    assert not bad, bad[:3]


def test_no_gpu_means_loud_failure(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_15197_b200 import LmmError, lmm_create
    with pytest.raises(LmmError):
        lmm_create(0)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2405_15197_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "mm_oracle" not in txt and "liborc" not in txt, f
