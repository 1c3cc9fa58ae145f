"""Probe: meta-mesh builds (context 1) concurrent with emission (context 0), two host threads.
python tools/overlap_probe2.py [config] [reps]"""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2405_15197_b200 import binding as B

cfg = sys.argv[1] if len(sys.argv) > 1 else "octet100"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
lat, _, _ = bench.make_config(cfg, 0, 1)
xyz_d, ends_d, rend_d = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (lat.xyz, lat.ends, lat.r_end))
streams = [torch.cuda.Stream() for _ in range(2)]
hs = [B.lmm_create(0, s.cuda_stream) for s in streams]
out = torch.empty(bench.EMIT_CHUNK * bench.STL, dtype=torch.uint8, device="cuda")
for h in hs:
    B.lmm_load_lattice(h, xyz_d, ends_d, rend_d)
    B.lmm_build_metamesh(h)
T = B.lmm_triangulate(hs[0], 1e-3)
torch.cuda.synchronize()


def emit():
    for _ in range(reps):
        for f in range(0, T, bench.EMIT_CHUNK):
            B.lmm_write_triangles(hs[0], f, min(bench.EMIT_CHUNK, T - f), out)
    streams[0].synchronize()


def build():
    for _ in range(reps):
        B.lmm_load_lattice(hs[1], xyz_d, ends_d, rend_d)
        B.lmm_build_metamesh(hs[1])
    streams[1].synchronize()


def timed(fns):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=f) for f in fns]
    for t in th: t.start()
    for t in th: t.join()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


emit(); build()
for r in range(2):
    te, tb = timed([emit]), timed([build])
    tboth = timed([emit, build])
    print(f"{cfg}: emit {te:.1f} ms, build {tb:.1f} ms, sum {te + tb:.1f}, concurrent {tboth:.1f} ms")
