"""Per-call wall-clock breakdown of one hot-path step (diagnostic, not a benchmark)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2405_15197_b200 import binding as B

cfg = sys.argv[1] if len(sys.argv) > 1 else "octet100"
n = int(cfg.replace("octet", ""))
lat = synth.graded_radii(synth.octet(n, n, n), 0.03, 0.06, axis=0)
xyz, ends, rend = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (lat.xyz, lat.ends, lat.r_end))
h = B.lmm_create(0, torch.cuda.current_stream().cuda_stream)
out = torch.empty((1 << 28) * 50, dtype=torch.uint8, device="cuda")
for it in range(4):
    ts = {}
    def tm(name, f):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
        ts[name] = (time.perf_counter() - t0) * 1e3
        return r
    tm("load", lambda: B.lmm_load_lattice(h, xyz, ends, rend))
    tm("build", lambda: B.lmm_build_metamesh(h))
    T = tm("triangulate", lambda: B.lmm_triangulate(h, 1e-3))
    def em():
        for f in range(0, T, 1 << 28):
            B.lmm_write_triangles(h, f, min(1 << 28, T - f), out)
    tm("emit", em)
    print(it, {k: round(v, 2) for k, v in ts.items()}, "total", round(sum(ts.values()), 1), flush=True)

# ---- variants: bench-style loop (no syncs) with timing events and/or nvidia-smi sampling
import subprocess
def loop(tag, timing=False, smi=False, steps=3):
    B.lmm_timing(h, timing)
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.sw_power_cap", "--format=csv,noheader",
                          "-lms", "200"], stdout=subprocess.DEVNULL) if smi else None
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(steps):
        B.lmm_load_lattice(h, xyz, ends, rend); B.lmm_build_metamesh(h); T = B.lmm_triangulate(h, 1e-3)
        for f in range(0, T, 1 << 28):
            B.lmm_write_triangles(h, f, min(1 << 28, T - f), out)
    torch.cuda.synchronize(); ms = (time.perf_counter() - t0) * 1e3 / steps
    if p: p.terminate(); p.wait()
    B.lmm_timing(h, False)
    print(tag, "ms/step", round(ms, 1), flush=True)
loop("plain")
loop("timing", timing=True)
loop("smi", smi=True)
loop("timing+smi", timing=True, smi=True)
