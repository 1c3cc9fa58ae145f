"""configs[3] executed whole on ONE B200: the ~1.0B-strut BCC lattice (250 x 250 x 2000 cells) as the
8 z-slabs the 8-GPU run gives its ranks (bench.make_config("bcc250", r, 8): slab + 2-layer halo,
emit masks), meta-meshed, triangulated and emitted one after another on one device (device output
in bench.py's 2^28-triangle chunks).  Each slab is timed with CUDA events around
load + build + triangulate + emit (inputs already on the device, as bench.py's `value`); the
sum is the single-GPU time of the billion-strut job, and the max over slabs is what 8 GPUs
would take under weak scaling with no other cost (the only collective is an all-gather of 8
counts).  Not the driver's bench line: a measurement tool.

python tools/billion_serial.py [CE] > billion.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import bench
from paper_2405_15197_b200 import binding as B


def main():
    ce = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
    world = 8
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    out = torch.empty(bench.EMIT_CHUNK * bench.STL, dtype=torch.uint8, device="cuda")
    slabs, t_all = [], time.time()
    for r in range(world):
        tg = time.time()
        lat, (nmask, smask), desc = bench.make_config("bcc250", r, world)
        gen_s = time.time() - tg
        xyz = torch.from_numpy(np.ascontiguousarray(lat.xyz)).cuda()
        ends = torch.from_numpy(np.ascontiguousarray(lat.ends)).cuda()
        rend = torch.from_numpy(np.ascontiguousarray(lat.r_end)).cuda()
        nm, sm = torch.from_numpy(nmask).cuda(), torch.from_numpy(smask).cuda()
        h = B.lmm_create(0, stream.cuda_stream)

        def step():
            B.lmm_load_lattice(h, xyz, ends, rend)
            B.lmm_set_emit_mask(h, nm, sm)
            B.lmm_build_metamesh(h)
            T = B.lmm_triangulate(h, ce)
            for f in range(0, T, bench.EMIT_CHUNK):
                B.lmm_write_triangles(h, f, min(bench.EMIT_CHUNK, T - f), out)
            return T

        step()   # warm-up (allocations, attributes)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        T = step()
        e1.record(stream)
        torch.cuda.synchronize()
        st = B.lmm_metamesh_stats(h)
        slabs.append({"rank": r, "ms": e0.elapsed_time(e1), "struts_owned": int(smask.sum()),
                      "struts_local": int(lat.n_struts), "nodes_local": int(lat.n_nodes), "triangles": int(T),
                      "error_nodes": int(st["n_error_nodes"]), "generate_s": round(gen_s, 1)})
        B.lmm_destroy(h)
        del xyz, ends, rend, nm, sm, lat
        torch.cuda.empty_cache()
        print(json.dumps(slabs[-1]), file=sys.stderr, flush=True)
    ms_sum = sum(s["ms"] for s in slabs)
    ms_max = max(s["ms"] for s in slabs)
    S = sum(s["struts_owned"] for s in slabs)
    T = sum(s["triangles"] for s in slabs)
    print(json.dumps({
        "workload": "configs[3]: BCC 250x250x2000 cells (1.0B struts) as 8 z-slabs + 2-layer halos, one B200, serial",
        "chord_error": ce, "struts": S, "triangles": T, "error_nodes": sum(s["error_nodes"] for s in slabs),
        "device_ms_sum": ms_sum, "struts_per_s_one_gpu": S / (ms_sum / 1e3), "triangles_per_s_one_gpu": T / (ms_sum / 1e3),
        "device_ms_max_slab": ms_max, "struts_per_s_8gpu_weak_bound": S / (ms_max / 1e3),
        "stl_bytes": 50 * T, "wall_s_incl_generation": round(time.time() - t_all, 1), "slabs": slabs}))


if __name__ == "__main__":
    main()
