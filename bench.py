#!/usr/bin/env python
"""Benchmark of the lattice meta-meshing + triangulation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config octet100]

A step is one pass of the whole hot path over one lattice resident in HBM: device CSR
build + degree buckets (lmm_load_lattice), per-node meta-mesh (lmm_build_metamesh),
count pass + scans at chord error CE (lmm_triangulate), and emission of every
triangle as binary-STL records into an HBM output buffer (lmm_write_triangles, in
chunks of 2^28 triangles = 13.4 GB, far larger than the 126 MB L2).  Multi-GPU: one
process per GPU, each owning one spatial block of the lattice (weak scaling), timed
as the max over ranks.  Prints ONE JSON line on rank 0.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "struts/s meta-meshing and triangles/s triangulation at 1/2/4/8 B200; % HBM peak"
STL = 50
EMIT_CHUNK = 1 << int(os.environ.get("LMM_BENCH_CHUNK_LOG2", "28"))   # triangles per device output chunk


def make_config(name: str, rank: int = 0, world: int = 1):
    """Synthetic workload of BASELINE.json's configs.  Weak scaling: the global lattice is
    `world` blocks stacked along z; rank r gets its slab plus a 2-layer halo and the emit
    masks of the nodes / struts it owns (paper_2405_15197_b200.partition)."""
    from paper_2405_15197_b200 import partition as P
    import re
    m = re.fullmatch(r"(octet|bcc|stoch)(\d+)", name)
    fam, n = (m.group(1), int(m.group(2))) if m else (name, 0)
    if fam == "octet":
        # configs[1] (octet100: 24.12M struts) and configs[4]'s fixed meta-mesh (octet160: 98.6M)
        k_top = 2 * n * world
        k_lo, k_hi = P.window(rank, world, k_top) if world > 1 else (0, k_top)
        lat = synth.octet_window(n, n, n * world, k_lo, k_hi, radius=0.03, r_max=0.06)
        masks = P.emit_masks(lat.ijk[:, 2], lat.ends, rank, world, k_top) if world > 1 else (None, None)
        desc = (f"octet-truss {n}x{n}x{n} cells per GPU (global {n}x{n}x{n * world}), conical struts "
                f"(node radii graded 0.03-0.06 along x, pitch 1)")
    elif fam == "bcc" and name != "bcc10":
        # configs[3]: the ~1B-strut BCC lattice of 8 GPUs = 8 blocks of 250^3 cells (125M struts each)
        k_top = 2 * n * world
        k_lo, k_hi = P.window(rank, world, k_top) if world > 1 else (0, k_top)
        lat = synth.bcc_window(n, n, n * world, k_lo, k_hi, radius=0.05)
        masks = P.emit_masks(lat.ijk[:, 2], lat.ends, rank, world, k_top) if world > 1 else (None, None)
        desc = (f"BCC {n}x{n}x{n} cells per GPU (global {n}x{n}x{n * world}, {8 * n ** 3 * world / 1e9:.3f}B struts), "
                f"uniform radius 0.05, pitch 1")
    elif fam == "stoch":
        # configs[2]: ONE stochastic Voronoi-style lattice, degrees 3..30, ~1e8 struts per GPU at n = 290,
        # n x n x (n * world) nodes; rank r gets its z-slab plus a 4-layer halo (struts span up to 2
        # layers, so the far ends of its struts see their whole neighbourhood)
        k_top = n * world - 1
        k_lo, k_hi = P.window(rank, world, k_top, halo=4) if world > 1 else (0, k_top)
        lat = synth.stochastic_window(n, n * world, k_lo, k_hi, seed=0)
        masks = P.emit_masks(lat.ijk[:, 2], lat.ends, rank, world, k_top) if world > 1 else (None, None)
        desc = (f"stochastic Voronoi-style lattice {n}x{n}x{n} nodes per GPU (global {n}x{n}x{n * world}): jittered grid, "
                "Zipf target degrees 3-30, cone radii U(0.02, 0.04), >=25 deg between struts at a node "
                "(synth.stochastic_window: blocks of 10 layers + seams, spatially partitioned along z)")
    elif name == "bcc10":
        lat = synth.bcc(10, 10, 10)
        masks = (None, None)
        desc = "BCC 10x10x10 cells, uniform strut radius 0.05 (pitch 1)"
    else:
        raise SystemExit(f"unknown config {name}")
    return lat, masks, desc


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.lines, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def _sample_lattice(config: str, n: int):
    """A small lattice of the same family as `config` (for the oracle's bounded samples)."""
    if config.startswith("bcc"):
        return synth.bcc(n, n, n), f"bcc {n}x{n}x{n}"
    if config.startswith("stoch"):
        side = int(round((n ** 3 * 8) ** (1 / 3)))
        return synth.stochastic_window(side, side, 0, side - 1, seed=0), f"stochastic {side}^3"
    return synth.graded_radii(synth.octet(n, n, n), 0.03, 0.06, axis=0), f"octet {n}x{n}x{n} graded"


def cpu_baseline(ce, config: str = "octet100", sweep=None, budget_s: float = 20.0):
    """The oracle as it stands, single-threaded on this host, on a bounded sample of the
    same workload family -- a reported baseline, not the target."""
    import oracle
    oracle.build_oracle()
    ces = sweep or [ce]
    n = 6
    while True:
        lat, name = _sample_lattice(config, n)
        t0 = time.perf_counter()
        orc = oracle.Oracle.from_lattice(lat)
        if not sweep:
            orc.metamesh()
        else:
            orc.metamesh()
            t0 = time.perf_counter()    # sweep: the meta-mesh is built outside the timed region
        T = 0
        for c in ces:
            Tc = orc.triangulate(c)
            for f in range(0, Tc, 1 << 21):
                orc.write_triangles(f, min(1 << 21, Tc - f))
            T += Tc
        dt = time.perf_counter() - t0
        if dt > budget_s / 4 or n >= 24:
            break
        n = int(n * 1.5)
    v, unit = (T / dt, "triangles/s") if sweep else (lat.n_struts / dt, "struts/s")
    return {"value": v, "unit": unit, "cores": 1, "kind": "oracle",
            "sample": f"{name} ({lat.n_struts} struts, {T} triangles, CE={ces}) in {dt:.1f} s",
            "triangles_per_s": T / dt}


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on bounded samples."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build_oracle()
    lat, name = _sample_lattice(args.config, 8)
    sweep = [float(x) for x in args.ce_sweep.split(",") if x] if args.ce_sweep else None
    fixed = oracle.Oracle.from_lattice(lat) if sweep else None
    if sweep:
        fixed.metamesh()     # the sweep re-triangulates one meta-mesh built outside the timed region

    def step():
        orc = fixed
        if orc is None:
            orc = oracle.Oracle.from_lattice(lat)
            orc.metamesh()
        T = 0
        for ce in sweep or [args.ce]:
            Tc = orc.triangulate(ce)
            for f in range(0, Tc, 1 << 21):
                orc.write_triangles(f, min(1 << 21, Tc - f))
            T += Tc
        return T
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        T = step()
    dt = (time.perf_counter() - t0) / args.steps
    v, unit = (T / dt, "triangles/s") if sweep else (lat.n_struts / dt, "struts/s")
    sample = f"{name} ({lat.n_struts} struts, {T} triangles) per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": sample, "chord_error": sweep or args.ce},
        "cpu_baseline": {"value": v, "unit": unit, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="octet100")
    ap.add_argument("--ce", type=float, default=1e-3)
    ap.add_argument("--ce-sweep", default="",
                    help="comma-separated chord errors: re-triangulate ONE meta-mesh (built before the timed "
                         "region) at each CE per step (configs[4], multi-resolution reuse)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2405_15197_b200 import binding as B

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # LMM_BENCH_ONE_GPU=1: every rank on cuda:0 with a gloo group (tests the multi-rank path
    # on a single device; timings are then not scaling numbers)
    one_gpu = os.environ.get("LMM_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    coll_dev = "cpu" if one_gpu else "cuda"
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    lat, (node_mask, strut_mask), desc = make_config(args.config, rank, world)
    S, N = lat.n_struts, lat.n_nodes
    S_own = int(strut_mask.sum()) if strut_mask is not None else S
    xyz_h = torch.from_numpy(np.ascontiguousarray(lat.xyz)).pin_memory()
    ends_h = torch.from_numpy(np.ascontiguousarray(lat.ends)).pin_memory()
    rend_h = torch.from_numpy(np.ascontiguousarray(lat.r_end)).pin_memory()
    xyz_d, ends_d, rend_d = xyz_h.cuda(), ends_h.cuda(), rend_h.cuda()
    stream = torch.cuda.current_stream()
    h = B.lmm_create(local, stream.cuda_stream)
    out = torch.empty(EMIT_CHUNK * STL, dtype=torch.uint8, device="cuda")

    nmask_d = torch.from_numpy(node_mask).cuda() if node_mask is not None else None
    smask_d = torch.from_numpy(strut_mask).cuda() if strut_mask is not None else None
    cnt = torch.zeros(1, dtype=torch.int64, device=coll_dev)
    cnts = torch.zeros(world, dtype=torch.int64, device=coll_dev)
    offsets = {"base": 0, "total": 0}

    sweep = [float(x) for x in args.ce_sweep.split(",") if x] if args.ce_sweep else None
    ces = sweep or [args.ce]
    per_ce, per_ce_path = {}, {}

    def load_and_build():
        B.lmm_load_lattice(h, xyz_d, ends_d, rend_d)
        if world > 1:
            B.lmm_set_emit_mask(h, nmask_d, smask_d)
        B.lmm_build_metamesh(h)

    def step():
        if not sweep:
            load_and_build()
        T = 0
        for ce in ces:
            Tc = B.lmm_triangulate(h, ce)
            if world > 1:   # global output offsets: all-gather of the per-rank triangle counts
                cnt.fill_(Tc)
                parts = list(cnts.split(1))
                dist.all_gather(parts, cnt)
                c = [int(x) for x in torch.cat(parts).tolist()]
                offsets["base"], offsets["total"] = sum(c[:rank]), sum(c)
            for f in range(0, Tc, EMIT_CHUNK):
                B.lmm_write_triangles(h, f, min(EMIT_CHUNK, Tc - f), out)
            per_ce[ce] = Tc
            per_ce_path[ce] = B.lmm_emit_path(h)
            T += Tc
        return T

    if sweep:
        load_and_build()    # the fixed meta-mesh: built once, outside the timed region

    for _ in range(max(args.warmup, 0)):
        T = step()
    torch.cuda.synchronize()
    B.lmm_reset_kernel_times(h)
    B.lmm_timing(h, True)
    l0 = B.lmm_launch_count(h)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            T = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    B.lmm_timing(h, False)
    launches = B.lmm_launch_count(h) - l0
    st = B.lmm_metamesh_stats(h)
    ms = ev0.elapsed_time(ev1) / args.steps
    kt = B.lmm_kernel_times(h)
    t = torch.tensor([ms], dtype=torch.float64, device=coll_dev)
    tot = torch.tensor([float(S_own), float(T)], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms_max = float(t.item())
    S_all, T_all = float(tot[0].item()), float(tot[1].item())

    # ---- e2e: host inputs (pinned) -> device -> host triangle records, through the C-ABI
    e2e = None
    if args.e2e_steps > 0 and not sweep:
        ring = torch.empty((1 << 24) * STL, dtype=torch.uint8).pin_memory()
        h2 = h           # same context, host inputs/outputs (its device-resident copies are replaced)
        del out
        torch.cuda.empty_cache()
        chunk = 1 << 24

        def e2e_step():
            B.lmm_load_lattice(h2, xyz_h, ends_h, rend_h)
            if world > 1:
                B.lmm_set_emit_mask(h2, node_mask, strut_mask)
            B.lmm_build_metamesh(h2)
            T2 = B.lmm_triangulate(h2, args.ce)
            for f in range(0, T2, chunk):
                B.lmm_write_triangles(h2, f, min(chunk, T2 - f), ring)
            return T2
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            T2 = e2e_step()
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=coll_dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item())
        in_bytes = lat.xyz.nbytes + lat.ends.nbytes + lat.r_end.nbytes
        e2e = {"value": S_all / (e2e_ms / 1e3), "unit": "struts/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": int(T2) * STL,
               "triangles_per_s": T_all / (e2e_ms / 1e3)}

    if rank != 0:
        B.lmm_destroy(h)
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (emit): algorithmic bytes = 50 B per triangle
    emit_ms, emit_n = kt["emit"]
    peak, src = peaks()
    emit_bytes = float(T) * STL * args.steps
    achieved = emit_bytes / (emit_ms / 1e3) / 1e9 if emit_ms > 0 else None
    mm_ms = kt["csr"][0] + kt["bucket"][0] + kt["metamesh"][0]
    tri_ms = kt["count"][0] + kt["scan"][0] + kt["emit"][0]
    # the kernel that emitted the band region (k_emit: warp per band; k_emit_span: CTA windows)
    kinds = sorted({"k_emit_span" if per_ce_path.get(ce) == 1 else "k_emit" for ce in ces})
    emit_kernel = "+".join(kinds)
    traffic, bpt = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "emit_traffic.json")) as f:
            tj = json.load(f)
        bk = tj.get("by_kernel", {})
        bpt = (bk.get(emit_kernel, {}).get("bytes_per_triangle", tj.get("bytes_per_triangle")) if len(kinds) == 1
               else tj.get("bytes_per_triangle"))
        traffic = bpt * float(T) * args.steps / emit_n if emit_n else None   # DRAM bytes per launch
    except (OSError, ValueError, TypeError, AttributeError):
        pass
    res = {
        "metric": METRIC,
        "value": S_all / (ms_max / 1e3),
        "unit": "struts/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": desc, "chord_error": args.ce, "n_struts": int(S_all), "n_struts_local": S,
                   "n_nodes_local": N, "global_output_offset_rank0": offsets["base"],
                   "triangles_per_step": int(T), "triangles_per_step_all_ranks": int(T_all),
                   "parallelism": f"dp{world} (one spatial block per GPU)",
                   "l2": "output chunks of 13.4 GB >> 126 MB L2 (no flush needed)",
                   "error_nodes": st["n_error_nodes"], "spilled_nodes": st["n_spilled_nodes"],
                   "error_codes": {str(i): int(x) for i, x in enumerate(st["err_hist"]) if i and x}},
        "metamesh_struts_per_s": S_own * args.steps / (mm_ms / 1e3) if mm_ms else None,
        "triangles_per_s": T_all / (ms_max / 1e3),
        "triangulate_triangles_per_s": T * args.steps / (tri_ms / 1e3) if tri_ms else None,
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items()},
        "roofline": {"bound": "hbm", "kernel": emit_kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "peak_source": src,
                     "traffic": traffic, "traffic_bytes_per_triangle": bpt, "algorithmic_bytes_per_triangle": STL,
                     "launches": emit_n, "avg_launch_ms": emit_ms / emit_n if emit_n else None},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(args.ce, args.config, sweep)
    if sweep:   # configs[4]: re-triangulation of the fixed meta-mesh, triangles/s over the sweep
        res["value"] = T_all / (ms_max / 1e3)
        res["unit"] = "triangles/s"
        res["config"]["chord_error"] = sweep
        res["config"]["triangles_per_ce"] = {str(k): int(v) for k, v in per_ce.items()}
        res["config"]["metamesh"] = "built once before the timed region (multi-resolution reuse)"
        res["metamesh_struts_per_s"] = None
    if one_gpu and world > 1:
        res["config"]["note"] = (f"{world} ranks time-sharing cuda:0 over gloo (LMM_BENCH_ONE_GPU=1): a functional "
                                 "check of the multi-rank path, not a scaling number")
    if args.config.startswith("stoch"):
        dh = [int(x) for x in st["degree_hist"]]
        res["config"]["degree_hist"] = {str(d): c for d, c in enumerate(dh) if c}
    print(json.dumps(res))
    B.lmm_destroy(h)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
