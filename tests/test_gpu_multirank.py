"""bench.py's multi-rank path on one GPU: `torchrun --nproc-per-node 2` with
LMM_BENCH_ONE_GPU=1 (both ranks on cuda:0, gloo for the all-gathers).  Each rank meta-meshes
its z-slab plus halo and emits only what it owns (paper_2405_15197_b200.partition); the
union must be the global lattice exactly once: strut total and triangle total equal a
single-process run over the whole global lattice, with no node in error.  This exercises
the code the 8-GPU configs[3] run takes (window/halo, emit masks, count all-gather, global
offsets, max-over-ranks timing); only the collective backend differs (gloo here, NCCL there).
"""
import json
import os
import subprocess
import sys

import pytest

import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _global_lattice(name):
    """The global lattice bench.make_config partitions for world = 2 (two blocks along z)."""
    if name.startswith("octet"):
        n = int(name[5:])
        return synth.octet_window(n, n, 2 * n, 0, 4 * n, radius=0.03, r_max=0.06)
    if name.startswith("bcc"):
        n = int(name[3:])
        return synth.bcc_window(n, n, 2 * n, 0, 4 * n, radius=0.05)
    n = int(name[5:])
    return synth.stochastic_window(n, 2 * n, 0, 2 * n - 1, seed=0)


@pytest.mark.parametrize("name", ["octet12", "bcc12", "stoch24"])
def test_two_ranks_cover_the_global_lattice_once(name):
    from paper_2405_15197_b200 import MetaMesher
    lat = _global_lattice(name)
    mm = MetaMesher(0).load_lattice(lat).build()
    T_ref = mm.triangulate(1e-3)
    assert mm.stats()["n_error_nodes"] == 0
    mm.close()

    env = dict(os.environ, LMM_BENCH_ONE_GPU="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", name, "--steps", "1", "--warmup", "3",
           "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert d["config"]["n_struts"] == lat.n_struts
    assert d["config"]["triangles_per_step_all_ranks"] == T_ref
    assert d["config"]["error_nodes"] == 0
    assert d["gpu_launches"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] == d["config"]["triangles_per_step"] * 50
