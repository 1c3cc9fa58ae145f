"""Multi-GPU host logic on CPU: spatial slabs with halo recompute, emit masks, and the
all-gather of triangle counts (gloo, world size 2)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2405_15197_b200 import partition as P

NX, NY, NZ = 3, 2, 4
K_TOP = 2 * NZ


def _windows(world):
    out = []
    for r in range(world):
        k_lo, k_hi = P.window(r, world, K_TOP)
        lat = synth.octet_window(NX, NY, NZ, k_lo, k_hi, radius=0.03, r_max=0.06)
        nm, sm = P.emit_masks(lat.ijk[:, 2], lat.ends, r, world, K_TOP)
        out.append((lat, nm, sm))
    return out


@pytest.mark.parametrize("world", [2, 3, 4])
def test_slabs_partition_nodes_and_struts(world):
    full = synth.octet_window(NX, NY, NZ, 0, K_TOP)
    gstrut = {(int(full.gid[a]), int(full.gid[b])) for a, b in full.ends}
    owned_nodes, owned_struts = [], []
    for lat, nm, sm in _windows(world):
        owned_nodes += list(lat.gid[nm.astype(bool)])
        owned_struts += [(int(lat.gid[a]), int(lat.gid[b])) for a, b in lat.ends[sm.astype(bool)]]
    assert sorted(owned_nodes) == sorted(full.gid.tolist())          # each node owned once
    assert len(owned_struts) == len(set(owned_struts)) == len(gstrut)  # each strut emitted once
    assert set(owned_struts) == gstrut


@pytest.mark.parametrize("world", [2, 3])
def test_owned_struts_have_complete_end_neighbourhoods(world):
    """The band of an owned strut needs the meta-mesh of both its end nodes: both must see
    their full global degree in the local window (the halo is deep enough)."""
    full = synth.octet_window(NX, NY, NZ, 0, K_TOP)
    gdeg = dict(zip(full.gid.tolist(), full.degrees().tolist()))
    for lat, nm, sm in _windows(world):
        deg = lat.degrees()
        ends = lat.ends[sm.astype(bool)]
        for n in np.unique(ends):
            assert deg[n] == gdeg[int(lat.gid[n])]
        for n in np.nonzero(nm)[0]:
            assert deg[n] == gdeg[int(lat.gid[n])]


def test_union_of_rank_outputs_is_the_global_mesh():
    """Per-rank oracle runs on the windows, restricted to the emit masks, reproduce the global
    triangulation exactly (bitwise, as a set): the halo recompute is seamless."""
    full = synth.octet_window(NX, NY, NZ, 0, K_TOP, radius=0.03, r_max=0.06)
    og = oracle.Oracle.from_lattice(full)
    assert og.metamesh() == 0
    og.triangulate(5e-3)
    ref = og.write_triangles()
    parts = []
    for lat, nm, sm in _windows(2):
        o = oracle.Oracle.from_lattice(lat)
        o.metamesh()
        o.triangulate(5e-3)
        for s in np.nonzero(sm)[0]:
            parts.append(o.strut_triangles(int(s)))
        for n in np.nonzero(nm)[0]:
            t = o.node_hole_triangles(int(n))
            if len(t):
                parts.append(t)
    got = np.concatenate(parts)
    assert len(got) == len(ref)
    key = lambda a: np.unique(a.reshape(len(a), -1), axis=0)
    assert np.array_equal(key(got), key(ref))


def _gather_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k_lo, k_hi = P.window(rank, world, K_TOP)
    lat = synth.octet_window(NX, NY, NZ, k_lo, k_hi, radius=0.03, r_max=0.06)
    nm, sm = P.emit_masks(lat.ijk[:, 2], lat.ends, rank, world, K_TOP)
    o = oracle.Oracle.from_lattice(lat)
    o.metamesh()
    o.triangulate(1e-2)
    bn, _ = o.band_info()
    base, M, _ = o.hole_info()
    mine = int(bn[sm.astype(bool), :2].sum())
    for n in np.nonzero(nm)[0]:
        mine += int(M[base[n]:base[n + 1]].sum())
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([mine], dtype=torch.int64))
    offs = P.global_offsets([int(c) for c in counts])
    out[rank] = (mine, offs[rank], sum(int(c) for c in counts))
    dist.destroy_process_group()


def test_allgather_of_counts_gives_global_offsets_gloo():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, port, out), nprocs=world, join=True)
    full = synth.octet_window(NX, NY, NZ, 0, K_TOP, radius=0.03, r_max=0.06)
    og = oracle.Oracle.from_lattice(full)
    og.metamesh()
    total = og.triangulate(1e-2)
    assert out[0][2] == out[1][2] == total
    assert out[0][1] == 0 and out[1][1] == out[0][0]


# ---- configs[2]: ONE stochastic lattice split into z-slabs (bench.make_config("stochN", r, W)) ----
@pytest.mark.parametrize("world", [2, 3])
def test_stochastic_slabs_partition_one_lattice(world):
    """bench.make_config("stoch12", r, world) over all ranks: every node of the ONE global
    stochastic lattice (12 x 12 x 12*world) is owned exactly once, every strut emitted exactly
    once, and both ends of an owned strut -- and every owned node -- see their full global
    neighbourhood in the rank's window (so their meta-meshes equal the single-lattice ones)."""
    import bench
    n = 12
    full = synth.stochastic_window(n, n * world, 0, n * world - 1, seed=0)
    gstrut = {(int(full.gid[a]), int(full.gid[b])) for a, b in full.ends}
    gdeg = dict(zip(full.gid.tolist(), full.degrees().tolist()))
    owned_nodes, owned_struts = [], []
    for r in range(world):
        lat, (nm, sm), _ = bench.make_config(f"stoch{n}", r, world)
        owned_nodes += list(lat.gid[nm.astype(bool)])
        owned_struts += [(int(lat.gid[a]), int(lat.gid[b])) for a, b in lat.ends[sm.astype(bool)]]
        deg = lat.degrees()
        for v in np.unique(lat.ends[sm.astype(bool)]):
            assert deg[v] == gdeg[int(lat.gid[v])]
        for v in np.nonzero(nm)[0]:
            assert deg[v] == gdeg[int(lat.gid[v])]
        # the window's positions / radii / struts are those of the global lattice
        idx = np.searchsorted(full.gid, lat.gid)
        assert np.array_equal(lat.xyz, full.xyz[idx]) and np.array_equal(lat.node_r, full.node_r[idx])
    assert sorted(owned_nodes) == sorted(full.gid.tolist())
    assert len(owned_struts) == len(set(owned_struts)) == len(gstrut)
    assert set(owned_struts) == gstrut
    assert full.degrees().max() <= 30 and np.percentile(full.degrees(), 50) <= 6   # skewed 3..30


def test_stochastic_windows_agree_with_the_global_lattice():
    """Any z-window of stochastic_window equals the global lattice restricted to its layers
    (blocks of 10 layers generated independently + seam passes: the generator is local)."""
    g = synth.stochastic_window(14, 37, 0, 36, seed=3)
    nxy = 14 * 14
    ge = {tuple(e) for e in g.gid[g.ends].tolist()}
    for lo, hi in [(0, 9), (5, 23), (18, 36), (9, 10)]:
        w = synth.stochastic_window(14, 37, lo, hi, seed=3)
        we = {tuple(e) for e in w.gid[w.ends].tolist()}
        inside = {e for e in ge if lo * nxy <= e[0] < (hi + 1) * nxy and lo * nxy <= e[1] < (hi + 1) * nxy}
        assert we == inside
        assert np.array_equal(w.xyz, g.xyz[w.gid - g.gid[0]])
