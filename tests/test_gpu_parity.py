"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.

Topology -- vertex/arc/hole counts, tie masks, arc endpoints, loop order, hole contours,
per-arc parameter ranges and stitch angles (binary32 decision values), subdivision
counts, band sizes and rotations, triangle offsets -- must be bit-exact.  Geometry: the
kernel's binary32 against the oracle's binary64 within 1e-4 x the minimum strut radius
(north star), plus the binary32 rounding of absolute coordinates for triangles.
"""
import numpy as np
import pytest

import oracle
import synth
from _parity import GEOM_TOL, GEOM_TOL_SHARP, assert_node_parity, assert_triangles_close

pytestmark = pytest.mark.gpu



def _lat(name):
    return {
        "single": lambda: synth.single_strut(1.0, 0.1, 0.1),
        "cone": lambda: synth.single_strut(1.0, 0.1, 0.06),
        "chain-bent": lambda: synth.chain(5, 1.0, 0.1, 50.0),
        "star-bcc": lambda: synth.star([[1, 1, 1], [1, 1, -1], [1, -1, 1], [1, -1, -1], [-1, 1, 1], [-1, 1, -1],
                                        [-1, -1, 1], [-1, -1, -1]], 1.0, 0.1),
        "cubic3": lambda: synth.cubic(3, 3, 3),
        "bcc3": lambda: synth.bcc(3, 3, 3),
        "octet2": lambda: synth.octet(2, 2, 2),
        "octet2-graded": lambda: synth.graded_radii(synth.octet(2, 2, 2), 0.03, 0.06),
        "bcc3-jitter": lambda: synth.jitter(synth.bcc(3, 3, 3), 0.05, 1),
        "cubic4-graded-jitter": lambda: synth.jitter(synth.graded_radii(synth.cubic(4, 4, 4), 0.06, 0.12, 2), 0.04, 2),
        "voronoi": lambda: synth.voronoi_like(300, seed=3, radius=0.05),
        # configs[2] shape: skewed degrees 3..30, cones; configs[3] shape: a BCC spatial block
        "stochastic9": lambda: synth.stochastic(9, seed=7),
        # the sharp-angle family: struts down to 10 degrees apart at a node (long strut-strut
        # intersections, near-parabolic sections, short-strut limits)
        "sharp10": lambda: synth.stochastic_window(9, 9, 0, 8, seed=21, min_angle_deg=10.0),
        "bccwin": lambda: synth.bcc_window(4, 3, 5, 3, 8),
        # a strut ringed by 16 neighbours: its loop has 16 entries (> the emit pass's arc cache,
        # so its band takes the windowed path)
        "crown16": lambda: synth.star([[0, 0, 1]] + [[np.sin(0.7) * np.cos(t), np.sin(0.7) * np.sin(t), np.cos(0.7)]
                                                     for t in np.linspace(0, 2 * np.pi, 16, endpoint=False)], 1.0, 0.05),
        # BASELINE.json configs[0]: 10x10x10 BCC, uniform radius, eps = 1e-3 r
        "bcc10": lambda: synth.bcc(10, 10, 10),
    }[name]()


NAMES = ["single", "cone", "chain-bent", "star-bcc", "cubic3", "bcc3", "octet2", "octet2-graded", "bcc3-jitter",
         "cubic4-graded-jitter", "voronoi", "stochastic9", "sharp10", "bccwin", "crown16", "bcc10"]


@pytest.fixture(scope="module")
def built():
    from paper_2405_15197_b200 import build as b
    b.build()
    cache = {}

    def get(name):
        if name not in cache:
            from paper_2405_15197_b200 import MetaMesher
            lat = _lat(name)
            mm = MetaMesher(0).load_lattice(lat).build()
            orc = oracle.Oracle.from_lattice(lat)
            orc.metamesh()
            cache[name] = (lat, mm, orc, mm.buffers())
        return cache[name]
    return get


GEOM_TOL_BY_NAME = {"sharp10": GEOM_TOL_SHARP}   # the 10-degree family (tests/_parity.py)


@pytest.mark.parametrize("name", NAMES)
def test_metamesh_topology_bit_exact_and_geometry(built, name):
    from paper_2405_15197_b200 import decode_node
    lat, mm, orc, bufs = built(name)
    tol = GEOM_TOL_BY_NAME.get(name, GEOM_TOL) * float(lat.node_r.min())
    for n in range(lat.n_nodes):
        assert_node_parity(decode_node(bufs, n), orc.node(n), tol, n)


def _mesh_edges_ok(tris):
    V = tris[:, 1:, :].reshape(-1, 3)
    uniq, inv = np.unique(V, axis=0, return_inverse=True)
    F = inv.reshape(-1, 3)
    e = np.sort(np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]]), axis=1)
    eu, cnt = np.unique(e, axis=0, return_counts=True)
    return set(cnt.tolist()), len(uniq) - len(eu) + len(F)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("ce", [1e-2, 1e-3])
def test_triangulation_parity(built, name, ce):
    _triangulation_parity(built, name, ce)


@pytest.mark.parametrize("name", ["octet2-graded", "stochastic9", "crown16", "chain-bent"])
@pytest.mark.parametrize("ce", [3e-4, 1e-4, 1e-5])
def test_triangulation_parity_fine(built, name, ce):
    """Fine chord errors: long bands, the emit pass's larger point caches (up to the largest,
    mean band > 627 triangles at CE 1e-5) and windows."""
    _triangulation_parity(built, name, ce)


def _triangulation_parity(built, name, ce):
    lat, mm, orc, _ = built(name)
    assert mm.stats()["n_error_nodes"] == 0
    T = mm.triangulate(ce)
    To = orc.triangulate(ce)
    assert T == To
    tb = mm.tri_buffers()
    bn, soff = orc.band_info()
    assert np.array_equal(tb["band"][:, :3].astype(np.int64), bn)
    assert np.array_equal(tb["strut_off"], soff)
    base, M, bp = orc.hole_info()
    assert np.array_equal(tb["hole_M"].astype(np.int64), M)
    assert np.array_equal(tb["node_hole0"], base)
    tri = mm.triangles(0, T).astype(np.float64)
    ref = orc.write_triangles()
    r = float(lat.node_r.min())
    assert_triangles_close(tri, ref, r, (name, ce), GEOM_TOL_BY_NAME.get(name, GEOM_TOL))
    # facet normals agree wherever the facet is not tiny
    # facet normals: error bounded by vertex error / shortest altitude
    v1, v2, v3 = ref[:, 1], ref[:, 2], ref[:, 3]
    area2 = np.linalg.norm(np.cross(v2 - v1, v3 - v1), axis=1)
    longest = np.max(np.stack([np.linalg.norm(v2 - v1, axis=1), np.linalg.norm(v3 - v2, axis=1),
                               np.linalg.norm(v1 - v3, axis=1)]), axis=0)
    alt = area2 / np.maximum(longest, 1e-300)
    verr = np.max(np.abs(tri[:, 1:] - ref[:, 1:]), axis=(1, 2))
    ok = alt > 0
    nerr = np.max(np.abs(tri[ok, 0] - ref[ok, 0]), axis=1)
    # the kernel's normal comes from the binary32 vertices it writes, each off the binary64
    # point by its own error plus the 2^-24 |x| rounding of the absolute coordinate
    rep = 2.0 ** -24 * np.max(np.abs(ref[:, 1:]), axis=(1, 2))
    assert np.all(nerr <= 4 * (verr[ok] + rep[ok]) / alt[ok] + 1e-5)
    # the kernel's own output is watertight: welded by exact binary32 coordinates
    counts, chi = _mesh_edges_ok(mm.triangles(0, T))
    assert counts == {2}
    assert chi == 2 - 2 * lat.genus()


@pytest.mark.parametrize("ce", [1e-2, 1e-3])
def test_ranges_and_device_output(built, ce):
    """Arbitrary [first, first+count) windows equal the full emission; device destination."""
    import torch
    lat, mm, orc, _ = built("bcc3-jitter")
    T = mm.triangulate(ce)
    full = mm.triangles(0, T)
    rng = np.random.default_rng(0)
    for _ in range(20):
        a = int(rng.integers(0, T))
        b = int(rng.integers(a, min(T, a + 5000) + 1))
        assert np.array_equal(mm.triangles(a, b - a).view(np.uint32), full[a:b].view(np.uint32))
    dev = torch.zeros(T * 50 + 16, dtype=torch.uint8, device="cuda")
    mm.write(0, T, dev)
    torch.cuda.synchronize()
    from paper_2405_15197_b200 import stl_records_to_array
    got = stl_records_to_array(dev[: T * 50].cpu().numpy())
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


def test_remesh_reuses_metamesh(built):
    """Algorithm 1: a chord-error list re-triangulates one meta-mesh; counts are monotone."""
    lat, mm, orc, _ = built("octet2-graded")
    counts = [mm.triangulate(ce) for ce in (1e-4, 1e-3, 1e-2, 5e-2)]
    assert all(a >= b for a, b in zip(counts, counts[1:]))
    assert counts[-1] == orc.triangulate(5e-2)


def test_ce_sweep_on_one_metamesh_matches_oracle_each_time(built):
    """BASELINE configs[4] in miniature: ONE meta-mesh re-triangulated at 1e-2, 1e-3, 1e-4 and
    again at 1e-2 (state from the finer pass must not leak): every pass equals the oracle."""
    lat, mm, orc, _ = built("octet2-graded")
    r = float(lat.node_r.min())
    for ce in (1e-2, 1e-3, 1e-4, 1e-2):
        T = mm.triangulate(ce)
        assert T == orc.triangulate(ce)
        assert_triangles_close(mm.triangles(0, T), orc.write_triangles(), r, ce)


def test_csr_offsets_are_the_degree_prefix_sum(built):
    """PAPER.md Sec. 4.3.2 index region = exclusive prefix sum (device scan), here of the
    node degrees; incident struts ascending per node."""
    from paper_2405_15197_b200 import lmm_buffer
    from paper_2405_15197_b200 import binding as B
    lat, mm, orc, _ = built("voronoi")
    off = lmm_buffer(mm.h, B.LMM_BUF_CSR_OFF, np.int32)
    ent = lmm_buffer(mm.h, B.LMM_BUF_CSR_ENT, np.int32, 2)
    assert np.array_equal(off.astype(np.int64), np.concatenate([[0], np.cumsum(lat.degrees())]))
    o_off, o_st = orc.csr()
    assert np.array_equal(off.astype(np.int64), o_off)
    assert np.array_equal(ent[:, 0].astype(np.int64), o_st)


@pytest.mark.parametrize("family", ["octet", "bcc", "stoch"])
@pytest.mark.parametrize("path", ["0", "1"], ids=["band-path", "cta-windows"])
def test_virtual_ranks_union_equals_global_gpu(family, path, monkeypatch):
    """The multi-GPU path on one device: slab windows with halo recompute + emit masks.  The
    union of the per-rank STL outputs equals the single-lattice output bitwise (as a set),
    so the global mesh is seamless across rank boundaries -- through either emit path (the
    masked struts are empty bands inside the CTA windows)."""
    monkeypatch.setenv("LMM_EMIT_PATH", path)
    from paper_2405_15197_b200 import MetaMesher
    from paper_2405_15197_b200 import partition as P
    nx, ny, nz = 4, 3, 6
    k_top, halo = 2 * nz, 2
    gen = (lambda lo, hi: synth.octet_window(nx, ny, nz, lo, hi, radius=0.03, r_max=0.06)) if family == "octet" \
        else (lambda lo, hi: synth.bcc_window(nx, ny, nz, lo, hi, radius=0.05))
    if family == "stoch":   # configs[2]: one stochastic lattice, 10 x 10 x 30 nodes, 4-layer halos
        k_top, halo = 29, 4
        gen = lambda lo, hi: synth.stochastic_window(10, 30, lo, hi, seed=0)
    full = gen(0, k_top)
    mm = MetaMesher(0).load_lattice(full).build()
    T = mm.triangulate(5e-3)
    ref = mm.triangles(0, T)
    parts, counts = [], []
    for r in range(3):
        k_lo, k_hi = P.window(r, 3, k_top, halo)
        lat = gen(k_lo, k_hi)
        nm, sm = P.emit_masks(lat.ijk[:, 2], lat.ends, r, 3, k_top)
        m = MetaMesher(0).load_lattice(lat).build().set_emit_mask(nm, sm)
        Tr = m.triangulate(5e-3)
        counts.append(Tr)
        parts.append(m.triangles(0, Tr))
        m.close()
    assert sum(counts) == T
    got = np.concatenate(parts)
    key = lambda a: np.unique(a.reshape(len(a), -1).view(np.uint32), axis=0)
    assert np.array_equal(key(got), key(ref))
    mm.close()


def _random_lattice(seed):
    """Seeded mixes of the generators: jittered, graded, stochastic, with radii spanning 2x."""
    rng = np.random.default_rng(seed)
    kind = seed % 4
    if kind == 0:
        lat = synth.stochastic(int(rng.integers(5, 9)), seed=seed, r_min=0.015, r_max=0.05)
    elif kind == 1:
        lat = synth.jitter(synth.graded_radii(synth.octet(3, 2, 2), 0.02, 0.05, axis=int(rng.integers(0, 3))), 0.04, seed)
    elif kind == 2:
        lat = synth.jitter(synth.graded_radii(synth.bcc(3, 3, 2), 0.03, 0.07, axis=2), 0.06, seed)
    else:
        lat = synth.jitter(synth.graded_radii(synth.cubic(4, 3, 3), 0.05, 0.11, axis=1), 0.05, seed)
    return lat


@pytest.mark.parametrize("seed", list(range(48)))
def test_random_lattices_parity(seed):
    """Stress: 48 seeded random lattices (all generator families, jitter, graded radii);
    per node topology bit-exact and geometry within 1e-4 r_min, then the whole STL."""
    from paper_2405_15197_b200 import MetaMesher, decode_node
    lat = _random_lattice(seed)
    mm = MetaMesher(0).load_lattice(lat).build()
    orc = oracle.Oracle.from_lattice(lat)
    orc.metamesh()
    bufs = mm.buffers()
    tol = GEOM_TOL * float(lat.node_r.min())
    for n in range(lat.n_nodes):
        assert_node_parity(decode_node(bufs, n), orc.node(n), tol, n)
    ce = (2e-3, 5e-3, 1e-3, 3e-3)[seed % 4]
    T = mm.triangulate(ce)
    assert T == orc.triangulate(ce)
    assert_triangles_close(mm.triangles(0, T), orc.write_triangles(), float(lat.node_r.min()), seed)
    mm.close()


@pytest.mark.parametrize("seed", list(range(8)))
def test_medium_random_lattices_parity(seed):
    """Stress at medium size (10-40k struts): every node of a stochastic / jittered graded /
    sharp-angle (10 deg) lattice bit-exact in topology, and the whole STL within tolerance."""
    from paper_2405_15197_b200 import MetaMesher, decode_node
    lat = [lambda: synth.stochastic(16 + seed, seed=1000 + seed, r_min=0.015, r_max=0.05),
           lambda: synth.jitter(synth.graded_radii(synth.octet(7, 6, 6), 0.02, 0.06, seed % 3), 0.05, 1000 + seed),
           lambda: synth.jitter(synth.graded_radii(synth.bcc(12, 10, 9), 0.03, 0.07, seed % 3), 0.08, 1000 + seed),
           # sharp-angle family: >= 10 degrees between struts at a node
           lambda: synth.stochastic_window(16 + seed, 16 + seed, 0, 15 + seed, seed=2000 + seed, min_angle_deg=10.0)][seed % 4]()
    mm = MetaMesher(0).load_lattice(lat).build()
    orc = oracle.Oracle.from_lattice(lat)
    assert orc.metamesh() == mm.stats()["n_error_nodes"]
    bufs = mm.buffers()
    gt = GEOM_TOL_SHARP if seed % 4 == 3 else GEOM_TOL
    tol = gt * float(lat.node_r.min())
    for n in range(lat.n_nodes):
        assert_node_parity(decode_node(bufs, n), orc.node(n), tol, n)
    T = mm.triangulate(2e-3)
    assert T == orc.triangulate(2e-3)
    assert_triangles_close(mm.triangles(0, T), orc.write_triangles(), float(lat.node_r.min()), seed, gt)
    mm.close()
