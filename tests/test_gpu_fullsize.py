"""Parity at BASELINE.json's full single-GPU sizes, in the launch configuration bench.py
times (the meta-mesh of every node in one lmm_build_metamesh, the triangles emitted into a
device buffer in bench.py's 2^28-triangle chunks), CE = 1e-3 (and octet100 at CE 1e-2, whose
48-triangle bands take the CTA-window emit path):
  octet100 -- configs[1]: 100^3-cell graded octet truss, 24.12M struts (the headline bench);
  bcc250   -- configs[3]: one GPU's 250^3-cell block of the 1B-strut BCC lattice, 125M struts;
  stoch290 -- configs[2]: stochastic lattice, degrees 3..30, 102M struts;
  octet160 at CE = 1e-4 -- configs[4]'s fixed 98.6M-strut meta-mesh at its finest chord error.

The oracle cannot meta-mesh 4M nodes in seconds, so it computes SAMPLED outputs one by
one (orc_metamesh on a node subset; a band needs only its two end nodes):
  * sampled nodes (random, every degree class, lattice corners/edges/faces): topology
    bit-exact, geometry within 1e-4 r_min;
  * sampled struts: band sizes and rotation bit-exact, the band's triangles (sliced out of
    the bench-sized device chunk that holds them) within tolerance;
  * sampled hole fans of boundary nodes: triangle counts exact, triangles within tolerance;
and properties that hold at any size are checked on the whole output: offsets are the
exclusive prefix sums of the band / hole sizes, no node in error, every strut has its band,
totals consistent; and sampled neighbourhoods (a node's fans + all its bands) are welded
and checked watertight (manifold, oriented, bounded only by the far-end rings).
"""
import numpy as np
import pytest

import bench
import oracle
from _parity import assert_node_parity, assert_triangles_close

pytestmark = pytest.mark.gpu

N_NODES_SAMPLE = 4000
N_STRUTS_SAMPLE = 4000


@pytest.fixture(scope="module", params=[("octet100", 1e-3), ("bcc250", 1e-3), ("stoch290", 1e-3), ("octet160", 1e-4),
                                        ("octet100", 1e-2)],
                ids=["octet100", "bcc250", "stoch290", "octet160-ce1e-4", "octet100-ce1e-2"])
def full(request):
    import torch
    from paper_2405_15197_b200 import MetaMesher
    name, ce = request.param
    lat, _, _ = bench.make_config(name)
    lat.ce = ce
    mm = MetaMesher(0).load_lattice(lat).build()
    T = mm.triangulate(ce)
    orc = oracle.Oracle.from_lattice(lat)
    out = torch.empty(bench.EMIT_CHUNK * bench.STL, dtype=torch.uint8, device="cuda")
    yield lat, mm, T, orc, out
    mm.close()
    del out
    torch.cuda.empty_cache()


def _sample_nodes(lat, rng):
    deg = lat.degrees()
    pick = [rng.choice(lat.n_nodes, N_NODES_SAMPLE, replace=False)]
    for d in np.unique(deg):                      # every degree class (boundary nodes have 3..11)
        idx = np.flatnonzero(deg == d)
        pick.append(rng.choice(idx, min(8, len(idx)), replace=False))
    lo, hi = lat.xyz.min(0), lat.xyz.max(0)
    corner = np.all((np.abs(lat.xyz - lo) < 1e-3) | (np.abs(lat.xyz - hi) < 1e-3), axis=1)
    pick.append(np.flatnonzero(corner))
    pick.append([0, lat.n_nodes - 1])
    return np.unique(np.concatenate([np.asarray(p, np.int64) for p in pick]))


def _error_nodes(mm):
    from paper_2405_15197_b200 import binding as B
    hdr = B.lmm_buffer(mm.h, B.LMM_BUF_NODE_HDR, np.int32, 4)
    return np.flatnonzero(hdr[:, 0] & 0xFF)


def test_fullsize_whole_output_properties(full):
    lat, mm, T, orc, _ = full
    st = mm.stats()
    assert st["n_struts"] == lat.n_struts and st["n_nodes"] == lat.n_nodes
    # every node the model defines is meshed: no node in error, so every strut has its band
    bad = _error_nodes(mm)
    assert len(bad) == st["n_error_nodes"]
    if len(bad):        # diagnose before failing: the oracle must agree on each of them
        orc.metamesh(bad)
        print("error nodes:", [(int(n), orc.node(int(n))["status"]) for n in bad[:20]])
    assert len(bad) == 0, (len(bad), st["err_hist"])
    tb = mm.tri_buffers()
    band = tb["band"].astype(np.int64)
    soff = tb["strut_off"]
    assert soff[0] == 0 and np.array_equal(np.diff(soff), band[:, 0] + band[:, 1])
    assert np.all(band[:, 0] > 0) and np.all(band[:, 1] > 0)
    hoff = tb["hole_off"]                             # hole offsets follow the bands
    assert hoff[0] == 0 and np.array_equal(np.diff(hoff), tb["hole_M"].astype(np.int64))
    assert soff[-1] + hoff[-1] == T
    h0 = tb["node_hole0"]
    assert h0[0] == 0 and np.all(np.diff(h0) >= 0) and h0[-1] == len(tb["hole_M"])


N_NEIGH_SAMPLE = 400


def test_fullsize_sampled_neighbourhoods_watertight(full):
    """Watertightness at full size, in the bench launch configuration: for sampled nodes (random
    and every degree class) the patch of the node's hole fans plus the whole bands of all its
    struts, welded by exact binary32 coordinates, is a manifold, consistently oriented surface
    whose only boundary is the far-end rings of its bands (one closed ring per strut).  Every
    seam of the mesh (band-band along a shared arc, band-fan, shared vertices) lies around some
    node, so the samples cover every kind of seam."""
    lat, mm, T, orc, out = full
    rng = np.random.default_rng(77)
    deg = lat.degrees()
    pick = [rng.choice(np.flatnonzero(deg > 0), N_NEIGH_SAMPLE, replace=False)]
    for d in np.unique(deg[deg > 0]):
        idx = np.flatnonzero(deg == d)
        pick.append(rng.choice(idx, min(4, len(idx)), replace=False))
    nodes = np.unique(np.concatenate(pick))
    tb = mm.tri_buffers()
    band, soff = tb["band"].astype(np.int64), tb["strut_off"]
    hoff, h0 = tb["hole_off"], tb["node_hole0"]
    nTb = int(soff[-1])
    inc = {}
    for n in nodes:
        inc[int(n)] = np.flatnonzero((lat.ends[:, 0] == n) | (lat.ends[:, 1] == n))
    # every requested record range, fetched in output order through the bench-sized chunks
    req = []
    for n, ss in inc.items():
        for s_ in ss:
            req.append((int(soff[s_]), int(soff[s_ + 1] - soff[s_]), n))
        a, b = nTb + int(hoff[h0[n]]), nTb + int(hoff[h0[n + 1]])
        if b > a:
            req.append((a, b - a, n))
    got = {n: [] for n in inc}
    cache = {}
    for first, cnt, n in sorted(req):
        got[n].append(_chunk_records(mm, out, T, first, cnt, cache))
    for n, ss in inc.items():
        tris = np.concatenate(got[n])
        V = tris[:, 1:, :].reshape(-1, 3)
        _, inv = np.unique(V, axis=0, return_inverse=True)
        F = inv.reshape(-1, 3)
        e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])
        und, cnt = np.unique(np.sort(e, axis=1), axis=0, return_counts=True)
        _, dcnt = np.unique(e, axis=0, return_counts=True)
        assert set(cnt.tolist()) <= {1, 2}, (n, set(cnt.tolist()))
        assert not np.any(dcnt > 1), n                      # seams traversed in opposite directions
        far = np.where(lat.ends[ss, 0] == n, band[ss, 1], band[ss, 0])   # far-end ring sizes
        assert int((cnt == 1).sum()) == int(far.sum()), (n, int((cnt == 1).sum()), int(far.sum()))


def test_fullsize_sampled_nodes(full):
    from paper_2405_15197_b200 import decode_node
    lat, mm, T, orc, _ = full
    nodes = _sample_nodes(lat, np.random.default_rng(2405))
    assert orc.metamesh(nodes) == 0
    tol = 1e-4 * float(lat.node_r.min())
    for n in nodes:
        assert_node_parity(decode_node(mm.node_buffers(int(n)), 0), orc.node(int(n)), tol, int(n))


def _chunk_records(mm, out, T, first, count, cache):
    """Records [first, first+count) taken from the bench-sized device chunk(s) holding them."""
    from paper_2405_15197_b200 import stl_records_to_array
    import bench as b
    res = []
    while count > 0:
        c = first // b.EMIT_CHUNK
        if cache.get("chunk") != c:
            f0 = c * b.EMIT_CHUNK
            mm.write(f0, min(b.EMIT_CHUNK, T - f0), out)
            cache["chunk"] = c
        lo = first - c * b.EMIT_CHUNK
        k = min(count, b.EMIT_CHUNK - lo)
        res.append(stl_records_to_array(out[lo * b.STL:(lo + k) * b.STL].cpu().numpy()))
        first += k
        count -= k
    return np.concatenate(res) if res else np.zeros((0, 4, 3), np.float32)


def test_fullsize_sampled_bands_and_holes(full):
    lat, mm, T, orc, out = full
    rng = np.random.default_rng(1505)
    struts = np.unique(np.concatenate([rng.choice(lat.n_struts, N_STRUTS_SAMPLE, replace=False),
                                       [0, lat.n_struts - 1]]))
    deg = lat.degrees()
    bnd = np.flatnonzero(deg < deg.max())             # lattice-boundary nodes carry hole fans
    hnodes = np.unique(rng.choice(bnd, 1000, replace=False))
    need = np.unique(np.concatenate([lat.ends[struts].ravel(), hnodes]))
    assert orc.metamesh(need) == 0
    orc.triangulate(lat.ce)                           # bands of struts with both ends done
    bn, _ = orc.band_info()
    orc._bn = bn                                      # strut_triangles() reuses it
    base, M, _ = orc.hole_info()
    tb = mm.tri_buffers()
    band, soff = tb["band"].astype(np.int64), tb["strut_off"]
    hoff, h0 = tb["hole_off"], tb["node_hole0"]
    r = float(lat.node_r.min())
    # walk the samples in output order so each bench-sized chunk is emitted once
    items = [(int(soff[s]), "band", int(s)) for s in struts] + [(int(soff[-1] + hoff[h0[n]]), "hole", int(n)) for n in hnodes]
    cache = {}
    for first, kind, i in sorted(items):
        if kind == "band":
            assert np.array_equal(band[i, :3], bn[i]), i
            n = int(band[i, 0] + band[i, 1])
            got = _chunk_records(mm, out, T, first, n, cache)
            assert_triangles_close(got, orc.strut_triangles(i), r, ("strut", i))
        else:
            gm = tb["hole_M"][h0[i]:h0[i + 1]].astype(np.int64)
            om = M[base[i]:base[i + 1]]
            assert np.array_equal(gm, om), i
            got = _chunk_records(mm, out, T, first, int(gm.sum()), cache)
            assert_triangles_close(got, orc.node_hole_triangles(i), r, ("holes", i))
