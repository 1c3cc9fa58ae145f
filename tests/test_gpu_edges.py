"""Edge cases of the CUDA path through the C-ABI: empty and degenerate inputs, node degrees
across the bucket limit (31) up to the model's limit (63) and one past it, nodes whose
junctions / vertices / arcs exceed their degree bucket's workspace (the spill kernel),
isolated nodes, ragged sizes, argument and state errors (fail loudly, never silently)."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_node_parity, assert_triangles_close

pytestmark = pytest.mark.gpu


def _fib_dirs(k):
    """k well-spread unit directions (Fibonacci sphere)."""
    i = np.arange(k) + 0.5
    phi = np.arccos(1 - 2 * i / k)
    th = np.pi * (1 + 5 ** 0.5) * i
    return np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], 1)


def _mm(lat):
    from paper_2405_15197_b200 import MetaMesher
    return MetaMesher(0).load_lattice(lat).build()


def _full_parity(lat, ce=5e-3):
    from paper_2405_15197_b200 import decode_node
    mm = _mm(lat)
    orc = oracle.Oracle.from_lattice(lat)
    orc.metamesh()
    bufs = mm.buffers()
    tol = 1e-4 * float(lat.node_r.min()) if lat.n_nodes else 0.0
    for n in range(lat.n_nodes):
        assert_node_parity(decode_node(bufs, n), orc.node(n), tol, n)
    T = mm.triangulate(ce)
    assert T == orc.triangulate(ce)
    if T:
        assert_triangles_close(mm.triangles(0, T), orc.write_triangles(), float(lat.node_r.min()), lat.name)
    return mm, orc, T


def test_no_struts_gives_no_triangles():
    lat = synth.Lattice(np.zeros((5, 3), np.float32), np.zeros((0, 2), np.int64), np.full(5, 0.1, np.float32))
    mm, orc, T = _full_parity(lat)
    assert T == 0
    assert mm.stats()["n_error_nodes"] == 0
    mm.write(0, 0, np.zeros(16, np.uint8))          # an empty range is a valid call
    mm.close()


def test_empty_lattice():
    lat = synth.Lattice(np.zeros((0, 3), np.float32), np.zeros((0, 2), np.int64), np.zeros(0, np.float32))
    mm = _mm(lat)
    assert mm.triangulate(1e-3) == 0
    st = mm.stats()
    assert st["n_nodes"] == 0 and st["n_struts"] == 0
    mm.close()


def test_isolated_nodes_next_to_struts():
    base = synth.bcc(2, 1, 1)
    xyz = np.concatenate([base.xyz, [[10, 10, 10], [-5, 0, 0]]]).astype(np.float32)
    r = np.concatenate([base.node_r, [0.05, 0.05]]).astype(np.float32)
    lat = synth.Lattice(xyz, base.ends.copy(), r, "bcc+isolated")
    mm, _, T = _full_parity(lat)
    assert T > 0
    mm.close()


@pytest.mark.parametrize("k", [31, 32, 40, 63])
def test_high_degree_star_parity(k):
    """Degree 31 is the last degree bucket; 32..63 go to the spill kernel (Sec. 4.3.3:
    "multiple warps to meta-mesh a single strut"): bit-exact with the oracle, no error node."""
    lat = synth.star(_fib_dirs(k), 1.0, 0.05)
    mm, _, T = _full_parity(lat)
    assert mm.stats()["n_error_nodes"] == 0 and T > 0
    mm.close()


def test_degree_64_is_flagged_like_the_oracle():
    """One past the model's limit (sides 0..63 in one 64-bit tie mask): status 1 on both sides;
    its struts contribute no band, the far nodes still get their meta-mesh."""
    lat = synth.star(_fib_dirs(64), 1.0, 0.05)
    mm, orc, T = _full_parity(lat)
    st = mm.stats()
    assert st["n_error_nodes"] == 1 and st["err_hist"][1] == 1
    assert st["degree_hist"][32] == 1
    mm.close()


@pytest.mark.parametrize("dims", [(1, 1, 1), (7, 5, 3), (11, 2, 1)])
def test_ragged_lattice_sizes(dims):
    """Node/strut counts that are not multiples of a warp, a block or a bucket chunk."""
    lat = synth.jitter(synth.graded_radii(synth.bcc(*dims), 0.04, 0.07, axis=1), 0.03, sum(dims))
    mm, _, T = _full_parity(lat, 2e-3)
    mm.close()


def test_errors_are_loud():
    from paper_2405_15197_b200 import LmmError, MetaMesher
    lat = synth.bcc(2, 2, 2)
    mm = MetaMesher(0)
    with pytest.raises(LmmError):                       # build before load
        mm.build()
    from paper_2405_15197_b200 import binding as B
    r1 = np.full((1, 2), lat.node_r[0], np.float32)
    for ends in ([[0, 0]], [[0, lat.n_nodes]], [[-1, 2]]):   # self-loop, out-of-range end nodes
        with pytest.raises(LmmError):
            B.lmm_load_lattice(mm.h, lat.xyz, np.array(ends, np.int64), r1)
    r_end = lat.r_end.copy()
    hub = int(np.argmax(lat.degrees()))                 # a node several struts meet at
    s, e = np.argwhere(lat.ends == hub)[0]
    r_end[s, e] *= 1.5                                  # one end radius disagrees with the nodal sphere
    with pytest.raises(LmmError):
        B.lmm_load_lattice(mm.h, lat.xyz, lat.ends, r_end)
    mm.load_lattice(lat).build()
    for ce in (0.0, -1e-3, 1.5, float("nan")):
        with pytest.raises(LmmError):
            mm.triangulate(ce)
    with pytest.raises(LmmError):                       # write before triangulate
        mm.write(0, 1, np.zeros(64, np.uint8))
    T = mm.triangulate(1e-2)
    with pytest.raises(LmmError):
        mm.write(T - 1, 2, np.zeros(200, np.uint8))
    import torch
    dev = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    with pytest.raises(LmmError):                       # device output must be 16-byte aligned
        mm.write(0, 2, dev[1:])
    mm.close()


@pytest.mark.parametrize("k", [8, 11, 12, 16, 24])
def test_umbrella_vertex_any_valence(k):
    """k struts on a cone around an axis meet in ONE k-valent vertex (C(k, 3) junctions at a
    point).  Beyond the junction workspace of the node's degree bucket the node goes to the
    spill kernel: 0 error nodes, bit-exact with the oracle, for every k."""
    d = [[np.sin(1.0) * np.cos(t), np.sin(1.0) * np.sin(t), np.cos(1.0)] for t in np.linspace(0, 2 * np.pi, k, endpoint=False)]
    lat = synth.star(d, 1.0, 0.05)
    mm, orc, T = _full_parity(lat)
    assert mm.stats()["n_error_nodes"] == 0
    assert orc.node(0)["nv"] == k + 1          # the apex plus k sphere junctions around the hole
    mm.close()


def _cone_star(dirs, R, r_far, name):
    """A hub of sphere radius R whose struts narrow to r_far at unit length (strongly conical)."""
    dirs = np.asarray(dirs, float)
    dirs /= np.linalg.norm(dirs, axis=1)[:, None]
    xyz = np.concatenate([[[0.0, 0.0, 0.0]], dirs]).astype(np.float32)
    r = np.concatenate([[R], [r_far] * len(dirs)]).astype(np.float32)
    ends = np.array([[0, i + 1] for i in range(len(dirs))], np.int64)
    return synth.Lattice(xyz, ends, r, name)


@pytest.mark.parametrize("shape,R,holes", [("tet", 0.5, 4), ("tet", 0.6, 4), ("oct", 0.65, 8), ("oct", 0.68, 8)])
def test_many_hole_short_cone_nodes(shape, R, holes):
    """Short, strongly tapered struts whose end circles cut the nodal sphere into several
    exposed regions (4 holes at a tetrahedral hub, 8 at an octahedral one): more vertices
    than the bucket's vertex slab holds (2d + 2), so the node is meta-meshed by the spill
    kernel into an overflow slab slot.  Bit-exact with the oracle, watertight output."""
    dirs = {"tet": [[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]],
            "oct": [[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]]}[shape]
    lat = _cone_star(dirs, R, 0.05, f"{shape}-cone{R}")
    mm, orc, T = _full_parity(lat)
    assert mm.stats()["n_error_nodes"] == 0
    assert orc.node(0)["nh"] == holes
    from test_gpu_parity import _mesh_edges_ok
    counts, chi = _mesh_edges_ok(mm.triangles(0, T))
    assert counts == {2} and chi == 2
    mm.close()


def test_spill_mixed_with_buckets():
    """Spilled hubs next to ordinary bucketed nodes in one lattice: the bands of struts between
    a spilled node and a regular node join the overflow slab slot with the regular one."""
    hubs = []
    xyz, ends, r = [], [], []
    for h, (k, base) in enumerate([(40, (0, 0, 0)), (12, (5, 0, 0)), (33, (10, 0, 0))]):
        c = len(xyz)
        xyz.append(base)
        r.append(0.05)
        for u in _fib_dirs(k):
            ends.append((c, len(xyz)))
            xyz.append(tuple(np.asarray(base) + u))
            r.append(0.05)
    # join hub 0's and hub 1's neighbourhoods with a strut between two leaves
    ends.append((1, 42))
    lat = synth.Lattice(np.array(xyz, np.float32), np.array(ends, np.int64), np.array(r, np.float32), "hubs")
    mm, orc, T = _full_parity(lat)
    assert mm.stats()["n_error_nodes"] == 0
    mm.close()


def test_redecided_stars_parity():
    """tests/golden/stoch290_redecided_stars.json: the configs[2] nodes whose topology closes
    only at a coarser vertex resolution (reading R10): the kernel re-decides them
    exactly like the oracle (spill kernel, levels 1..4), 0 error nodes, watertight output."""
    import json
    import os
    from test_gpu_parity import _mesh_edges_ok
    J = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "stoch290_redecided_stars.json")))
    for st in J["stars"]:
        lat = synth.Lattice(np.array(st["xyz"], np.float32), np.array(st["ends"], np.int64),
                            np.array(st["r"], np.float32), f"star{st['node']}")
        for ce in (1e-2, 1e-3):
            mm, orc, T = _full_parity(lat, ce)
            assert mm.stats()["n_error_nodes"] == 0, st["node"]
            counts, chi = _mesh_edges_ok(mm.triangles(0, T))
            assert counts == {2} and chi == 2, (st["node"], ce)
            mm.close()


def test_index_region_worked_example():
    """PAPER.md Sec. 4.3.2: an index region [0, 5, 15, 32, 47, ...] is the exclusive prefix sum of
    per-item counts 5, 10, 17, 15.  Four hub nodes of degree 5, 10, 17 and 15 (ids 0-3, leaves
    after them) must give exactly those CSR offsets from the device scan."""
    from paper_2405_15197_b200 import MetaMesher, lmm_buffer
    from paper_2405_15197_b200 import binding as B
    degs = [5, 10, 17, 15]
    xyz, ends = [], []
    hubs = [np.array([4.0 * i, 0.0, 0.0]) for i in range(4)]
    xyz.extend(hubs)
    for h, dg in enumerate(degs):
        for u in _fib_dirs(dg):
            ends.append((h, len(xyz)))
            xyz.append(hubs[h] + u)
    lat = synth.Lattice(np.array(xyz, np.float32), np.array(ends, np.int64), np.full(len(xyz), 0.05, np.float32))
    mm = MetaMesher(0).load_lattice(lat)
    off = lmm_buffer(mm.h, B.LMM_BUF_CSR_OFF, np.int32)
    assert off[:5].tolist() == [0, 5, 15, 32, 47]
    mm.close()
