"""Edge cases of the CUDA path through the C-ABI: empty and degenerate inputs, the
maximum supported node degree (31) and one past it, isolated nodes, ragged sizes,
argument and state errors (fail loudly, never silently)."""
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


def test_max_degree_31_parity():
    lat = synth.star(_fib_dirs(31), 1.0, 0.05)
    mm, _, T = _full_parity(lat)
    assert mm.stats()["n_error_nodes"] == 0 and T > 0
    mm.close()


def test_degree_32_is_flagged_like_the_oracle():
    """One past the supported degree: the node gets status 1 (degree > 31) on both sides;
    its struts contribute no band, the far nodes still get their meta-mesh."""
    lat = synth.star(_fib_dirs(32), 1.0, 0.05)
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


@pytest.mark.parametrize("k", [8, 11, 12, 16])
def test_umbrella_vertex_capacity_like_the_oracle(k):
    """k struts on a cone around an axis meet in ONE k-valent vertex (C(k, 3) junctions at a
    point): representable up to the junction capacity of the degree class (R13),
    flagged JCAP beyond it -- identically by kernel and oracle."""
    d = [[np.sin(1.0) * np.cos(t), np.sin(1.0) * np.sin(t), np.cos(1.0)] for t in np.linspace(0, 2 * np.pi, k, endpoint=False)]
    lat = synth.star(d, 1.0, 0.05)
    mm, orc, T = _full_parity(lat)
    st = mm.stats()
    assert st["n_error_nodes"] == (1 if k >= 12 else 0)
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
