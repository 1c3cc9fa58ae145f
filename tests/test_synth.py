"""The seeded input generators (synth/): shapes of the paper's workloads, determinism and
the structural guarantees the benchmark configs rely on.  No meta-meshing here."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("gen", ["stochastic", "stochastic_window"])
def test_stochastic_degrees_angles_and_determinism(gen):
    """configs[2]'s generators: skewed degrees 3..30, >= 25 deg between struts at a node,
    deterministic per seed (stochastic_window: the windowable one bench.py uses)."""
    make = (lambda sd: synth.stochastic(12, seed=sd)) if gen == "stochastic" else \
        (lambda sd: synth.stochastic_window(12, 24, 0, 23, seed=sd))
    a = make(3)
    b = make(3)
    assert np.array_equal(a.ends, b.ends) and np.array_equal(a.xyz, b.xyz) and np.array_equal(a.node_r, b.node_r)
    assert not np.array_equal(a.ends, make(4).ends)
    deg = a.degrees()
    assert deg.max() <= 30 and deg.max() >= 20          # high-degree hubs exist
    assert np.median(deg) <= 6                          # ... but most nodes are low-degree (skew)
    assert np.all(a.ends[:, 0] < a.ends[:, 1])
    key = a.ends[:, 0] * a.n_nodes + a.ends[:, 1]
    assert np.all(np.diff(key) > 0)                     # sorted, no duplicate struts
    # every two struts at a node are >= 25 degrees apart
    xyz = a.xyz.astype(np.float64)
    dirs = [[] for _ in range(a.n_nodes)]
    for i, j in a.ends:
        u = xyz[j] - xyz[i]
        u /= np.linalg.norm(u)
        dirs[i].append(u)
        dirs[j].append(-u)
    cmax = max((np.max(np.triu(np.array(d) @ np.array(d).T, 1)) for d in dirs if len(d) > 1))
    assert cmax <= np.cos(np.deg2rad(25.0)) + 1e-5
    r = a.r_end
    assert r.min() >= 0.02 and r.max() <= 0.04 and np.any(r[:, 0] != r[:, 1])   # cones


def _coord_struts(lat):
    p = np.round(lat.xyz.astype(np.float64) * 2).astype(np.int64)
    e = np.sort(np.stack([p[lat.ends[:, 0]] @ [1 << 40, 1 << 20, 1], p[lat.ends[:, 1]] @ [1 << 40, 1 << 20, 1]], 1), 1)
    return set(map(tuple, e.tolist()))


def test_bcc_window_full_equals_bcc():
    full = synth.bcc(3, 4, 2)
    win = synth.bcc_window(3, 4, 2, 0, 4)
    assert win.n_struts == full.n_struts == 8 * 3 * 4 * 2 and win.n_nodes == full.n_nodes
    assert _coord_struts(win) == _coord_struts(full)
    assert np.all(np.diff(win.gid) > 0)
    assert win.genus() == full.genus()


@pytest.mark.parametrize("world", [2, 3])
def test_bcc_windows_cover_the_lattice(world):
    from paper_2405_15197_b200 import partition as P
    nx, ny, nz = 2, 3, 4
    k_top = 2 * nz
    full = _coord_struts(synth.bcc_window(nx, ny, nz, 0, k_top))
    owned = set()
    for r in range(world):
        lo, hi = P.window(r, world, k_top)
        lat = synth.bcc_window(nx, ny, nz, lo, hi)
        _, sm = P.emit_masks(lat.ijk[:, 2], lat.ends, r, world, k_top)
        sub = synth.Lattice(lat.xyz, lat.ends[sm.astype(bool)], lat.node_r)
        mine = _coord_struts(sub)
        assert not (owned & mine)
        owned |= mine
    assert owned == full
