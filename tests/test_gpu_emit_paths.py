"""The two emit paths of the band region -- the band path (k_emit: warp per band) and the
CTA-window path (k_emit_span: windows of whole bands, groups across band boundaries) -- write
the same STL records, bit for bit, for any triangle range.  Both evaluate Eq. 12 through the
one arc_pt formula and write the shared meta-mesh vertices at entry starts,
so any difference is a placement or indexing error in one of them.  The CTA path is stressed
with small windows (many bands too large for a window: its band-path fallback; long rings),
tiny spans (bands clipped at span starts and ends) and unaligned ranges; the band path is
the one the oracle parity tests of test_gpu_parity.py cover at the default setting, and the
CTA path is also checked against the oracle directly here."""
import os

import numpy as np
import pytest

import oracle
import synth
from _parity import assert_triangles_close

pytestmark = pytest.mark.gpu

LATTICES = {
    "octet2-graded": lambda: synth.graded_radii(synth.octet(2, 2, 2), 0.03, 0.06),
    "bcc3-jitter": lambda: synth.jitter(synth.bcc(3, 3, 3), 0.05, 1),
    "stochastic9": lambda: synth.stochastic(9, seed=7),
    "crown16": lambda: synth.star([[0, 0, 1]] + [[np.sin(0.7) * np.cos(t), np.sin(0.7) * np.sin(t), np.cos(0.7)]
                                                 for t in np.linspace(0, 2 * np.pi, 16, endpoint=False)], 1.0, 0.05),
    "voronoi": lambda: synth.voronoi_like(300, seed=3, radius=0.05),
}

# (path, window points, span triangles): the band path; the CTA path at its default; small
# windows (long-band fallback inside a span); tiny spans (every band clipped somewhere)
SETTINGS = [("0", None, None), ("1", None, None), ("1", "256", None), ("1", None, "128"), ("1", "256", "64")]


@pytest.fixture(scope="module")
def meshes():
    from paper_2405_15197_b200 import MetaMesher
    from paper_2405_15197_b200 import build as b
    b.build()
    cache = {}

    def get(name):
        if name not in cache:
            lat = LATTICES[name]()
            cache[name] = (lat, MetaMesher(0).load_lattice(lat).build())
        return cache[name]
    return get


def _emit(mm, T, setting, ranges=()):
    from paper_2405_15197_b200 import binding as B
    path, pcw, span = setting
    keys = {"LMM_EMIT_PATH": path, "LMM_SPCW": pcw, "LMM_SPAN": span}
    old = {k: os.environ.get(k) for k in keys}
    try:
        for k, v in keys.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        full = mm.triangles(0, T)
        assert B.lmm_emit_path(mm.h) == int(path)   # the kernel that wrote the band region
        parts = [mm.triangles(a, b - a) for a, b in ranges]
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return full, parts


@pytest.mark.parametrize("name", list(LATTICES))
@pytest.mark.parametrize("ce", [5e-2, 1e-2, 1e-3])
def test_emit_paths_bit_identical(meshes, name, ce):
    lat, mm = meshes(name)
    T = mm.triangulate(ce)
    rng = np.random.default_rng(int(ce * 1e6) + len(name))
    ranges = []
    for _ in range(6):
        a = int(rng.integers(0, T))
        ranges.append((a, int(rng.integers(a, min(T, a + 3000) + 1))))
    ref, ref_parts = _emit(mm, T, SETTINGS[0], ranges)
    for s in SETTINGS[1:]:
        got, parts = _emit(mm, T, s, ranges)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (name, ce, s)
        for (a, b), p, q in zip(ranges, parts, ref_parts):
            assert np.array_equal(p.view(np.uint32), q.view(np.uint32)), (name, ce, s, a, b)
            assert np.array_equal(p.view(np.uint32), ref[a:b].view(np.uint32)), (name, ce, s, a, b)


@pytest.mark.parametrize("name", ["stochastic9", "voronoi"])
def test_cta_path_matches_oracle(meshes, name):
    lat, mm = meshes(name)
    orc = oracle.Oracle.from_lattice(lat)
    assert orc.metamesh() == 0
    for ce in (1e-2, 1e-3):
        T = mm.triangulate(ce)
        assert T == orc.triangulate(ce)
        got, _ = _emit(mm, T, ("1", "256", "128"))
        assert_triangles_close(got.astype(np.float64), orc.write_triangles(), float(lat.node_r.min()), (name, ce))
