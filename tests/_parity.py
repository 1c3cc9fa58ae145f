"""Shared parity assertions of the GPU tests (CUDA path vs CPU oracle, per node / per band)."""
import numpy as np

# north_star: geometry within 1e-4 x the minimum strut radius (binary32 kernel vs binary64 oracle)
GEOM_TOL = 1e-4


def assert_node_parity(g: dict, o: dict, tol: float, n) -> None:
    """Topology bit-exact (counts, masks, endpoints, loop order, binary32 decision values),
    geometry within `tol`."""
    assert (g["status"], g["d"]) == (o["status"], o["d"]), (n, g["status"], o["status"])
    if o["status"]:
        return
    assert (g["nv"], g["na"], g["nh"]) == (o["nv"], o["na"], o["nh"]), n
    assert np.array_equal(g["v_mask"], o["v_mask"]), n
    assert np.array_equal(g["v_pos32"].view(np.uint32), o["v_pos32"].view(np.uint32)), n
    assert np.array_equal(g["a_int"], o["a_int"]), n
    assert np.array_equal(g["a_f32"].view(np.uint32), o["a_f32"].view(np.uint32)), n   # t0, dt, conic (binary32)
    assert np.array_equal(g["loop_off"], o["loop_off"]), n
    assert np.array_equal(g["l_int"], o["l_int"]), n
    assert np.array_equal(g["l_f32"].view(np.uint32), o["l_f32"].view(np.uint32)), n
    assert np.array_equal(g["hole_off"], o["hole_off"]) and np.array_equal(g["h_int"], o["h_int"]), n
    if g["nv"]:
        assert np.max(np.abs(g["v_pos32"] - o["v_pos64"])) < tol, n
    if g["na"]:
        assert np.max(np.abs(g["a_f32"][:, 2:] - o["a_f64"][:, 2:])) < tol, n


# binary32 conditioning allowance for lattices with struts 10 degrees apart: their
# near-parabolic Eq. 7 sections (|a| ~ 10 R) carry errors up to 1.9e-4 r_min in the conic and
# on the arc in ~0.4 % of nodes (R13); topology stays bit-exact
GEOM_TOL_SHARP = 2.5e-4


def triangle_tolerance(ref: np.ndarray, r_min: float, geom_tol: float = GEOM_TOL) -> np.ndarray:
    """Per-coordinate bound for a binary32 triangle vertex against the binary64 oracle:
    north_star's 1e-4 x r_min plus one unit in the last place of the binary32 coordinate
    (the output is binary32 STL, so its own rounding of |x| is unavoidable)."""
    return geom_tol * r_min + np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)


def assert_triangles_close(tri: np.ndarray, ref: np.ndarray, r_min: float, what, geom_tol: float = GEOM_TOL) -> float:
    """Triangle vertices: binary32 kernel vs binary64 oracle, every coordinate within
    1e-4 r_min + ulp(|x_ref|).  Returns the largest error / tolerance ratio."""
    assert tri.shape == ref.shape, (what, tri.shape, ref.shape)
    if len(tri) == 0:
        return 0.0
    err = np.abs(tri[:, 1:].astype(np.float64) - ref[:, 1:])
    tol = triangle_tolerance(ref[:, 1:], r_min, geom_tol)
    ratio = float(np.max(err / tol))
    assert ratio <= 1.0, (what, float(err.max()), ratio)
    return ratio
