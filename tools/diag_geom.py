"""Locate the largest kernel-vs-oracle triangle vertex error (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from test_gpu_parity import _lat
from paper_2405_15197_b200 import MetaMesher, decode_node
name = sys.argv[1] if len(sys.argv) > 1 else "voronoi"
ce = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
lat = _lat(name)
mm = MetaMesher(0).load_lattice(lat).build()
orc = oracle.Oracle.from_lattice(lat); orc.metamesh()
T = mm.triangulate(ce); orc.triangulate(ce)
tri = mm.triangles(0, T).astype(np.float64); ref = orc.write_triangles()
err = np.abs(tri[:, 1:] - ref[:, 1:]).max(axis=2)   # [T,3]
t, v = np.unravel_index(np.argmax(err), err.shape)
print("max err", err.max(), "triangle", t, "vertex", v, "ref", ref[t, 1 + v], "gpu", tri[t, 1 + v])
bn, soff = orc.band_info()
s = int(np.searchsorted(soff, t, side="right") - 1)
print("strut", s, "ends", lat.ends[s] if s < lat.n_struts else None, "band", bn[s] if s < lat.n_struts else None)
# worst vertices per node: compare meta-mesh geometry and conditioning
bufs = mm.buffers()
worst = []
for n in lat.ends[s] if s < lat.n_struts else []:
    g, o = decode_node(bufs, int(n)), orc.node(int(n))
    ve = np.abs(g["v_pos32"] - o["v_pos64"]).max(axis=1)
    ae = np.abs(g["a_f32"][:, 2:] - o["a_f64"][:, 2:]).max(axis=1)
    A = o["a_f64"][:, 5:8]; Bv = o["a_f64"][:, 8:11]
    print("node", n, "R", lat.node_r[n], "vertex err max", ve.max(), "arc err max", ae.max())
    for i in np.argsort(-ae)[:3]:
        print("   arc", i, o["a_int"][i], "err", ae[i], "|a|", np.linalg.norm(A[i]), "|b|", np.linalg.norm(Bv[i]),
              "t0/dt f32", g["a_f32"][i, :2], "f64", o["a_f64"][i, :2])
