"""ctypes wrapper of oracle/mm_oracle.c -- TEST INFRASTRUCTURE ONLY (see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mm_oracle.c")
_LIBS = {32: os.path.join(_HERE, "liborc.so"), 64: os.path.join(_HERE, "liborc64.so")}
_lock = threading.Lock()
_libs = {}

# binary32 topology decisions must not be contracted into FMAs or reassociated
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared", "-Wall"]
# liborc64.so: the same source with every decision in binary64 (DESIGN.md Sec. 9 pin)
CFLAGS64 = ["-DORC_REAL64"]

ORC_STATUS = {0: "ok", 1: "degree>63", 2: "bad strut", 3: "(reserved)", 4: "(reserved)",
              5: "(reserved)", 6: "unbounded conic", 7: "unreferenced vertex", 8: "loop chain",
              9: "loop angle sum", 10: "empty loop", 11: "hole chain", 12: "strut too short",
              13: "(reserved)"}
MAX_DEGREE = 63


def build_oracle(force: bool = False) -> str:
    """Compile the C oracle (binary32 decisions) and its binary64-decision twin with gcc
    (building the checker is not using it)."""
    with _lock:
        for bits, lib in _LIBS.items():
            if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(_SRC):
                tmp = lib + f".tmp{os.getpid()}"
                subprocess.check_call(["gcc", *CFLAGS, *(CFLAGS64 if bits == 64 else []), "-o", tmp, _SRC, "-lm"])
                os.replace(tmp, lib)
    return _LIBS[32]


def _load(bits: int = 32):
    if bits not in _libs:
        build_oracle()
        lib = C.CDLL(_LIBS[bits])
        P = C.c_void_p
        i64, i32, f32, f64 = C.c_int64, C.c_int32, C.c_float, C.c_double
        lib.orc_create.restype = P
        lib.orc_create.argtypes = [P, P, i64, P, i64]
        lib.orc_destroy.argtypes = [P]
        lib.orc_metamesh.restype = C.c_int
        lib.orc_metamesh.argtypes = [P, P, i64]
        lib.orc_metamesh_scan.argtypes = [P, P, i64, P, P]
        lib.orc_set_jitter.argtypes = [P, f64, C.c_uint64]
        lib.orc_node_counts.restype = C.c_int
        lib.orc_node_counts.argtypes = [P, i64, P]
        for name in ("orc_node_verts", "orc_node_arcs", "orc_node_loops"):
            getattr(lib, name).argtypes = [P, i64, P, P, P]
        lib.orc_node_holes.argtypes = [P, i64, P, P]
        lib.orc_csr.argtypes = [P, P, P]
        lib.orc_triangulate.restype = i64
        lib.orc_triangulate.argtypes = [P, f64]
        lib.orc_band_info.argtypes = [P, P, P]
        lib.orc_n_holes.restype = i64
        lib.orc_n_holes.argtypes = [P]
        lib.orc_hole_info.argtypes = [P, P, P, P]
        lib.orc_strut_triangles.restype = i64
        lib.orc_strut_triangles.argtypes = [P, i64, P]
        lib.orc_node_hole_triangles.restype = i64
        lib.orc_node_hole_triangles.argtypes = [P, i64, P]
        lib.orc_write_triangles.restype = i64
        lib.orc_write_triangles.argtypes = [P, i64, i64, P]
        lib.orc_atan2p.restype = f32
        lib.orc_atan2p.argtypes = [f32, f32]
        lib.orc_theta0.restype = f32
        lib.orc_theta0.argtypes = [f64]
        lib.orc_subdiv_count.restype = C.c_int
        lib.orc_subdiv_count.argtypes = [f32, f32]
        lib.orc_eq7.argtypes = [P, f64, f64, P, f64, P, P]
        lib.orc_aux_plane.argtypes = [P, f64, P, f64, f64, P, P]
        lib.orc_eq9.restype = C.c_int
        lib.orc_eq9.argtypes = [P, P, P, P, P, P, P]
        _libs[bits] = lib
    return _libs[bits]


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Per-lattice oracle state: CSR, per-node meta-meshes, triangulation."""

    def __init__(self, xyz, node_r, ends, bits: int = 32):
        """bits = 32: the oracle (binary32 decisions); bits = 64: its binary64-decision twin."""
        self.lib = _load(bits)
        self.xyz = np.ascontiguousarray(xyz, dtype=np.float32)
        self.node_r = np.ascontiguousarray(node_r, dtype=np.float32)
        self.ends = np.ascontiguousarray(ends, dtype=np.int64)
        self.n_nodes = len(self.xyz)
        self.n_struts = len(self.ends)
        self.h = self.lib.orc_create(_p(self.xyz), _p(self.node_r), self.n_nodes, _p(self.ends), self.n_struts)

    @classmethod
    def from_lattice(cls, lat, bits: int = 32):
        return cls(lat.xyz, lat.node_r, lat.ends, bits)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_destroy(self.h)
            self.h = None

    # ---- meta-mesh ------------------------------------------------------------------
    def metamesh(self, nodes=None) -> int:
        """Compute the meta-mesh of `nodes` (all when None); returns #nodes in error."""
        if nodes is None:
            return self.lib.orc_metamesh(self.h, None, 0)
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        return self.lib.orc_metamesh(self.h, _p(nodes), len(nodes))

    def scan(self, nodes) -> tuple[np.ndarray, np.ndarray]:
        """Meta-mesh `nodes` one at a time, keeping nothing: (status int32, topology digest uint64)."""
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        st = np.zeros(len(nodes), np.int32)
        hs = np.zeros(len(nodes), np.uint64)
        self.lib.orc_metamesh_scan(self.h, _p(nodes), len(nodes), _p(st), _p(hs))
        return st, hs

    def set_jitter(self, eps: float, seed: int) -> None:
        """binary64 twin only: seeded relative jitter of the side parameters (0 = off)."""
        self.lib.orc_set_jitter(self.h, float(eps), int(seed))

    def csr(self):
        off = np.zeros(self.n_nodes + 1, np.int64)
        st = np.zeros(2 * self.n_struts, np.int64)
        self.lib.orc_csr(self.h, _p(off), _p(st))
        return off, st

    def node(self, n: int) -> dict:
        cnt = np.zeros(7, np.int32)
        done = self.lib.orc_node_counts(self.h, n, _p(cnt))
        status, d, nv, na, nh, nle, nhe = (int(x) for x in cnt)
        out = dict(done=bool(done), status=status, d=d, nv=nv, na=na, nh=nh)
        mask = np.zeros(nv, np.uint64)
        p32 = np.zeros((nv, 3), np.float32)
        p64 = np.zeros((nv, 3), np.float64)
        self.lib.orc_node_verts(self.h, n, _p(mask), _p(p32), _p(p64))
        ai = np.zeros((na, 4), np.int32)
        af = np.zeros((na, 11), np.float32)
        ad = np.zeros((na, 11), np.float64)
        self.lib.orc_node_arcs(self.h, n, _p(ai), _p(af), _p(ad))
        loff = np.zeros(d + 1, np.int32)
        li = np.zeros((nle, 2), np.int32)
        lf = np.zeros((nle, 2), np.float32)
        self.lib.orc_node_loops(self.h, n, _p(loff), _p(li), _p(lf))
        hoff = np.zeros(nh + 1, np.int32)
        hi = np.zeros((nhe, 2), np.int32)
        self.lib.orc_node_holes(self.h, n, _p(hoff), _p(hi))
        out.update(v_mask=mask, v_pos32=p32, v_pos64=p64, a_int=ai, a_f32=af, a_f64=ad,
                   loop_off=loff, l_int=li, l_f32=lf, hole_off=hoff, h_int=hi)
        return out

    # ---- triangulation ----------------------------------------------------------------
    def triangulate(self, ce: float) -> int:
        return int(self.lib.orc_triangulate(self.h, float(ce)))

    def band_info(self):
        bn = np.zeros((self.n_struts, 3), np.int64)
        off = np.zeros(self.n_struts + 1, np.int64)
        self.lib.orc_band_info(self.h, _p(bn), _p(off))
        return bn, off

    def hole_info(self):
        H = int(self.lib.orc_n_holes(self.h))
        base = np.zeros(self.n_nodes + 1, np.int64)
        M = np.zeros(H, np.int64)
        bp = np.zeros((H, 3), np.float64)
        self.lib.orc_hole_info(self.h, _p(base), _p(M), _p(bp))
        return base, M, bp

    def strut_triangles(self, s: int) -> np.ndarray:
        bn, _ = self.band_info() if not hasattr(self, "_bn") else (self._bn, None)
        n = int(bn[s, 0] + bn[s, 1])
        out = np.zeros((max(n, 1), 12), np.float64)
        k = self.lib.orc_strut_triangles(self.h, s, _p(out))
        return out[:k].reshape(-1, 4, 3)

    def node_hole_triangles(self, n: int) -> np.ndarray:
        k = self.lib.orc_node_hole_triangles(self.h, n, None)
        out = np.zeros((max(k, 1), 12), np.float64)
        self.lib.orc_node_hole_triangles(self.h, n, _p(out))
        return out[:k].reshape(-1, 4, 3)

    def write_triangles(self, first: int = 0, count: int | None = None) -> np.ndarray:
        """Triangles in the global order as float64 [count, 4, 3] = normal, v1, v2, v3."""
        total = self.n_tri_total()
        if count is None:
            count = total - first
        out = np.zeros((max(count, 1), 12), np.float64)
        k = self.lib.orc_write_triangles(self.h, first, count, _p(out))
        return out[:k].reshape(-1, 4, 3)

    def n_tri_total(self) -> int:
        bn, off = self.band_info()
        _, M, _ = self.hole_info()
        return int(off[-1] + M.sum())


# ---- building blocks (pins) -----------------------------------------------------------
def atan2p(y: float, x: float) -> float:
    return float(_load().orc_atan2p(np.float32(y), np.float32(x)))


def theta0(ce: float) -> float:
    return float(_load().orc_theta0(ce))


def subdiv_count(dt: float, th0: float) -> int:
    return int(_load().orc_subdiv_count(np.float32(dt), np.float32(th0)))


def eq7(u, s, R, n, pc, e1):
    """Eq. 7 ellipse of the cone (node at origin, radius R, unit direction u, sin(beta)=s)
    cut by the plane n.y = pc; returns (o, a, b) float64."""
    u = np.ascontiguousarray(u, np.float64)
    n = np.ascontiguousarray(n, np.float64)
    e1 = np.ascontiguousarray(e1, np.float64)
    out = np.zeros(9, np.float64)
    _load().orc_eq7(_p(u), float(s), float(R), _p(n), float(pc), _p(e1), _p(out))
    return out[0:3], out[3:6], out[6:9]


def aux_plane(ua, sa, ub, sb, R):
    ua = np.ascontiguousarray(ua, np.float64)
    ub = np.ascontiguousarray(ub, np.float64)
    n = np.zeros(3, np.float64)
    pc = np.zeros(1, np.float64)
    _load().orc_aux_plane(_p(ua), float(sa), _p(ub), float(sb), float(R), _p(n), _p(pc))
    return n, float(pc[0])


def eq9(o, a, b, n, p):
    """Returns (kind, lo, length): kind 1 FULL, 0 EMPTY, 2 range [lo, lo+length)."""
    arrs = [np.ascontiguousarray(x, np.float64) for x in (o, a, b, n, p)]
    lo = np.zeros(1)
    ln = np.zeros(1)
    k = _load().orc_eq9(*[_p(x) for x in arrs], _p(lo), _p(ln))
    return int(k), float(lo[0]), float(ln[0])
