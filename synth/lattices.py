"""Seeded synthetic lattices shaped like the paper's workloads (Sec. 6,
Table 1: uniform cells, graded radii, irregular high-degree node mixes).

Every generator returns a `Lattice`: float32 node positions, int64 strut index
pairs, float32 node (sphere) radii and the per-end strut radii derived from them
(struts are tangent to the nodal spheres, Sec. 4.1 last paragraph, so a
strut's radius at an end is that node's sphere radius).

Node order is lattice (spatially coherent) order; struts are sorted by
(min endpoint, max endpoint).  Nothing here computes any meta-mesh quantity.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class Lattice:
    xyz: np.ndarray      # float32 [N, 3]
    ends: np.ndarray     # int64   [S, 2]
    node_r: np.ndarray   # float32 [N]
    name: str = "lattice"
    ijk: np.ndarray | None = None   # int64 [N, 3] integer lattice coordinates (windowed generators)
    gid: np.ndarray | None = None   # int64 [N] global node ids (windowed generators), ascending

    @property
    def n_nodes(self) -> int:
        return int(self.xyz.shape[0])

    @property
    def n_struts(self) -> int:
        return int(self.ends.shape[0])

    @property
    def r_end(self) -> np.ndarray:
        """Per-end strut radii, float32 [S, 2] (r_i^0, r_i^1 of PAPER.md Sec. 4.3.1)."""
        return self.node_r[self.ends].astype(np.float32)

    def degrees(self) -> np.ndarray:
        return np.bincount(self.ends.ravel(), minlength=self.n_nodes)

    def genus(self) -> int:
        """Cycle rank S - N + C of the strut graph = genus of the lattice's boundary
        surface (the boundary of a thickened connected graph is a closed surface of
        genus equal to the graph's first Betti number)."""
        n = self.n_nodes
        parent = np.arange(n)

        def find(a):
            while parent[a] != a:
                parent[a] = parent[parent[a]]
                a = parent[a]
            return a
        used = np.zeros(n, dtype=bool)
        for a, b in self.ends:
            used[a] = used[b] = True
            ra, rb = find(a), find(b)
            if ra != rb:
                parent[ra] = rb
        comps = len({find(i) for i in range(n) if used[i]})
        return int(self.n_struts - int(used.sum()) + comps)


def _finish(xyz, ends, node_r, name) -> Lattice:
    ends = np.asarray(ends, dtype=np.int64).reshape(-1, 2)
    n = max(len(xyz), 1)
    key = np.sort(np.minimum(ends[:, 0], ends[:, 1]) * n + np.maximum(ends[:, 0], ends[:, 1]))
    ends = np.stack([key // n, key % n], axis=1)   # sorted by (min endpoint, max endpoint)
    return Lattice(np.ascontiguousarray(xyz, dtype=np.float32), np.ascontiguousarray(ends),
                   np.ascontiguousarray(node_r, dtype=np.float32), name)


def _radii(n, radius):
    return np.full(n, radius, dtype=np.float32)


def cubic(nx: int, ny: int, nz: int, pitch: float = 1.0, radius: float = 0.1) -> Lattice:
    """Simple cubic grid with nx*ny*nz NODES and axis-aligned struts
    (SPEC.md lattice_io example: grid(3,3,3) -> 27 nodes, 54 struts)."""
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    idx = lambda i, j, k: (i * ny + j) * nz + k
    ends = []
    for ax, lim in enumerate((nx, ny, nz)):
        m = g[:, ax] < lim - 1
        a = g[m]
        b = a.copy()
        b[:, ax] += 1
        ends.append(np.stack([idx(*a.T), idx(*b.T)], 1))
    xyz = g.astype(np.float64) * pitch
    return _finish(xyz, np.concatenate(ends), _radii(len(g), radius), f"cubic{nx}x{ny}x{nz}")


def bcc(nx: int, ny: int, nz: int, pitch: float = 1.0, radius: float = 0.05) -> Lattice:
    """Body-centred cubic lattice of nx*ny*nz CELLS: cell corners plus one centre node
    per cell, each centre joined to its 8 corners (8 struts per cell; 10x10x10 cells
    = 8000 struts, BASELINE.json configs[0])."""
    cx, cy, cz = nx + 1, ny + 1, nz + 1
    corners = np.stack(np.meshgrid(np.arange(cx), np.arange(cy), np.arange(cz), indexing="ij"), -1).reshape(-1, 3)
    cells = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    n_corner = len(corners)
    cidx = lambda i, j, k: (i * cy + j) * cz + k
    ends = []
    centre_ids = n_corner + np.arange(len(cells))
    for di in (0, 1):
        for dj in (0, 1):
            for dk in (0, 1):
                ends.append(np.stack([centre_ids, cidx(cells[:, 0] + di, cells[:, 1] + dj, cells[:, 2] + dk)], 1))
    xyz = np.concatenate([corners.astype(np.float64), cells.astype(np.float64) + 0.5]) * pitch
    return _finish(xyz, np.concatenate(ends), _radii(len(xyz), radius), f"bcc{nx}x{ny}x{nz}")


def bcc_slab(nx: int, ny: int, nz: int, z0: int, z1: int, pitch: float = 1.0, radius: float = 0.05) -> Lattice:
    """The cells with z-index in [z0, z1) of an nx*ny*nz-cell BCC lattice (a spatial
    block for multi-GPU partitioning).  Node positions are the global ones."""
    lat = bcc(nx, ny, z1 - z0, pitch, radius)
    xyz = lat.xyz.astype(np.float64)
    xyz[:, 2] += z0 * pitch
    return Lattice(xyz.astype(np.float32), lat.ends, lat.node_r, f"bccslab{nx}x{ny}x{nz}[{z0}:{z1}]")


def octet(nx: int, ny: int, nz: int, pitch: float = 1.0, radius: float = 0.04) -> Lattice:
    """Octet truss of nx*ny*nz cubic CELLS = FCC points (cell corners + face centres)
    joined to their 12 nearest neighbours (24 struts per cell; 100^3 cells ~ 24M)."""
    # FCC points = integer points of [0,2nx]x[0,2ny]x[0,2nz] with even coordinate sum.
    g = np.stack(np.meshgrid(np.arange(2 * nx + 1), np.arange(2 * ny + 1), np.arange(2 * nz + 1),
                             indexing="ij"), -1).reshape(-1, 3)
    g = g[(g.sum(1) % 2) == 0]
    lut = -np.ones((2 * nx + 1, 2 * ny + 1, 2 * nz + 1), dtype=np.int64)
    lut[g[:, 0], g[:, 1], g[:, 2]] = np.arange(len(g))
    offs = np.array([(1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1), (0, 1, 1), (0, 1, -1)])
    ends = []
    lim = np.array([2 * nx, 2 * ny, 2 * nz])
    for o in offs:
        q = g + o
        m = np.all((q >= 0) & (q <= lim), axis=1)
        ends.append(np.stack([np.nonzero(m)[0], lut[q[m, 0], q[m, 1], q[m, 2]]], 1))
    xyz = g.astype(np.float64) * (0.5 * pitch)
    return _finish(xyz, np.concatenate(ends), _radii(len(g), radius), f"octet{nx}x{ny}x{nz}")


def octet_window(nx: int, ny: int, nz: int, k_lo: int, k_hi: int, pitch: float = 1.0,
                 radius: float = 0.04, r_max: float | None = None) -> Lattice:
    """The part of the octet truss of nx*ny*nz cells whose FCC points have half-pitch z index
    k in [k_lo, k_hi] (clipped to [0, 2nz]), with the struts among them.  Nodes are listed in
    ascending global id gid = (i*(2ny+1) + j)*(2nz+1) + k and struts in ascending (gid, gid),
    so any two windows order the struts of a shared node identically.  With r_max given, node
    radii are graded radius..r_max along x (as graded_radii on the full lattice)."""
    k_lo, k_hi = max(0, k_lo), min(2 * nz, k_hi)
    I, J, K = np.meshgrid(np.arange(2 * nx + 1), np.arange(2 * ny + 1), np.arange(k_lo, k_hi + 1), indexing="ij")
    g = np.stack([I, J, K], -1).reshape(-1, 3)
    g = g[(g.sum(1) % 2) == 0]
    lut = -np.ones((2 * nx + 1, 2 * ny + 1, k_hi - k_lo + 1), dtype=np.int64)
    lut[g[:, 0], g[:, 1], g[:, 2] - k_lo] = np.arange(len(g))
    offs = np.array([(1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1), (0, 1, 1), (0, 1, -1)])
    ends = []
    lim_lo = np.array([0, 0, k_lo])
    lim_hi = np.array([2 * nx, 2 * ny, k_hi])
    for o in offs:
        q = g + o
        m = np.all((q >= lim_lo) & (q <= lim_hi), axis=1)
        ends.append(np.stack([np.nonzero(m)[0], lut[q[m, 0], q[m, 1], q[m, 2] - k_lo]], 1))
    xyz = g.astype(np.float64) * (0.5 * pitch)
    if r_max is None:
        r = np.full(len(g), radius)
    else:
        x = g[:, 0].astype(np.float64) / (2 * nx)
        r = radius + (r_max - radius) * x
    lat = _finish(xyz, np.concatenate(ends), r, f"octetwin{nx}x{ny}x{nz}[{k_lo}:{k_hi}]")
    lat.ijk = g.astype(np.int64)
    lat.gid = (g[:, 0].astype(np.int64) * (2 * ny + 1) + g[:, 1]) * (2 * nz + 1) + g[:, 2]
    return lat


def star(directions, lengths=1.0, radius: float = 0.1, far_radii=None) -> Lattice:
    """One centre node (index 0) joined to far nodes along `directions`."""
    d = np.asarray(directions, dtype=np.float64)
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    ln = np.broadcast_to(np.asarray(lengths, dtype=np.float64), (len(d),))
    xyz = np.concatenate([np.zeros((1, 3)), d * ln[:, None]])
    r = np.full(len(xyz), radius, dtype=np.float64)
    if far_radii is not None:
        r[1:] = far_radii
    ends = np.stack([np.zeros(len(d), dtype=np.int64), 1 + np.arange(len(d))], 1)
    return _finish(xyz, ends, r, f"star{len(d)}")


def single_strut(length: float = 1.0, r0: float = 0.1, r1: float = 0.1) -> Lattice:
    xyz = np.array([[0.0, 0.0, 0.0], [length, 0.0, 0.0]])
    return _finish(xyz, [[0, 1]], np.array([r0, r1]), "single")


def chain(n: int = 3, pitch: float = 1.0, radius: float = 0.1, bend_deg: float = 0.0) -> Lattice:
    """n nodes on a polyline; each interior node bends the chain by bend_deg."""
    pts = [np.zeros(3)]
    ang = 0.0
    for _ in range(n - 1):
        pts.append(pts[-1] + pitch * np.array([np.cos(ang), np.sin(ang), 0.0]))
        ang += np.deg2rad(bend_deg)
    ends = [[i, i + 1] for i in range(n - 1)]
    return _finish(np.array(pts), ends, _radii(n, radius), f"chain{n}")


def jitter(lat: Lattice, amount: float, seed: int = 0) -> Lattice:
    """Perturb node positions by uniform noise in [-amount, amount]^3 (seeded)."""
    rng = np.random.default_rng(seed)
    xyz = lat.xyz.astype(np.float64) + rng.uniform(-amount, amount, size=lat.xyz.shape)
    return Lattice(xyz.astype(np.float32), lat.ends.copy(), lat.node_r.copy(), lat.name + f"+jit{amount}")


def graded_radii(lat: Lattice, r_min: float, r_max: float, axis: int = 0) -> Lattice:
    """Node radius graded linearly along `axis` from r_min to r_max (conical struts
    wherever an edge is not perpendicular to `axis`; BASELINE.json configs[1])."""
    x = lat.xyz[:, axis].astype(np.float64)
    span = max(float(x.max() - x.min()), 1e-30)
    r = r_min + (r_max - r_min) * (x - x.min()) / span
    return Lattice(lat.xyz.copy(), lat.ends.copy(), r.astype(np.float32), lat.name + "+graded")


def voronoi_like(n_nodes: int, seed: int = 0, deg_min: int = 3, deg_max: int = 30,
                 radius: float = 0.03, min_angle_deg: float = 28.0) -> Lattice:
    """Stochastic lattice with skewed node degrees (BASELINE.json configs[2] shape).

    Nodes: a jittered grid.  Each node draws a target degree from a Zipf-like
    distribution on [deg_min, deg_max]; candidate struts are the node's nearest
    neighbours, accepted greedily (shortest first) while both endpoints stay under
    their target degree and every pair of struts at a node stays at least
    `min_angle_deg` apart (so strut pairs meet in bounded conics)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    side = int(np.ceil(n_nodes ** (1 / 3)))
    g = np.stack(np.meshgrid(np.arange(side), np.arange(side), np.arange(side), indexing="ij"), -1).reshape(-1, 3)[:n_nodes]
    xyz = g + rng.uniform(-0.3, 0.3, size=g.shape)
    ks = np.arange(deg_min, deg_max + 1)
    p = 1.0 / (ks - deg_min + 1.0) ** 1.3
    target = rng.choice(ks, size=n_nodes, p=p / p.sum())
    tree = cKDTree(xyz)
    k = min(deg_max + 12, n_nodes)
    dist, nbr = tree.query(xyz, k=k)
    cand = [(dist[i, j], i, nbr[i, j]) for i in range(n_nodes) for j in range(1, k) if i < nbr[i, j]]
    cand.sort()
    cos_lim = np.cos(np.deg2rad(min_angle_deg))
    dirs = [[] for _ in range(n_nodes)]
    deg = np.zeros(n_nodes, dtype=np.int64)
    ends = []
    for _, a, b in cand:
        if deg[a] >= target[a] or deg[b] >= target[b]:
            continue
        v = xyz[b] - xyz[a]
        v = v / np.linalg.norm(v)
        if any(float(v @ w) > cos_lim for w in dirs[a]) or any(float(-v @ w) > cos_lim for w in dirs[b]):
            continue
        dirs[a].append(v)
        dirs[b].append(-v)
        deg[a] += 1
        deg[b] += 1
        ends.append((a, b))
    return _finish(xyz, ends, _radii(n_nodes, radius), f"voronoi{n_nodes}")


_STOCH_LIB = None


def _stoch_lib():
    """gcc-built helper of stochastic() (strut selection loop; input generation only)."""
    global _STOCH_LIB
    if _STOCH_LIB is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, so = os.path.join(here, "_stochastic.c"), os.path.join(here, "_stochastic.so")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            tmp = so + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, src, "-lm"])
            os.replace(tmp, so)
        lib = ctypes.CDLL(so)
        P = ctypes.c_void_p
        lib.stoch_struts.restype = ctypes.c_int64
        lib.stoch_struts.argtypes = [P, ctypes.c_int64, P, P, ctypes.c_double, ctypes.c_int64, P]
        i64 = ctypes.c_int64
        lib.stoch_zone.restype = i64
        lib.stoch_zone.argtypes = [P, i64, i64, i64, i64, i64, P, P, ctypes.c_double, i64, P, P, i64, P]
        _STOCH_LIB = lib
    return _STOCH_LIB


def stochastic(side: int, seed: int = 0, deg_min: int = 3, deg_max: int = 30, r_min: float = 0.02,
               r_max: float = 0.04, min_angle_deg: float = 25.0, zipf: float = 1.1) -> Lattice:
    """Stochastic Voronoi-style lattice with skewed node degrees 3..30 (BASELINE.json
    configs[2]: "~100M struts, load-balance stress"; side = 300 gives ~1e8 struts).

    Nodes: a side^3 grid jittered by U(-0.3, 0.3) per axis.  Each node draws a target
    degree from a Zipf-like law p(k) ~ (k - deg_min + 1)^-zipf on [deg_min, deg_max] and
    a sphere radius U(r_min, r_max) (so struts are cones).  Struts: nodes in descending
    target order take their nearest neighbours (5x5x5 surrounding cells) while both ends
    are under target and every two struts at a node stay >= min_angle_deg apart
    (synth/_stochastic.c).  Isolated nodes are possible and carry no surface."""
    rng = np.random.default_rng(seed)
    n = side ** 3
    g = np.stack(np.meshgrid(np.arange(side), np.arange(side), np.arange(side), indexing="ij"), -1).reshape(-1, 3)
    xyz = g + rng.uniform(-0.3, 0.3, size=g.shape)
    del g
    ks = np.arange(deg_min, deg_max + 1)
    p = 1.0 / (ks - deg_min + 1.0) ** zipf
    target = rng.choice(ks, size=n, p=p / p.sum()).astype(np.int32)
    radius = rng.uniform(r_min, r_max, size=n)
    order = np.argsort(-target, kind="stable").astype(np.int64)
    cap = int(target.astype(np.int64).sum() // 2) + 1
    ends = np.zeros((cap, 2), np.int64)
    xyz = np.ascontiguousarray(xyz, np.float64)
    S = _stoch_lib().stoch_struts(xyz.ctypes.data, side, target.ctypes.data, order.ctypes.data,
                                  float(np.cos(np.deg2rad(min_angle_deg))), cap, ends.ctypes.data)
    if S < 0:
        raise RuntimeError(f"stochastic lattice generator failed ({S})")
    return _finish(xyz, ends[:S], radius, f"stochastic{side}^3")


def bcc_window(nx: int, ny: int, nz: int, k_lo: int, k_hi: int, pitch: float = 1.0,
               radius: float = 0.05) -> Lattice:
    """The part of the BCC lattice of nx*ny*nz cells whose nodes have half-pitch z index k in
    [k_lo, k_hi] (clipped to [0, 2nz]), with the struts among them (spatial blocks of the
    multi-GPU partition, BASELINE.json configs[3]).  In half-pitch integer coordinates the
    cell corners are the all-even points and the cell centres the all-odd ones; each centre
    joins its 8 corners (offsets (+-1, +-1, +-1)).  Nodes ascend in global id
    gid = (i*(2ny+1) + j)*(2nz+1) + k, struts in (gid, gid), as octet_window."""
    k_lo, k_hi = max(0, k_lo), min(2 * nz, k_hi)
    I, J, K = np.meshgrid(np.arange(2 * nx + 1, dtype=np.int32), np.arange(2 * ny + 1, dtype=np.int32),
                          np.arange(k_lo, k_hi + 1, dtype=np.int32), indexing="ij")
    par = (I & 1)
    keep = (par == (J & 1)) & (par == (K & 1))
    g = np.stack([I[keep], J[keep], K[keep]], -1)      # meshgrid order = ascending gid
    del I, J, K, par, keep
    nk = k_hi - k_lo + 1
    lut = -np.ones((2 * nx + 1, 2 * ny + 1, nk), dtype=np.int64)
    lut[g[:, 0], g[:, 1], g[:, 2] - k_lo] = np.arange(len(g))
    cen = np.nonzero(g[:, 0] & 1)[0]
    gc = g[cen]
    ends = []
    for o in [(a, b, c) for a in (-1, 1) for b in (-1, 1) for c in (-1, 1)]:
        q = gc + np.array(o, np.int32)
        m = (q[:, 2] >= k_lo) & (q[:, 2] <= k_hi)        # x, y stay inside: centres are interior
        ends.append(np.stack([cen[m], lut[q[m, 0], q[m, 1], q[m, 2] - k_lo]], 1))
    del lut
    xyz = g.astype(np.float64) * (0.5 * pitch)
    lat = _finish(xyz, np.concatenate(ends), np.full(len(g), radius), f"bccwin{nx}x{ny}x{nz}[{k_lo}:{k_hi}]")
    lat.ijk = g.astype(np.int64)
    lat.gid = (lat.ijk[:, 0] * (2 * ny + 1) + lat.ijk[:, 1]) * (2 * nz + 1) + lat.ijk[:, 2]
    return lat


def _hash_uniform(gid: np.ndarray, seed: int, stream: int) -> np.ndarray:
    """Counter-based uniform [0, 1) per global node id (splitmix64 of (seed, stream, gid)), so any
    window of a lattice regenerates the same node attributes."""
    with np.errstate(over="ignore"):
        z = (gid.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.uint64((seed * 1_000_003 + stream) & 0xFFFFFFFF)
             * np.uint64(0xD1B54A32D192ED03))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


STOCH_BLOCK = 10     # layers per independently generated block of stochastic_window


def stochastic_window(side: int, nz: int, k_lo: int, k_hi: int, seed: int = 0, deg_min: int = 3, deg_max: int = 30,
                      r_min: float = 0.02, r_max: float = 0.04, min_angle_deg: float = 25.0, zipf: float = 1.1,
                      block: int = STOCH_BLOCK) -> Lattice:
    """The layers k in [k_lo, k_hi] of ONE stochastic Voronoi-style lattice on a side x side x nz
    jittered grid (BASELINE.json configs[2]; the multi-GPU spatial blocks of it), with the struts
    among them.  Node attributes -- jitter U(-0.3, 0.3), Zipf target degree on [deg_min, deg_max],
    radius U(r_min, r_max) -- are counter-based functions of the global id
    gid = (k * side + j) * side + i.  Struts: the greedy of stochastic() (descending target, nearest
    neighbours in the 5x5x5 surrounding cells, >= min_angle_deg between struts at a node) runs on
    each block of `block` layers independently, then on each block seam (2 layers either side)
    for the struts crossing it, continuing from the blocks' degrees.  So the lattice is local:
    a window needs only the blocks within 2 layers of it, and two windows agree on every node and
    strut they share.  Nodes ascend in gid, struts in (gid, gid)."""
    k_lo, k_hi = max(0, k_lo), min(nz - 1, k_hi)
    lib = _stoch_lib()
    b_lo, b_hi = max(0, k_lo - 2) // block, min(nz - 1, k_hi + 2) // block
    c_lo, c_hi = b_lo * block, min(nz, (b_hi + 1) * block)          # covered layers [c_lo, c_hi)
    nzc = c_hi - c_lo
    nxy = side * side
    gid = np.arange(c_lo * nxy, c_hi * nxy, dtype=np.int64)
    i, j, k = gid % side, (gid // side) % side, gid // nxy
    xyz = np.ascontiguousarray(np.stack([i, j, k], 1).astype(np.float64))
    for a in range(3):
        xyz[:, a] += 0.6 * _hash_uniform(gid, seed, a) - 0.3
    ks = np.arange(deg_min, deg_max + 1)
    p = 1.0 / (ks - deg_min + 1.0) ** zipf
    cdf = np.cumsum(p / p.sum())
    target = ks[np.minimum(np.searchsorted(cdf, _hash_uniform(gid, seed, 3), side="right"), len(ks) - 1)].astype(np.int32)
    radius = r_min + (r_max - r_min) * _hash_uniform(gid, seed, 4)
    n = len(gid)
    deg = np.zeros(n, np.uint8)
    nbr = np.zeros((n, 31), np.int32)
    cos_lim = float(np.cos(np.deg2rad(min_angle_deg)))
    ends_all = []

    def zone(z0, z1, seam):
        """greedy on global layers [z0, z1) of the covered grid; seam layer or -1"""
        a0, a1 = (z0 - c_lo) * nxy, (z1 - c_lo) * nxy
        t = target[a0:a1]
        order = (np.lexsort((np.arange(a1 - a0), -t)) + a0).astype(np.int64)   # descending target, then gid
        cap = int(t.astype(np.int64).sum() // 2) + 1
        ends = np.zeros((cap, 2), np.int64)
        S = lib.stoch_zone(xyz.ctypes.data, side, side, nzc, z0 - c_lo, z1 - c_lo, target.ctypes.data, order.ctypes.data,
                           cos_lim, (seam - c_lo) if seam >= 0 else -1, deg.ctypes.data, nbr.ctypes.data, cap,
                           ends.ctypes.data)
        if S < 0:
            raise RuntimeError(f"stochastic_window zone generator failed ({S})")
        ends_all.append(ends[:S])

    for b in range(b_lo, b_hi + 1):                          # blocks, each on its own
        zone(b * block, min(nz, (b + 1) * block), -1)
    for b in range(b_lo + 1, b_hi + 1):                      # seams between covered blocks
        s0 = b * block
        zone(max(c_lo, s0 - 2), min(c_hi, s0 + 2), s0)
    ends = np.concatenate(ends_all) if ends_all else np.zeros((0, 2), np.int64)
    keep = (k >= k_lo) & (k <= k_hi)
    newid = -np.ones(n, np.int64)
    newid[keep] = np.arange(int(keep.sum()))
    e = newid[ends]
    e = e[(e >= 0).all(1)]
    lat = _finish(xyz[keep], e, radius[keep], f"stochwin{side}x{side}x{nz}[{k_lo}:{k_hi}]")
    lat.ijk = np.stack([i[keep], j[keep], k[keep]], 1).astype(np.int64)
    lat.gid = gid[keep]
    return lat
