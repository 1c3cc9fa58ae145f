"""High-level driver over the C-ABI and the decoder of the device meta-mesh layout.

`MetaMesher` strings the C-ABI calls together (load -> build_metamesh -> triangulate ->
write_triangles).  `decode_node` turns the copied-out slabs of one node into plain
arrays (layouts: DESIGN.md Sec. 5) for parity tests; it does no geometry.
"""
from __future__ import annotations

import numpy as np

from . import binding as B


class MetaMesher:
    def __init__(self, device: int = 0, stream: int | None = None):
        self.h = B.lmm_create(device, stream)

    def close(self):
        if self.h is not None:
            B.lmm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, xyz, ends, r_end):
        B.lmm_load_lattice(self.h, xyz, ends, r_end)
        return self

    def load_lattice(self, lat):
        return self.load(np.ascontiguousarray(lat.xyz, np.float32), np.ascontiguousarray(lat.ends, np.int64),
                         np.ascontiguousarray(lat.r_end, np.float32))

    def build(self):
        B.lmm_build_metamesh(self.h)
        return self

    def stats(self) -> dict:
        return B.lmm_metamesh_stats(self.h)

    def set_emit_mask(self, node_mask=None, strut_mask=None):
        B.lmm_set_emit_mask(self.h, node_mask, strut_mask)
        return self

    def triangulate(self, chord_error: float) -> int:
        return B.lmm_triangulate(self.h, chord_error)

    def write(self, first: int, count: int, out):
        return B.lmm_write_triangles(self.h, first, count, out)

    def triangles(self, first: int = 0, count: int | None = None, n_total: int | None = None) -> np.ndarray:
        """Host copy of triangles as float32 [T, 4, 3] (normal, v1, v2, v3)."""
        if count is None:
            count = n_total - first
        buf = np.zeros(max(count, 1) * B.STL_RECORD, np.uint8)
        if count:
            B.lmm_write_triangles(self.h, first, count, buf)
        return B.stl_records_to_array(buf[: count * B.STL_RECORD])

    def buffers(self) -> dict:
        h = self.h
        return dict(
            csr_off=B.lmm_buffer(h, B.LMM_BUF_CSR_OFF, np.int32),
            csr_ent=B.lmm_buffer(h, B.LMM_BUF_CSR_ENT, np.int32, 2),
            node_hdr=B.lmm_buffer(h, B.LMM_BUF_NODE_HDR, np.int32, 4),
            skey=B.lmm_buffer(h, B.LMM_BUF_SLAB_KEY, np.int32, 2),
            vert=B.lmm_buffer(h, B.LMM_BUF_VERT, np.float32, 4),
            vmask_hi=B.lmm_buffer(h, B.LMM_BUF_VMASK_HI, np.uint32),
            arc=B.lmm_buffer(h, B.LMM_BUF_ARC, np.uint32, 12),
            loop_hdr=B.lmm_buffer(h, B.LMM_BUF_LOOP_HDR, np.int32, 2),
            loop=B.lmm_buffer(h, B.LMM_BUF_LOOP_ENT, np.uint32, 4),
            hole_hdr=B.lmm_buffer(h, B.LMM_BUF_HOLE_HDR, np.int32, 2),
            hole_ent=B.lmm_buffer(h, B.LMM_BUF_HOLE_ENT, np.uint32, 2),
        )

    def node_buffers(self, n: int) -> dict:
        """The slabs of node n only (rows copied by offset), in the layout decode_node
        expects for node index 0 -- for sampled parity checks on lattices too large to
        copy out whole."""
        h = self.h
        off = B.lmm_buffer(h, B.LMM_BUF_CSR_OFF, np.int32, None, n, 2).astype(np.int64)
        d = int(off[1] - off[0])
        key = B.lmm_buffer(h, B.LMM_BUF_SLAB_KEY, np.int32, 2, n, 1)[0].astype(np.int64)
        hdr = B.lmm_buffer(h, B.LMM_BUF_NODE_HDR, np.int32, 4, n, 1)
        N, S = self.stats_sizes()
        S2 = 2 * S
        # a spilled node's slots hold exactly its virtual degree; a regular node's its degree
        cap = _virtual_degree(hdr[0]) if key[1] >= N else d

        def slab(buf, k, dtype, cols):
            kk, k0 = B.SLAB[k]
            return B.lmm_buffer(h, buf, dtype, cols, kk * int(key[0]) + k0 * int(key[1]), kk * cap + k0)
        out = dict(
            csr_off=np.array([0, d], np.int32),
            node_hdr=hdr,
            skey=np.zeros((1, 2), np.int32),
            vert=slab(B.LMM_BUF_VERT, "v", np.float32, 4),
            vmask_hi=np.zeros(2 * cap + 2, np.uint32),
            arc=slab(B.LMM_BUF_ARC, "a", np.uint32, 12),
            loop_hdr=B.lmm_buffer(h, B.LMM_BUF_LOOP_HDR, np.int32, 2, int(off[0]), d),
            loop=slab(B.LMM_BUF_LOOP_ENT, "l", np.uint32, 4),
            hole_hdr=slab(B.LMM_BUF_HOLE_HDR, "h", np.int32, 2),
            hole_ent=slab(B.LMM_BUF_HOLE_ENT, "he", np.uint32, 2),
        )
        if key[1] >= N:      # a spilled node: its mask bits 32..63 from the overflow region
            kk, k0 = B.SLAB["v"]
            out["vmask_hi"] = B.lmm_buffer(h, B.LMM_BUF_VMASK_HI, np.uint32, None,
                                           kk * int(key[0] - S2) + k0 * int(key[1] - N), kk * cap + k0)
        out["skey_global"] = (int(key[0]), int(key[1]), S2, N)
        return out

    def stats_sizes(self):
        """(n_nodes, n_struts) of the loaded lattice."""
        if not hasattr(self, "_sizes"):
            off = B.lmm_buffer(self.h, B.LMM_BUF_CSR_OFF, np.int32)
            self._sizes = (len(off) - 1, int(off[-1]) // 2)
        return self._sizes

    def tri_buffers(self) -> dict:
        h = self.h
        return dict(
            band=B.lmm_buffer(h, B.LMM_BUF_BAND, np.int32, 4),
            strut_off=B.lmm_buffer(h, B.LMM_BUF_STRUT_OFF, np.int64),
            hole_M=B.lmm_buffer(h, B.LMM_BUF_HOLE_M, np.int32),
            hole_off=B.lmm_buffer(h, B.LMM_BUF_HOLE_OFF, np.int64),
            hole_bp=B.lmm_buffer(h, B.LMM_BUF_HOLE_BP, np.float32, 4),
            node_hole0=B.lmm_buffer(h, B.LMM_BUF_NODE_HOLE0, np.int64),
        )


def _virtual_degree(hdr) -> int:
    """The smallest degree whose slab capacities (K d + K0) hold the node's counts."""
    nv, na = int(hdr[1]) & 0xFFFF, (int(hdr[1]) >> 16) & 0xFFFF
    nh, nle = int(hdr[2]) & 0xFFFF, (int(hdr[2]) >> 16) & 0xFFFF
    nhe = int(hdr[3])
    D = 0
    for cnt, k in ((nv, "v"), (na, "a"), (nle, "l"), (nh, "h"), (nhe, "he")):
        kk, k0 = B.SLAB[k]
        D = max(D, -(-(cnt - k0) // kk))
    return D


def decode_node(bufs: dict, n: int) -> dict:
    """The meta-mesh of node n in the oracle's per-node format (slabs at the node's slab key)."""
    off = bufs["csr_off"]
    hdr = bufs["node_hdr"][n]
    status, d = int(hdr[0]) & 0xFF, int(hdr[0]) >> 8
    nv, na = int(hdr[1]) & 0xFFFF, (int(hdr[1]) >> 16) & 0xFFFF
    nh, nle = int(hdr[2]) & 0xFFFF, (int(hdr[2]) >> 16) & 0xFFFF
    nhe = int(hdr[3])
    koff, kn = (int(x) for x in bufs["skey"][n])

    def base(k):
        kk, k0 = B.SLAB[k]
        return kk * koff + k0 * kn
    vb, ab, lb, hb, heb = (base(k) for k in ("v", "a", "l", "h", "he"))
    v = bufs["vert"][vb:vb + nv]
    mask = v[:, 3].copy().view(np.uint32).astype(np.uint64)
    if "skey_global" in bufs:                       # node_buffers(): the slabs were sliced out
        gk, gn, S2, N = bufs["skey_global"]
        spilled = gn >= N
        hi = bufs["vmask_hi"][:nv]
    else:
        S2, N = int(off[-1]), len(off) - 1
        spilled = kn >= N
        kk, k0 = B.SLAB["v"]
        hb0 = vb - (kk * S2 + k0 * N)
        hi = bufs["vmask_hi"][hb0:hb0 + nv] if spilled else None
    if spilled and hi is not None and len(hi):
        mask |= hi.astype(np.uint64) << np.uint64(32)
    a = bufs["arc"][ab:ab + na]
    ids = a[:, 0].astype(np.int64)
    a_int = np.stack([ids & 63, (ids >> 6) & 63, (ids >> 12) & 1023, ids >> 22], 1).astype(np.int32)
    lh = bufs["loop_hdr"][off[n]:off[n] + d]
    loop_off = np.zeros(d + 1, np.int32)
    if d:
        loop_off[:d] = lh[:, 0]
        loop_off[d] = lh[-1, 0] + lh[-1, 1]
    le = bufs["loop"][lb:lb + nle]
    hh = bufs["hole_hdr"][hb:hb + nh]
    hole_off = np.zeros(nh + 1, np.int32)
    if nh:
        hole_off[:nh] = hh[:, 0]
        hole_off[nh] = hh[-1, 0] + hh[-1, 1]
    he = bufs["hole_ent"][heb:heb + nhe]
    return dict(
        status=status, d=d, nv=nv, na=na, nh=nh, spilled=bool(spilled),
        v_mask=mask, v_pos32=v[:, :3].copy(),
        a_int=a_int, a_f32=a[:, 1:12].copy().view(np.float32),
        loop_off=loop_off,
        l_int=np.stack([le[:, 0] & 0xFFFF, (le[:, 0] >> 16) & 1], 1).astype(np.int32),
        l_N=(le[:, 0] >> 17).astype(np.int32),
        l_f32=le[:, 1:3].copy().view(np.float32),
        l_cum=(le[:, 3] & 0x3FFFFF).astype(np.int32),
        l_vid=(le[:, 3] >> 22).astype(np.int32),
        hole_off=hole_off,
        h_int=np.stack([he[:, 0] & 0xFFFF, (he[:, 0] >> 16) & 1], 1).astype(np.int32),
    )
