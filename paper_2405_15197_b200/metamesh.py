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
            vert=B.lmm_buffer(h, B.LMM_BUF_VERT, np.float32, 4),
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

        def slab(buf, key, dtype, cols):
            k, k0 = B.SLAB[key]
            return B.lmm_buffer(h, buf, dtype, cols, k * int(off[0]) + k0 * n, k * d + k0)
        return dict(
            csr_off=np.array([0, d], np.int32),
            node_hdr=B.lmm_buffer(h, B.LMM_BUF_NODE_HDR, np.int32, 4, n, 1),
            vert=slab(B.LMM_BUF_VERT, "v", np.float32, 4),
            arc=slab(B.LMM_BUF_ARC, "a", np.uint32, 12),
            loop_hdr=B.lmm_buffer(h, B.LMM_BUF_LOOP_HDR, np.int32, 2, int(off[0]), d),
            loop=slab(B.LMM_BUF_LOOP_ENT, "l", np.uint32, 4),
            hole_hdr=slab(B.LMM_BUF_HOLE_HDR, "h", np.int32, 2),
            hole_ent=slab(B.LMM_BUF_HOLE_ENT, "he", np.uint32, 2),
        )

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


def _base(off, n, key):
    k, k0 = B.SLAB[key]
    return k * int(off[n]) + k0 * n


def decode_node(bufs: dict, n: int) -> dict:
    """The meta-mesh of node n in the oracle's per-node format."""
    off = bufs["csr_off"]
    hdr = bufs["node_hdr"][n]
    status, d = int(hdr[0]) & 0xFF, int(hdr[0]) >> 8
    nv, na = int(hdr[1]) & 0xFFFF, (int(hdr[1]) >> 16) & 0xFFFF
    nh, nle = int(hdr[2]) & 0xFFFF, (int(hdr[2]) >> 16) & 0xFFFF
    nhe = int(hdr[3])
    vb, ab, lb, hb, heb = (_base(off, n, k) for k in ("v", "a", "l", "h", "he"))
    v = bufs["vert"][vb:vb + nv]
    a = bufs["arc"][ab:ab + na]
    ids = a[:, 0].astype(np.int64)
    a_int = np.stack([ids & 0xFF, (ids >> 8) & 0xFF, (ids >> 16) & 0xFF, ids >> 24], 1).astype(np.int32)
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
        status=status, d=d, nv=nv, na=na, nh=nh,
        v_mask=v[:, 3].copy().view(np.uint32), v_pos32=v[:, :3].copy(),
        a_int=a_int, a_f32=a[:, 1:12].copy().view(np.float32),
        loop_off=loop_off,
        l_int=np.stack([le[:, 0] & 0xFFFF, (le[:, 0] >> 16) & 1], 1).astype(np.int32),
        l_N=(le[:, 0] >> 17).astype(np.int32),
        l_f32=le[:, 1:3].copy().view(np.float32),
        l_cum=(le[:, 3] & 0xFFFFFF).astype(np.int32),
        l_vid=(le[:, 3] >> 24).astype(np.int32),
        hole_off=hole_off,
        h_int=np.stack([he[:, 0] & 0xFFFF, (he[:, 0] >> 16) & 1], 1).astype(np.int32),
    )
