"""Thin ctypes binding of liblmm.so with the C-ABI's names (include/lmm.h).

Argument marshalling only: every step of the path runs in the library's CUDA kernels.
There is no CPU fallback -- if liblmm.so is missing or no sm_100 device is present the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "liblmm.so")

LMM_HOST, LMM_DEVICE = 0, 1
(LMM_BUF_CSR_OFF, LMM_BUF_CSR_ENT, LMM_BUF_NODE_HDR, LMM_BUF_VERT, LMM_BUF_ARC, LMM_BUF_LOOP_HDR,
 LMM_BUF_LOOP_ENT, LMM_BUF_HOLE_HDR, LMM_BUF_HOLE_ENT, LMM_BUF_BAND, LMM_BUF_STRUT_OFF, LMM_BUF_HOLE_M,
 LMM_BUF_HOLE_OFF, LMM_BUF_HOLE_BP, LMM_BUF_NODE_HOLE0, LMM_BUF_SLAB_KEY, LMM_BUF_VMASK_HI) = range(17)
KERNEL_CLASSES = ["csr", "bucket", "metamesh", "count", "scan", "emit"]
STL_RECORD = 50
# slab layout constants (lmm_common.cuh): base = K * off + K0 * n for the node's slab key (off, n)
SLAB = {"v": (2, 2), "a": (3, 2), "l": (6, 4), "h": (2, 2), "he": (3, 2)}


class LmmError(RuntimeError):
    pass


class _Stats(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_struts", C.c_int64), ("n_vertices", C.c_int64),
                ("n_arcs", C.c_int64), ("n_elliptical_arcs", C.c_int64), ("n_circular_arcs", C.c_int64),
                ("n_loop_entries", C.c_int64), ("n_holes", C.c_int64), ("n_error_nodes", C.c_int64),
                ("err_hist", C.c_int64 * 14), ("degree_hist", C.c_int64 * 33),
                ("n_spilled_nodes", C.c_int64)]


_lib = None


def load_library():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LmmError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    P, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    lib.lmm_create.argtypes = [C.POINTER(P), i32, P]
    lib.lmm_destroy.argtypes = [P]
    lib.lmm_destroy.restype = None
    lib.lmm_load_lattice.argtypes = [P, P, i64, P, P, i64, i32]
    lib.lmm_build_metamesh.argtypes = [P]
    lib.lmm_metamesh_stats.argtypes = [P, C.POINTER(_Stats)]
    lib.lmm_triangulate.argtypes = [P, C.c_double, C.POINTER(i64)]
    lib.lmm_set_emit_mask.argtypes = [P, P, P, i32]
    lib.lmm_write_triangles.argtypes = [P, i64, i64, P, i32]
    lib.lmm_sync.argtypes = [P]
    lib.lmm_buffer_size.argtypes = [P, i32, C.POINTER(i64)]
    lib.lmm_copy_buffer.argtypes = [P, i32, i64, i64, P]
    lib.lmm_timing.argtypes = [P, i32]
    lib.lmm_kernel_times.argtypes = [P, C.POINTER(C.c_double), C.POINTER(i64)]
    lib.lmm_reset_kernel_times.argtypes = [P]
    lib.lmm_launch_count.argtypes = [P, C.POINTER(i64)]
    lib.lmm_emit_path.argtypes = [P, C.POINTER(i32)]
    lib.lmm_error_string.argtypes = [i32]
    lib.lmm_error_string.restype = C.c_char_p
    lib.lmm_version.restype = C.c_char_p
    for name in ("lmm_create", "lmm_load_lattice", "lmm_build_metamesh", "lmm_metamesh_stats", "lmm_triangulate",
                 "lmm_write_triangles", "lmm_sync", "lmm_buffer_size", "lmm_copy_buffer", "lmm_timing",
                 "lmm_kernel_times", "lmm_reset_kernel_times", "lmm_launch_count", "lmm_set_emit_mask",
                 "lmm_emit_path"):
        getattr(lib, name).restype = i32
    _lib = lib
    return lib


def _check(rc):
    if rc != 0:
        raise LmmError(f"liblmm: {load_library().lmm_error_string(rc).decode()} ({rc})")


def _ptr(x):
    """(pointer, where) of a numpy array or a torch tensor."""
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data_as(C.c_void_p), LMM_HOST
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(x.data_ptr()), (LMM_DEVICE if x.is_cuda else LMM_HOST)
    raise TypeError(type(x))


def _dtype_name(x) -> str:
    return str(x.dtype).replace("torch.", "")


def _nbytes(x) -> int:
    return int(x.nbytes) if isinstance(x, np.ndarray) else int(x.numel() * x.element_size())


def _require(x, dtype: str, shape_tail: tuple, what: str):
    """Validate dtype and trailing shape before a pointer crosses the C-ABI (a short or
    mistyped buffer would be read out of bounds)."""
    if _dtype_name(x) != dtype:
        raise TypeError(f"{what}: dtype {_dtype_name(x)}, expected {dtype}")
    shp = tuple(x.shape)
    if len(shp) != 1 + len(shape_tail) or shp[1:] != shape_tail:
        raise ValueError(f"{what}: shape {shp}, expected [n, {', '.join(map(str, shape_tail))}]")


def lmm_create(device: int = 0, stream: int | None = None):
    lib = load_library()
    h = C.c_void_p()
    _check(lib.lmm_create(C.byref(h), device, C.c_void_p(stream or 0)))
    return h


def lmm_destroy(h):
    load_library().lmm_destroy(h)


def lmm_load_lattice(h, xyz, ends, r_end):
    """xyz float32 [N,3], ends int64 [S,2], r_end float32 [S,2]: all host (numpy) or all device (torch)."""
    _require(xyz, "float32", (3,), "xyz")
    _require(ends, "int64", (2,), "ends")
    _require(r_end, "float32", (2,), "r_end")
    if r_end.shape[0] != ends.shape[0]:
        raise ValueError(f"r_end has {r_end.shape[0]} rows, ends {ends.shape[0]}")
    (px, wx), (pe, we), (pr, wr) = _ptr(xyz), _ptr(ends), _ptr(r_end)
    if not (wx == we == wr):
        raise ValueError("inputs must all be host or all device")
    _check(load_library().lmm_load_lattice(h, px, int(xyz.shape[0]), pe, pr, int(ends.shape[0]), wx))


def lmm_build_metamesh(h):
    _check(load_library().lmm_build_metamesh(h))


def lmm_metamesh_stats(h) -> dict:
    st = _Stats()
    _check(load_library().lmm_metamesh_stats(h, C.byref(st)))
    out = {f: getattr(st, f) for f, _ in _Stats._fields_ if f not in ("err_hist", "degree_hist")}
    out["err_hist"] = list(st.err_hist)
    out["degree_hist"] = list(st.degree_hist)
    return out


def lmm_set_emit_mask(h, node_mask=None, strut_mask=None):
    """uint8 masks (numpy host or torch device arrays), None = all."""
    for m, what in ((node_mask, "node_mask"), (strut_mask, "strut_mask")):
        if m is not None and _dtype_name(m) != "uint8":
            raise TypeError(f"{what}: dtype {_dtype_name(m)}, expected uint8")
    pn, wn = _ptr(node_mask) if node_mask is not None else (None, None)
    ps, ws = _ptr(strut_mask) if strut_mask is not None else (None, None)
    where = wn if wn is not None else (ws if ws is not None else LMM_HOST)
    _check(load_library().lmm_set_emit_mask(h, pn, ps, where))


def lmm_triangulate(h, chord_error: float) -> int:
    n = C.c_int64()
    _check(load_library().lmm_triangulate(h, float(chord_error), C.byref(n)))
    return int(n.value)


def lmm_write_triangles(h, first: int, count: int, out):
    """out: uint8 buffer of >= 50*count bytes (numpy host array, or torch tensor host/device)."""
    if _nbytes(out) < STL_RECORD * int(count):
        raise ValueError(f"output buffer holds {_nbytes(out)} bytes, {STL_RECORD * int(count)} needed")
    p, w = _ptr(out)
    _check(load_library().lmm_write_triangles(h, int(first), int(count), p, w))
    return out


def lmm_sync(h):
    _check(load_library().lmm_sync(h))


def lmm_buffer(h, buf_id: int, dtype, cols: int | None = None, first: int = 0,
               rows: int | None = None) -> np.ndarray:
    """Host copy of an internal buffer (rows [first, first+rows) when given; a row is
    `cols` elements of `dtype`, or one element)."""
    lib = load_library()
    n = C.c_int64()
    _check(lib.lmm_buffer_size(h, buf_id, C.byref(n)))
    row = np.dtype(dtype).itemsize * (cols or 1)
    total = n.value // row
    rows = total - first if rows is None else rows
    if first < 0 or rows < 0 or first + rows > total:
        raise LmmError(f"buffer {buf_id}: rows [{first}, {first + rows}) outside [0, {total})")
    a = np.zeros(rows * (cols or 1), dtype=dtype)
    if rows:
        _check(lib.lmm_copy_buffer(h, buf_id, first * row, rows * row, a.ctypes.data_as(C.c_void_p)))
    return a.reshape(-1, cols) if cols else a


def lmm_timing(h, enable: bool):
    _check(load_library().lmm_timing(h, int(bool(enable))))


def lmm_kernel_times(h) -> dict:
    ms = (C.c_double * 6)()
    ln = (C.c_int64 * 6)()
    _check(load_library().lmm_kernel_times(h, ms, ln))
    return {k: (ms[i], ln[i]) for i, k in enumerate(KERNEL_CLASSES)}


def lmm_reset_kernel_times(h):
    _check(load_library().lmm_reset_kernel_times(h))


def lmm_emit_path(h) -> int:
    """0: the band region was emitted warp per band (k_emit); 1: by CTA windows (k_emit_span)."""
    v = C.c_int32()
    _check(load_library().lmm_emit_path(h, C.byref(v)))
    return int(v.value)


def lmm_launch_count(h) -> int:
    n = C.c_int64()
    _check(load_library().lmm_launch_count(h, C.byref(n)))
    return int(n.value)


def stl_records_to_array(buf: np.ndarray) -> np.ndarray:
    """Decode packed 50-byte STL facet records into float32 [T, 4, 3] (normal, v1, v2, v3)."""
    raw = np.frombuffer(np.ascontiguousarray(buf).tobytes(), dtype=np.uint8)
    t = raw.size // STL_RECORD
    rec = raw[: t * STL_RECORD].reshape(t, STL_RECORD)
    return rec[:, :48].copy().view(np.float32).reshape(t, 4, 3)
