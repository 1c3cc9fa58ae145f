"""B200-native lattice meta-meshing and triangulation (Zou & Gao, arXiv 2405.15197).

The hot path lives in liblmm.so (hand-written sm_100a CUDA behind the C-ABI of
include/lmm.h); this package is its thin binding plus the meta-mesh decoder used by the
tests and the benchmark.  See DESIGN.md.
"""
from .binding import (LmmError, LMM_DEVICE, LMM_HOST, lmm_build_metamesh, lmm_buffer, lmm_create, lmm_destroy,
                      lmm_kernel_times, lmm_load_lattice, lmm_metamesh_stats, lmm_reset_kernel_times, lmm_set_emit_mask, lmm_sync,
                      lmm_timing, lmm_triangulate, lmm_write_triangles, load_library, stl_records_to_array)
from .metamesh import MetaMesher, decode_node

__all__ = ["LmmError", "LMM_DEVICE", "LMM_HOST", "MetaMesher", "decode_node", "lmm_build_metamesh", "lmm_buffer",
           "lmm_create", "lmm_destroy", "lmm_kernel_times", "lmm_load_lattice", "lmm_metamesh_stats",
           "lmm_reset_kernel_times", "lmm_set_emit_mask", "lmm_sync", "lmm_timing", "lmm_triangulate", "lmm_write_triangles",
           "load_library", "stl_records_to_array"]
