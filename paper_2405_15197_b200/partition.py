"""Spatial partitioning of a lattice across GPUs (host logic of the multi-GPU path).

Rank r owns the nodes whose integer z index lies in its slab [lo_r, hi_r) (the last rank
also owns z = top).  Its local lattice is the slab plus a halo of `halo` z-layers on each
side (positions and radii only): the 1-ring halo nodes then have complete neighbourhoods,
so every rank computes their meta-mesh itself (bit-identically to their owner, because a
node's meta-mesh depends only on its neighbourhood and the shared global strut order) --
the band of a strut crossing the slab boundary needs no exchanged loop data.  A strut is
emitted by the owner of its lower-id endpoint, a node's hole fans by the node's owner.
An all-gather of the per-rank triangle counts (NCCL) fixes each rank's global output offset.
DESIGN.md Sec. 11.
"""
from __future__ import annotations

import numpy as np


def slab(rank: int, world: int, k_top: int):
    """[lo, hi) of z indices owned by `rank` among 0..k_top (hi = k_top + 1 for the last rank)."""
    lo = rank * (k_top + 1) // world
    hi = (rank + 1) * (k_top + 1) // world
    return lo, hi


def window(rank: int, world: int, k_top: int, halo: int = 2):
    """Inclusive z range [k_lo, k_hi] of rank's local lattice (slab + halo layers).  The halo is
    twice the z reach of a strut: 2 layers for the octet/BCC windows (struts span one layer),
    4 for the stochastic lattice (struts span up to two)."""
    lo, hi = slab(rank, world, k_top)
    return max(0, lo - halo), min(k_top, hi - 1 + halo)


def emit_masks(k: np.ndarray, ends: np.ndarray, rank: int, world: int, k_top: int):
    """uint8 node mask (owned nodes) and strut mask (struts whose lower-id endpoint is
    owned) of a local lattice whose node z indices are `k`."""
    lo, hi = slab(rank, world, k_top)
    owned = (k >= lo) & (k < hi)
    node_mask = owned.astype(np.uint8)
    strut_mask = owned[ends[:, 0]].astype(np.uint8)
    return node_mask, strut_mask


def global_offsets(counts) -> list[int]:
    """Exclusive prefix of the per-rank triangle counts (the all-gathered vector)."""
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += int(c)
    return out
