"""Seeded synthetic lattice generators shared by the oracle tests and the CUDA path.

This package holds NO meta-meshing arithmetic: it only produces node positions,
strut index pairs and per-end radii (the inputs of the paper's problem statement,
PAPER.md Sec. 4.3.1 "a strut S_i is defined by its two end vertices v_i^0, v_i^1
and the corresponding radii r_i^0, r_i^1").  Both `oracle/` and the product
package may import it; it imports neither.
"""
from .lattices import (Lattice, bcc, octet, octet_window, cubic, star, single_strut, chain,
                       jitter, graded_radii, voronoi_like, bcc_slab, bcc_window, stochastic, stochastic_window)

__all__ = ["Lattice", "bcc", "octet", "octet_window", "cubic", "star", "single_strut", "chain",
           "jitter", "graded_radii", "voronoi_like", "bcc_slab", "bcc_window", "stochastic", "stochastic_window"]
