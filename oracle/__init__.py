"""CPU oracle for the lattice meta-meshing hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / reference
leg may import this package.  The product package `paper_2405_15197_b200` never
imports it, and the two share no code (only `synth/` input generators).

Parity status: every exported function is pinned by tests/test_oracle_pins.py
against values the paper or mathematics fixes.
"""
from .oracle import (Oracle, build_oracle, atan2p, theta0, subdiv_count, eq7, aux_plane,
                     eq9, ORC_STATUS)

__all__ = ["Oracle", "build_oracle", "atan2p", "theta0", "subdiv_count", "eq7", "aux_plane",
           "eq9", "ORC_STATUS"]
