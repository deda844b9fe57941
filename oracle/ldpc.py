"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — restatement of the
reference's peeling decoder, phy.peel_decode (phy.py:125-143): in rounds,
every check with exactly one erased neighbour recovers it (all such checks
of a round at once); success iff nothing stays erased."""

from __future__ import annotations

import numpy as np


def peel_decode(edge_var, edge_check, n_checks: int, erased) -> bool:
    erased = np.array(erased, dtype=bool)
    while True:
        live = erased[edge_var]
        per_check = np.bincount(edge_check[live], minlength=n_checks)
        recover = live & (per_check[edge_check] == 1)
        if not recover.any():
            return not erased.any()
        erased[edge_var[recover]] = False
