"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — Mode-R arrival tree.

No reference function builds a tree.  The oracle is the
composition of what the reference does per slot: for an admitted pattern
k_1..k_tau the applied rows are ``codebook.column(k_t)`` (engine.py:230) and
the per-user punctured total is their sum (engine.py:240-241, phy.py:201).

Layout (shared with the CUDA kernel): BFS over levels tau = 1..M, level tau
holds (cap+1)**tau nodes, node q of level tau has parent q // (cap+1) and
last digit q % (cap+1); the root (tau = 0, all zeros) is not stored.
"""

from __future__ import annotations

import numpy as np


def level_sizes(cap: int, minislots: int) -> list:
    return [(cap + 1) ** t for t in range(1, minislots + 1)]


def num_nodes(cap: int, minislots: int) -> int:
    return sum(level_sizes(cap, minislots))


def node_states(codebook, minislots: int) -> np.ndarray:
    """codebook (cap+1, E) -> cum (nodes, E) int64, BFS order."""
    book = np.asarray(codebook, dtype=np.int64)
    frontier = np.zeros((1, book.shape[1]), dtype=np.int64)
    levels = []
    for _ in range(minislots):
        frontier = (frontier[:, None, :] + book[None, :, :]).reshape(-1, book.shape[1])
        levels.append(frontier)
    return np.concatenate(levels)


def node_arrivals(cap: int, minislots: int) -> np.ndarray:
    """Total packets admitted along each node's path (from its digits)."""
    out = []
    acc = np.zeros(1, dtype=np.int64)
    for _ in range(minislots):
        acc = (acc[:, None] + np.arange(cap + 1)[None, :]).ravel()
        out.append(acc)
    return np.concatenate(out)
