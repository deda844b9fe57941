"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — leaf scoring of the
arrival tree, restated from the reference's TTI
step for every admissible arrival pattern:

  * applied rows = codebook columns of the leaf's digits      engine.py:230
  * per-user punctured total = sum over mini-slots            engine.py:240-241
  * threshold decode: n_e <= 0 or m_total <= margin*(M*n_e)   phy.py:73-80, 196-198
  * reward r = sum_e (ok_e - 1) * n_e / N                     core.py:132-146
  * goodput = sum_e ok_e * n_e                                core.py:149-153
  * leaf weight = prod over mini-slots of prob[tau][k_tau] (expectation
    over independent admitted counts; no reference counterpart)
"""

from __future__ import annotations

import numpy as np

from . import arrival_tree


def leaf_states(codebook, minislots: int) -> np.ndarray:
    states = arrival_tree.node_states(codebook, minislots)
    r = np.asarray(codebook).shape[0]
    return states[-r ** minislots:]


def score_leaves(codebook, alloc, margin, prob, minislots: int, total_scs: int):
    """(ok bitmask (leaves,), reward (leaves,), E[r], E[goodput], E[lost])."""
    cum = leaf_states(codebook, minislots).astype(np.int64)
    n = np.asarray(alloc, dtype=np.int64)
    budget = np.asarray(margin, dtype=np.float64) * (minislots * n)
    ok = (n[None, :] <= 0) | (cum <= budget[None, :])
    lost = ((~ok) * np.where(n > 0, n, 0)[None, :]).sum(axis=1)
    reward = -lost / total_scs
    bits = (ok.astype(np.int64) << np.arange(n.size)[None, :]).sum(axis=1)
    r = np.asarray(codebook).shape[0]
    w = np.ones(1)
    for tau in range(minislots):
        w = (w[:, None] * np.asarray(prob)[tau][None, :]).ravel()
    tot = int(np.where(n > 0, n, 0).sum())
    e_lost = float(np.sum(w * lost))
    return bits, reward, -e_lost / total_scs, float(np.sum(w * (tot - lost))), e_lost


def score_leaf_states(leaves, alloc, margin, prob, minislots: int, total_scs: int,
                      first: int = 0):
    """The same scoring from explicit leaf records (Mode-T trees): leaves
    (count, E) cumulative punctures of level-M nodes first .. first+count.
    Returns (ok bits, E[r], E[goodput], E[lost]) over those leaves."""
    cum = np.asarray(leaves, dtype=np.int64)
    n = np.asarray(alloc, dtype=np.int64)
    budget = np.asarray(margin, dtype=np.float64) * (minislots * n)
    ok = (n[None, :] <= 0) | (cum <= budget[None, :])
    lost = ((~ok) * np.where(n > 0, n, 0)[None, :]).sum(axis=1)
    bits = (ok.astype(np.int64) << np.arange(n.size)[None, :]).sum(axis=1)
    prob = np.asarray(prob)
    r = prob.shape[1]
    q = np.arange(first, first + cum.shape[0])
    w = np.ones(cum.shape[0])
    for tau in range(minislots - 1, -1, -1):
        w = w * prob[tau][q % r]
        q = q // r
    tot = int(np.where(n > 0, n, 0).sum())
    e_lost = float(np.sum(w * lost))
    return bits, -e_lost / total_scs, float(np.sum(w * (tot - lost))), e_lost
