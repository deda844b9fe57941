"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — Mode-T arrival tree:
the actor evaluated on every node's state (north star).

No reference function exists; the oracle is composed from the reference's
own size-agnostic pieces, each restated in oracle/:
  * actor forward + tanh-Gaussian head  neural.py:66-84, 144-165 (oracle.mlp)
  * SC mapping                          neural.py:181-183
  * one coupled enforcement per node    enforcer.py:201-207 (oracle.projection)
and the Mode-T feature layout of paper_2506_00167_b200/tree.py:
  [n/N (E), k/cap, cum/N (E), mcs/mcs_scale (E), arrivals/(M*cap), (tau-1)/M].
Children: k = 0 keeps the parent's state, k >= 1 adds the node's grant.
"""

from __future__ import annotations

import numpy as np

from . import mlp, projection


def mode_t_tree(weights, biases, alloc, mcs, total_scs: int, sc_len: int, minislots: int,
                eps=None, mcs_scale: float = 5.0, details: bool = False, stop_level=None):
    """alloc, mcs: (E,); eps: (cap, E) or None.  Returns node states (nodes, E)
    in BFS order (levels 1..M) and, with ``details``, per-level margins.
    ``stop_level`` < M stops after that level (the top of the same tree: the
    features still use M)."""
    alloc = np.asarray(alloc, dtype=np.float64)
    users = alloc.size
    cap = total_scs // sc_len
    r = cap + 1
    parents = np.zeros((1, users), dtype=np.int64)
    arrivals = np.zeros(1, dtype=np.int64)
    levels, margins = [], []
    mcs_feat = np.asarray(mcs, dtype=np.float64) / mcs_scale
    for tau in range(1, (stop_level or minislots) + 1):
        npar = parents.shape[0]
        cols = npar * cap
        x = np.empty((3 * users + 3, cols))
        k = np.tile(np.arange(1, cap + 1), npar)
        q = np.repeat(np.arange(npar), cap)
        x[:users] = (alloc / total_scs)[:, None]
        x[users] = k / cap
        x[users + 1:2 * users + 1] = (parents[q].T.astype(np.float64)) / total_scs
        x[2 * users + 1:3 * users + 1] = mcs_feat[:, None]
        x[3 * users + 1] = arrivals[q] / (minislots * cap)
        x[3 * users + 2] = (tau - 1) / minislots
        raw = mlp.forward(weights, biases, x)
        noise = None if eps is None else np.asarray(eps, dtype=np.float64)[k - 1].T
        a = mlp.head(raw, users, noise)
        b = mlp.to_subcarriers(a, alloc).T  # (cols, E)
        children = np.empty((npar, r, users), dtype=np.int64)
        children[:, 0] = parents
        lvl_margin = np.empty((npar, cap))
        for p in range(npar):
            rows = slice(p * cap, (p + 1) * cap)
            grants, info = projection.enforce(b[rows], np.tile(alloc, (cap, 1)),
                                              np.arange(1, cap + 1) * sc_len, with_details=True)
            children[p, 1:] = parents[p] + grants
            lvl_margin[p] = info["margin"]
        parents = children.reshape(-1, users)
        arrivals = (arrivals[:, None] + np.arange(r)[None, :]).ravel()
        levels.append(parents)
        margins.append(lvl_margin)
    states = np.concatenate(levels)
    return (states, margins) if details else states
