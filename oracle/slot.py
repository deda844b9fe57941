"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — one slot's puncturing
codebook, restating ``engine.build_codebook`` (engine.py:97-116).

Column 0 is the all-zero vector; column j (1..cap) is the enforced action of
branch j with demand j*L.  The cap branch rows of ONE slot form one coupled
enforcement call (engine.py:108-110), so the bisection iteration count is
shared inside a slot and independent across slots.
"""

from __future__ import annotations

import numpy as np

from . import mlp, projection


def slot_codebook(weights, biases, alloc, total_scs: int, sc_len: int, eps=None,
                  details: bool = False):
    """alloc: (E,) ints; eps: (cap, E) float64 branch noise or None.

    Returns codebook (cap+1, E) int64 and, with ``details``, the
    intermediate arrays (raw logits, a, b, m_hat, nu, iterations, margins).
    """
    alloc = np.asarray(alloc, dtype=np.float64)
    users = alloc.size
    cap = total_scs // sc_len
    raw = mlp.forward(weights, biases, mlp.branch_inputs(alloc, total_scs, cap))
    a = mlp.head(raw, users, None if eps is None else np.asarray(eps, dtype=np.float64).T)
    b = mlp.to_subcarriers(a, alloc)
    demands = np.arange(1, cap + 1, dtype=np.int64) * sc_len
    grants, info = projection.enforce(b.T, np.tile(alloc, (cap, 1)), demands,
                                      with_details=True)
    book = np.zeros((cap + 1, users), dtype=np.int64)
    book[1:] = grants
    if details:
        info.update(raw=raw, a=a, b=np.ascontiguousarray(b.T))
        return book, info
    return book


def batch_codebooks(weights, biases, allocs, total_scs: int, sc_len: int, eps=None,
                    details: bool = False):
    """allocs: (S, E); eps: (S, cap, E) or None -> (S, cap+1, E)."""
    allocs = np.asarray(allocs)
    books, infos = [], []
    for s in range(allocs.shape[0]):
        out = slot_codebook(weights, biases, allocs[s], total_scs, sc_len,
                            None if eps is None else eps[s], details=details)
        if details:
            books.append(out[0])
            infos.append(out[1])
        else:
            books.append(out)
    books = np.stack(books) if books else np.zeros((0,))
    return (books, infos) if details else books
