"""Mode-R arrival tree (north-star tree walk).

Every admissible URLLC arrival pattern of a slot — k_tau in {0..cap} per
mini-slot, tau = 1..M — is a node of a (cap+1)-ary tree.  In the reference's
semantics a pattern applies codebook column k_tau in mini-slot tau
(engine.py:230) and each user's decodability depends on its punctured total
(engine.py:240-241, phy.py:201), so the node state is

    cum[node][e] = sum over the path's mini-slots of codebook[k_tau][e]

with arrivals-so-far = sum of the path digits (derivable from the index).

Layout (shared with K1 and the oracle): per slot, BFS over levels 1..M;
level t has (cap+1)^t nodes; node q of level t has parent q // (cap+1) and
last digit q % (cap+1); records are int16 x Epad (Epad = roundup(E, 8)).
"""

from __future__ import annotations

import numpy as np

from . import _native


def num_nodes(cap: int, minislots: int) -> int:
    return int(_native.lib().cyr_tree_num_nodes(int(cap), int(minislots)))


def state_stride(num_users: int) -> int:
    return int(_native.lib().cyr_tree_state_stride(int(num_users)))


def level_offsets(cap: int, minislots: int) -> list:
    """Node offset of level t (t = 1..M) inside one slot's record array."""
    offs, acc = [], 0
    for t in range(1, minislots + 1):
        offs.append(acc)
        acc += (cap + 1) ** t
    return offs


def node_index(path, cap: int) -> int:
    """Global in-slot index of the node reached by arrival counts ``path``."""
    q = 0
    for k in path:
        if not 0 <= int(k) <= cap:
            raise ValueError("arrival count outside 0..cap")
        q = q * (cap + 1) + int(k)
    return level_offsets(cap, len(path))[-1] + q if path else -1


def check_tree_geometry(cell) -> None:
    """int16 records hold cumulative punctures up to M * N."""
    if cell.minislots * cell.total_scs > 32767:
        raise ValueError("M * N exceeds the int16 node-state range")


def expand_tree(codebooks, cell, out=None, stream=None):
    """codebooks: CUDA int32 (S, cap+1, E) -> node states int16
    (S, nodes, Epad), enqueued on the current stream."""
    import torch
    check_tree_geometry(cell)
    s, cols, e = codebooks.shape
    cap = cols - 1
    nodes = num_nodes(cap, cell.minislots)
    stride = state_stride(e)
    if out is None:
        out = torch.empty((s, nodes, stride), dtype=torch.int16, device=codebooks.device)
    codebooks = codebooks.contiguous()
    _native.check(_native.lib().cyr_tree_expand_device(
        codebooks.data_ptr(), s, e, cap, cell.minislots, out.data_ptr(),
        _native.stream_handle(stream)), "expand_tree")
    return out


def arrivals(cap: int, minislots: int) -> np.ndarray:
    """Arrivals-so-far of every node (BFS order), derived from the digits."""
    out, acc = [], np.zeros(1, dtype=np.int64)
    for _ in range(minislots):
        acc = (acc[:, None] + np.arange(cap + 1)[None, :]).ravel()
        out.append(acc)
    return np.concatenate(out)
