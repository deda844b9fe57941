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
last digit q % (cap+1); records are int16 x Epad (Epad = roundup(E, 2), packed: only the algorithmic bytes).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .policy import MlpParams, init_mlp

# engine._synthetic_schedule draws MCS indices from the 6-entry
# DEFAULT_MCS_TABLE (scheduler.py:32-39): Mode-T features use mcs / 5.
DEFAULT_MCS_SCALE = 5.0


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


# ----------------------------------------------------------------- Mode T
# North star: "walks the arrival tree level by level, and runs the SAC actor
# network on each node's state (per-UE allocated and already-punctured
# subcarriers, CQI/MCS, arrivals so far)".  The reference's actor sees only
# [n/N, j/cap] (sac.py:344-346); Mode T extends the input to
#     [n/N (E), k/cap, cum/N (E), mcs/5 (E), arrivals/(M*cap), (tau-1)/M]
# (3E+3) for the decision of mini-slot tau at a parent node with punctured
# totals `cum` and `arrivals` packets so far.  Each parent's cap branch rows
# are one coupled enforcement (a per-node build_codebook), child k's state is
# cum + grant.  A Mode-T actor whose extra 2E+2 input columns are zero is the
# reference actor at every node (bridge_actor): Mode T then reproduces
# Mode R exactly, which pins the Mode-T kernels against reference decisions.

def mode_t_sizes(cell, hidden) -> list:
    e = int(cell.num_embb)
    return [3 * e + 3, *[int(h) for h in hidden], 2 * e]


def make_mode_t_actor(cell, hidden, rng, final_scale: float = 0.01) -> MlpParams:
    """He-normal Mode-T actor (the init of neural.py:50-63 on 3E+3 inputs)."""
    return init_mlp(mode_t_sizes(cell, hidden), rng, final_scale=final_scale)


def bridge_actor(actor) -> MlpParams:
    """Mode-T actor equal to `actor` (a reference actor, inputs E+1) on the
    reference features and blind to the node-state ones (zero columns)."""
    w0 = np.asarray(actor.weights[0], dtype=np.float64)
    e = w0.shape[1] - 1
    padded = np.concatenate([w0, np.zeros((w0.shape[0], 2 * e + 2))], axis=1)
    return MlpParams([padded] + [np.array(w, dtype=np.float64) for w in actor.weights[1:]],
                     [np.array(b, dtype=np.float64) for b in actor.biases])


def build_tree_mode_t(policy, cell, allocs, mcs, eps=None, mcs_scale: float = DEFAULT_MCS_SCALE,
                      out=None, workspace=None, status=None, stream=None, shard=None):
    """Mode-T arrival tree for S slots on the current stream.

    policy: a DevicePolicy of a Mode-T actor; allocs, mcs: CUDA int32 (S, E);
    eps: CUDA float64 (S, cap, E) or None.  Returns node states int16
    (S, nodes, Epad) in the Mode-R layout.  ``shard`` = (level, first,
    count) builds only the subtrees below level-``level`` nodes
    [first, first + count) (plus the replicated levels <= ``level``); other
    records are left untouched (see subtree_ranges).
    """
    import torch
    check_tree_geometry(cell)
    lib = _native.lib()
    s, e = int(allocs.shape[0]), int(allocs.shape[1])
    cap, m = cell.num_branches, cell.minislots
    nodes = num_nodes(cap, m)
    dev = allocs.device
    if out is None:
        out = torch.empty((s, nodes, state_stride(e)), dtype=torch.int16, device=dev)
    if workspace is None:
        nbytes = lib.cyr_tree_mode_t_workspace_bytes(policy.handle, s, cap, m)
        workspace = torch.empty(max(1, nbytes), dtype=torch.uint8, device=dev)
    own_status = status is None
    if own_status:
        status = torch.zeros(1, dtype=torch.int32, device=dev)
    level, first, count = (0, 0, 1) if shard is None else (int(v) for v in shard)
    _native.check(lib.cyr_tree_mode_t_shard_device(
        policy.handle, allocs.data_ptr(), mcs.data_ptr(), None if eps is None else eps.data_ptr(),
        s, cell.total_scs, cell.urllc_sc_len, m, float(mcs_scale), level, first, count,
        out.data_ptr(), workspace.data_ptr(), status.data_ptr(), _native.stream_handle(stream)),
        "mode-T tree")
    if own_status:
        code = int(status.item())
        if code:
            _native.check(code, "mode-T tree")
    return out


# ------------------------------------------------------- Mode-T subtree shards
# below level l the subtrees are independent, so a tree is
# split across ranks by contiguous blocks of level-l nodes (l = 1: by the
# first mini-slot's arrival count, the north star's "first-mini-slot
# branch"; l = 2-3 balance 8 GPUs: 49 / 343 subtrees at cap 6).  Levels
# <= l are cheap and every rank builds them.  In BFS order the nodes of
# level tau below level-l nodes [a, b) are [a*R^(tau-l), b*R^(tau-l)), so a
# shard is one contiguous run per level.

def subtree_ranges(cap: int, minislots: int, level: int, first: int, count: int) -> list:
    """[(node offset, node count)] per level tau > level of the shard's
    records, in the slot's BFS record order."""
    r = cap + 1
    offs = level_offsets(cap, minislots)
    out = []
    for tau in range(level + 1, minislots + 1):
        span = r ** (tau - level)
        out.append((offs[tau - 1] + first * span, count * span))
    return out


def shard_extent(cap: int, minislots: int, level: int, world: int, rank: int) -> tuple:
    """(first, count) of rank's contiguous block of level-``level`` nodes."""
    from .sharding import shard_bounds
    lo, hi = shard_bounds((cap + 1) ** level, world, rank)
    return lo, hi - lo


def pack_shard(states, cap: int, minislots: int, level: int, first: int, count: int, width: int):
    """This rank's records (S, width * sum_tau R^(tau-level), Epad): the
    per-level runs back to back, each padded to ``width`` subtrees."""
    import torch
    r = cap + 1
    runs = subtree_ranges(cap, minislots, level, first, count)
    total = sum(width * r ** (tau - level) for tau in range(level + 1, minislots + 1))
    out = torch.zeros((states.shape[0], total, states.shape[2]), dtype=states.dtype,
                      device=states.device)
    pos = 0
    for (off, n), tau in zip(runs, range(level + 1, minislots + 1)):
        out[:, pos:pos + n] = states[:, off:off + n]
        pos += width * r ** (tau - level)
    return out


def gather_mode_t_tree(states, cap: int, minislots: int, level: int, group=None):
    """Assemble the whole Mode-T tree on every rank with ONE all-gather
    (NCCL over NVLink on GPUs, gloo in the CPU tests).  ``states`` is this
    rank's (S, nodes, Epad) array holding at least its shard's records and
    the replicated levels <= ``level``; returns the full tree."""
    import torch
    import torch.distributed as dist
    from .sharding import max_shard
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    width = max_shard((cap + 1) ** level, world)
    first, count = shard_extent(cap, minislots, level, world, rank)
    # int16 records travel as bytes (neither NCCL nor gloo has an int16 type)
    local = pack_shard(states, cap, minislots, level, first, count, width).contiguous()
    raw = local.view(torch.uint8)
    blocks = torch.empty((world,) + tuple(raw.shape), dtype=torch.uint8, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(blocks, raw, group=group)
    else:
        dist.all_gather(list(blocks.unbind(0)), raw, group=group)
    blocks = blocks.view(local.dtype)
    full = states.clone()
    r = cap + 1
    for src in range(world):
        f, c = shard_extent(cap, minislots, level, world, src)
        pos = 0
        for (off, n), tau in zip(subtree_ranges(cap, minislots, level, f, c),
                                 range(level + 1, minislots + 1)):
            full[:, off:off + n] = blocks[src][:, pos:pos + n]
            pos += width * r ** (tau - level)
    return full


# ------------------------------------------------------------ leaf scoring
# every leaf of the arrival tree is one full
# admitted-count pattern of the slot; the reference's TTI step decodes each
# user from its punctured total (threshold model, phy.py:73-80 via
# decode_user, phy.py:196-198) and scores the TTI (core.py:132-153).  K1
# evaluates that at every leaf while the leaf's state is in registers.

# code rates of scheduler.DEFAULT_MCS_TABLE (scheduler.py:31-38)
MCS_CODE_RATES = (1 / 3, 1 / 2, 1 / 2, 3 / 4, 2 / 3, 3 / 4)


def threshold_margins(mcs, margin=None, code_rates=MCS_CODE_RATES) -> np.ndarray:
    """Per-user puncture budget fraction of DecodabilityModel("threshold"):
    ``margin`` when given, else 1 - code_rate of the user's MCS (phy.py:197)."""
    mcs = np.asarray(mcs, dtype=np.int64)
    if margin is not None:
        if not 0.0 < float(margin) <= 1.0:
            raise ValueError("margin must lie in (0, 1]")
        return np.full(mcs.shape, float(margin))
    return 1.0 - np.asarray(code_rates, dtype=np.float64)[mcs]


def admitted_count_probs(cell, num_urllc: int = 12, per_ue_prob: float = 0.08) -> np.ndarray:
    """[M][cap+1] probability of k admitted packets per mini-slot for the
    reference's Bernoulli arrivals (traffic.py:46-52; TrafficConfig
    defaults) capped at cap with an empty carry-in queue."""
    from math import comb
    cap, m = cell.num_branches, cell.minislots
    pk = [comb(num_urllc, j) * per_ue_prob ** j * (1.0 - per_ue_prob) ** (num_urllc - j)
          for j in range(num_urllc + 1)]
    row = pk[:cap] + [sum(pk[cap:])] if num_urllc >= cap else pk + [0.0] * (cap - num_urllc)
    return np.tile(np.asarray(row[:cap + 1], dtype=np.float64), (m, 1))


def score_tree(codebooks, cell, allocs, margins, prob, out=None, leaf_ok: bool = True,
               stream=None):
    """K1 with the fused leaf epilogue.

    codebooks: CUDA int32 (S, cap+1, E); allocs: CUDA int32 (S, E); margins:
    CUDA float64 (S, E); prob: CUDA float64 (M, cap+1).  Returns (node
    states (S, nodes, Epad) int16, leaf_ok (S, (cap+1)^M) int32 bitmask of
    decoding users or None, expect (S, 3) float64 = E[reward], E[goodput],
    E[lost SCs]).
    """
    import torch
    check_tree_geometry(cell)
    s, cols, e = codebooks.shape
    cap, m = cols - 1, cell.minislots
    dev = codebooks.device
    if out is None:
        out = torch.empty((s, num_nodes(cap, m), state_stride(e)), dtype=torch.int16, device=dev)
    ok = torch.empty((s, (cap + 1) ** m), dtype=torch.int32, device=dev) if leaf_ok else None
    expect = torch.empty((s, 3), dtype=torch.float64, device=dev)
    prob = prob.contiguous()
    if tuple(prob.shape) != (m, cap + 1):
        raise ValueError("prob must be (M, cap+1)")
    _native.check(_native.lib().cyr_tree_score_device(
        codebooks.contiguous().data_ptr(), allocs.contiguous().data_ptr(),
        margins.contiguous().data_ptr(), prob.data_ptr(), s, e, cap, m, cell.total_scs,
        out.data_ptr(), None if ok is None else ok.data_ptr(), expect.data_ptr(),
        _native.stream_handle(stream)), "score tree")
    return out, ok, expect


# -------------------------------------------- Mode-T leaf summaries (§8(e))
# A subtree shard of a Mode-T tree keeps its node records on its GPU; what
# travels is a per-leaf SUMMARY: the decode bitmask of every leaf (4 B
# instead of the Epad*2-byte record chain) and the shard's partial
# expectations.  The expectations are additive over leaves, so the whole
# tree's E[r] / E[goodput] / E[lost] is the (rank-ordered) sum of the
# shards'.

def score_leaf_states(states, cell, allocs, margins, prob, first: int = 0, count=None,
                      leaf_ok: bool = True, stream=None):
    """Threshold decode + reward of leaves [first, first+count) of level M
    from node records (S, nodes, Epad) (cyr_tree_leaf_score_states_device).
    Returns (leaf_ok (S, count) int32 bitmask or None, expect (S, 3) float64
    = E[r], E[goodput SCs], E[lost SCs] over those leaves)."""
    import torch
    s, nodes, _ = states.shape
    cap, m, e = cell.num_branches, cell.minislots, cell.num_embb
    leaves = (cap + 1) ** m
    count = leaves - first if count is None else int(count)
    dev = states.device
    ok = torch.empty((s, count), dtype=torch.int32, device=dev) if leaf_ok else None
    expect = torch.zeros((s, 3), dtype=torch.float64, device=dev)
    prob = prob.contiguous()
    if tuple(prob.shape) != (m, cap + 1):
        raise ValueError("prob must be (M, cap+1)")
    _native.check(_native.lib().cyr_tree_leaf_score_states_device(
        states.data_ptr(), nodes, s, e, cap, m, int(first), count,
        allocs.contiguous().data_ptr(), margins.contiguous().data_ptr(), prob.data_ptr(),
        cell.total_scs, None if ok is None else ok.data_ptr(), expect.data_ptr(),
        _native.stream_handle(stream)), "leaf scoring")
    return ok, expect


def shard_leaf_range(cap: int, minislots: int, level: int, first: int, count: int) -> tuple:
    """(first leaf, leaf count) below level-``level`` nodes [first, first+count)."""
    span = (cap + 1) ** (minislots - level)
    return first * span, count * span


def gather_leaf_summary(expect, leaf_ok, total_scs: int, group=None, with_leaves: bool = True):
    """ONE all-gather of every rank's partial expectations (S, 3) (and, with
    ``with_leaves``, its leaves' decode bitmasks, padded to the widest shard)
    -> (whole-tree expectations (S, 3), leaf bitmasks (S, all leaves) or
    None, bytes this rank sent).  Rank r's leaves are the contiguous block
    of shard r (shard_extent / shard_leaf_range), so the bitmasks assemble by
    concatenation in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    s = expect.shape[0]
    width = 0
    if with_leaves:
        n = torch.tensor([leaf_ok.shape[1]], dtype=torch.int64, device=expect.device)
        sizes = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(sizes, n, group=group)
        sizes = [int(x.item()) for x in sizes]
        width = max(sizes)
    # one buffer: expectations as float64 + bitmasks as int32 pairs viewed as float64
    words = 3 + (width + 1) // 2
    local = torch.zeros((s, words), dtype=torch.float64, device=expect.device)
    local[:, :3] = expect
    if with_leaves:
        bits = torch.zeros((s, 2 * (words - 3)), dtype=torch.int32, device=expect.device)
        bits[:, :leaf_ok.shape[1]] = leaf_ok
        local[:, 3:] = bits.view(torch.float64)
    out = torch.empty((world, s, words), dtype=torch.float64, device=expect.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), local, group=group)
    lost = out[0, :, 2].clone()
    good = out[0, :, 1].clone()
    for r in range(1, world):  # rank order: deterministic
        lost += out[r, :, 2]
        good += out[r, :, 1]
    whole = torch.stack([-lost / total_scs, good, lost], dim=1)
    leaves = None
    if with_leaves:
        blocks = [out[r, :, 3:].contiguous().view(torch.int32)[:, :sizes[r]] for r in range(world)]
        leaves = torch.cat(blocks, dim=1)
    return whole, leaves, int(local.numel() * local.element_size())
