"""CPU, world_size 2 over gloo: the multi-GPU O-DU batch path's host logic.

Each rank computes its contiguous block of cells and one all-gather
assembles the batch (paper_2506_00167_b200/sharding.py).  On CPU the
per-shard compute is the oracle (test infrastructure); the assembled result
must equal the single-process oracle batch and the reference's codebooks.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cells, queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import slot
        from paper_2506_00167_b200 import sharding
        from tests.golden_util import Golden
        cfg = Golden.load().config("cfg2")
        agent = cfg.agent()
        allocs = np.asarray(cfg["alloc"][:cells])
        eps = np.asarray(cfg["eps"][:cells])

        def compute(a, e):
            books = slot.batch_codebooks(agent.actor.weights, agent.actor.biases, a,
                                         cfg.meta["total_scs"], cfg.meta["urllc_sc_len"], e)
            return torch.from_numpy(np.asarray(books, dtype=np.int32).reshape(len(a), -1, a.shape[1]))

        full, local = sharding.build_codebooks_sharded(compute, allocs, eps)
        lo, hi = sharding.shard_bounds(cells, world, rank)
        queue.put((rank, full.numpy(), (lo, hi), local.shape[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cells", [8, 7])
def test_two_rank_shard_and_gather(golden, cells):
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cells, queue)) for r in range(2)]
    for p in procs:
        p.start()
    results = [queue.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = golden.config("cfg2")["sto/codebook"][:cells]
    spans = {}
    for rank, full, span, n_local in results:
        assert np.array_equal(full, expect), f"rank {rank} assembled a different batch"
        assert n_local == span[1] - span[0]
        spans[rank] = span
    assert spans[0][1] == spans[1][0] and spans[1][1] == cells


def _tree_worker(rank, world, port, level, queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import arrival_tree
        from paper_2506_00167_b200 import tree
        from tests.golden_util import Golden
        cfg = Golden.load().config("cfg1")
        cap, m = cfg.cell.num_branches, cfg.meta["minislots"]
        whole = np.stack([arrival_tree.node_states(cfg["sto/codebook"][s], m) for s in range(2)])
        whole = torch.from_numpy(whole.astype(np.int16))
        # this rank holds the replicated levels and its own subtrees only
        mine = torch.full_like(whole, -1)
        top = tree.level_offsets(cap, m)[level - 1] + (cap + 1) ** level
        mine[:, :top] = whole[:, :top]
        first, count = tree.shard_extent(cap, m, level, world, rank)
        for off, n in tree.subtree_ranges(cap, m, level, first, count):
            mine[:, off:off + n] = whole[:, off:off + n]
        full = tree.gather_mode_t_tree(mine, cap, m, level)
        queue.put((rank, bool(torch.equal(full, whole))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,level", [(2, 1), (3, 2)])
def test_mode_t_subtree_gather(world, level):
    """Mode-T subtree shards (tree.shard_extent / subtree_ranges) are
    assembled on every rank by ONE all-gather (tree.gather_mode_t_tree)."""
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tree_worker, args=(r, world, port, level, queue))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [queue.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in results), results


def _summary_worker(rank, world, port, level, queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import arrival_tree, leaf_score
        from paper_2506_00167_b200 import tree
        from tests.golden_util import Golden
        cfg = Golden.load().config("cfg1")
        cap, m, n_total = cfg.cell.num_branches, cfg.meta["minislots"], cfg.meta["total_scs"]
        prob = tree.admitted_count_probs(cfg.cell)
        slots = 2
        first, count = tree.shard_leaf_range(cap, m, level,
                                             *tree.shard_extent(cap, m, level, world, rank))
        exp, bits = [], []
        for s in range(slots):
            leaves = arrival_tree.node_states(cfg["sto/codebook"][s], m)[-(cap + 1) ** m:]
            b, r, g, l = leaf_score.score_leaf_states(leaves[first:first + count],
                                                      cfg["alloc"][s], np.full(4, 0.3), prob, m,
                                                      n_total, first)
            exp.append([r, g, l])
            bits.append(b)
        whole, leaves_ok, sent = tree.gather_leaf_summary(
            torch.tensor(exp, dtype=torch.float64), torch.tensor(np.stack(bits), dtype=torch.int32),
            n_total)
        queue.put((rank, whole.numpy(), leaves_ok.numpy(), sent))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,level", [(2, 1), (3, 2)])
def test_mode_t_leaf_summary_gather(world, level):
    """shards keep their node records; ONE all-gather of the
    per-leaf decode bitmasks and partial expectations reassembles the whole
    tree's leaf scores (equal to scoring the whole tree at once)."""
    from oracle import arrival_tree, leaf_score
    from paper_2506_00167_b200 import tree
    from tests.golden_util import Golden
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_summary_worker, args=(r, world, port, level, queue))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [queue.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = Golden.load().config("cfg1")
    cap, m = cfg.cell.num_branches, cfg.meta["minislots"]
    prob = tree.admitted_count_probs(cfg.cell)
    for s in range(2):
        leaves = arrival_tree.node_states(cfg["sto/codebook"][s], m)[-(cap + 1) ** m:]
        bits, r, g, l = leaf_score.score_leaf_states(leaves, cfg["alloc"][s], np.full(4, 0.3),
                                                     prob, m, cfg.meta["total_scs"])
        want = leaf_score.score_leaves(cfg["sto/codebook"][s], cfg["alloc"][s], np.full(4, 0.3),
                                       prob, m, cfg.meta["total_scs"])
        assert np.array_equal(bits, want[0])   # states-based == codebook-based scoring
        for rank, whole, ok, sent in results:
            assert np.array_equal(ok[s], bits)
            assert np.allclose(whole[s], [r, g, l], rtol=1e-12, atol=0)
    nodes_bytes = 2 * tree.num_nodes(cap, m) * 4 * 2
    assert all(sent < nodes_bytes for *_, sent in results)
