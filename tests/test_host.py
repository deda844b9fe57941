"""CPU: host-side logic of the drop-in boundary (no kernels launched)."""

import os
import sys

import numpy as np
import pytest

from paper_2506_00167_b200 import engine, sharding, tree
from paper_2506_00167_b200.core import CellConfig, PuncturingVector, ScheduleVector
from paper_2506_00167_b200.policy import (AgentHyper, flatten_actor, load_mlp, make_agent,
                                          save_mlp)
from paper_2506_00167_b200.seeding import substream

REF_SRC = "/root/reference/pkg/src"


def test_cell_and_schedule_validation():
    cell = CellConfig(780, 10, 195)
    assert cell.num_branches == 4 and cell.num_rbs == 65
    with pytest.raises(ValueError):
        CellConfig(780, 10, 780)
    with pytest.raises(ValueError):
        ScheduleVector([1, -1], [0, 0])
    with pytest.raises(ValueError):
        PuncturingVector([3, 2]).check_against(ScheduleVector([2, 2], [0, 0]))


def test_branch_noise_block_equals_sequential_draws():
    a = engine.make_streams(11, 4)
    b = engine.make_streams(11, 4)
    block = engine.draw_branch_noise(a, 4, 10, slots=5)
    for s in range(5):
        for j in range(1, 5):
            assert np.array_equal(block[s, j - 1], b.branch[j].standard_normal(10))


def test_flatten_and_checkpoint_roundtrip(tmp_path):
    cell = CellConfig(96, 4, 24)
    agent = make_agent(cell, AgentHyper(actor_hidden=(16, 8)), substream(5, "agent-init"))
    sizes, blob = flatten_actor(agent.actor)
    assert sizes == [5, 16, 8, 8]
    assert blob.size == 5 * 16 + 16 + 16 * 8 + 8 + 8 * 8 + 8
    path = tmp_path / "actor.net"
    save_mlp(path, agent.actor)
    back = load_mlp(path)
    for w0, w1 in zip(agent.actor.weights, back.weights):
        assert np.array_equal(w0, w1)
    raw = path.read_bytes()
    (tmp_path / "bad.net").write_bytes(raw + b"x")
    with pytest.raises(ValueError):
        load_mlp(tmp_path / "bad.net")


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted")
def test_checkpoint_bytes_match_reference(tmp_path):
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    try:
        from punctsim import neural
    finally:
        sys.path.remove(REF_SRC)
    cell = CellConfig(96, 4, 24)
    agent = make_agent(cell, AgentHyper(actor_hidden=(16,)), substream(5, "agent-init"))
    save_mlp(tmp_path / "ours.net", agent.actor)
    neural.save_mlp(tmp_path / "ref.net", neural.MlpParams(agent.actor.weights, agent.actor.biases))
    assert (tmp_path / "ours.net").read_bytes() == (tmp_path / "ref.net").read_bytes()


def test_tree_index_helpers():
    assert tree.level_offsets(4, 3) == [0, 5, 30]
    assert tree.node_index((2,), 4) == 2
    assert tree.node_index((1, 3), 4) == 5 + 8
    assert tree.num_nodes(4, 7) == 97_655
    arr = tree.arrivals(4, 2)
    assert arr[tree.node_index((1, 3), 4)] == 4
    with pytest.raises(ValueError):
        tree.check_tree_geometry(CellConfig(7800, 10, 195, minislots=7, rb_size=12))


def test_shard_bounds_cover_and_balance():
    for total in (0, 1, 7, 256, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [sharding.shard_bounds(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
            assert max(sizes) <= sharding.max_shard(total, world)


def test_fastpath_noise_is_bit_identical_to_generator_draws():
    from paper_2506_00167_b200 import _fastpath
    a = engine.make_streams(9, 4)
    b = engine.make_streams(9, 4)
    addrs = engine.branch_bitgens(a, 4)
    for _ in range(3):  # consecutive calls advance each branch stream identically
        got = _fastpath.draw(addrs, 10)
        want = [list(b.branch[j].standard_normal(10)) for j in range(1, 5)]
        assert got == want
    assert engine.branch_bitgens(a, 4) is addrs          # cached
    a.branch[2] = b.branch[2]
    assert engine.branch_bitgens(a, 4)[1] != addrs[1]    # re-derived after a swap


def test_agent_checkpoint_roundtrip_matches_reference_bytes(tmp_path):
    """f3 on the host: the reference-written agent directory loads with the
    reference's digests, and save_agent writes byte-identical files."""
    import json
    import os
    from paper_2506_00167_b200 import AgentHyper, CellConfig
    from paper_2506_00167_b200.policy import NET_FILES, load_agent_host, save_agent
    from tests.golden_util import weights_digest
    golden = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    z = dict(np.load(os.path.join(golden, "agent_golden.npz")))
    m = json.loads(str(z["meta_json"]))
    cell = CellConfig(m["total_scs"], m["num_embb"], m["urllc_sc_len"], m["minislots"], 12)
    hyper = AgentHyper(actor_hidden=tuple(m["actor_hidden"]),
                       critic_hidden=tuple(m["critic_hidden"]), batch=m["batch"])
    agent = load_agent_host(os.path.join(golden, "agent_ckpt"), cell, hyper)
    assert weights_digest(agent.actor) == m["actor_sha256"]
    assert agent.adam_actor.t == m["adam_t"]
    save_agent(tmp_path, agent)
    names = [f"{n}.net" for n in NET_FILES] + ["actor.adam", "critic1.adam", "critic2.adam"]
    for name in names:
        with open(os.path.join(golden, "agent_ckpt", name), "rb") as a, \
                open(tmp_path / name, "rb") as b:
            assert a.read() == b.read(), name
    with pytest.raises(ValueError):
        load_agent_host(os.path.join(golden, "agent_ckpt"),
                        CellConfig(780, 4, 195, 7, 12), hyper)
    with pytest.raises(FileNotFoundError):
        load_agent_host(tmp_path / "missing", cell, hyper)
