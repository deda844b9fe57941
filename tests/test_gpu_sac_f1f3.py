"""SURVEY §8(f) rows f1 (actor objective forward) and f3 (agent checkpoint
ingest) on the GPU against fixtures frozen from the UNMODIFIED reference
(tests/golden/make_sac_golden.py).

Bars: objective, q1, q2 and log pi within 1e-4 (fp32 actor) / 1e-9 (fp64)
of max|.|; b (raw SC demands) within the same fraction of the allocation;
codebooks from a reference-written checkpoint bit-exact with the
reference's; critic targets within the critic-target tolerance.
"""

import json
import os

import numpy as np
import pytest
import torch

from paper_2506_00167_b200 import (AgentHyper, CellConfig, ScheduleVector, build_codebook,
                                   make_agent, make_streams, sac, substream)
from paper_2506_00167_b200.device import DeviceMlp
from tests.golden_util import weights_digest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = {"fp32": 1e-4, "fp64": 1e-9}


def _objective_cases():
    z = dict(np.load(os.path.join(GOLDEN, "objective_golden.npz")))
    meta = json.loads(str(z["meta_json"]))
    return z, meta


@pytest.mark.parametrize("name", ["cfg2", "paper", "stress", "cfg1"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_actor_objective_matches_reference(name, precision):
    z, meta = _objective_cases()
    m = meta[name]
    cell = CellConfig(m["total_scs"], m["num_embb"], m["urllc_sc_len"], m["minislots"], 12)
    hyper = AgentHyper(actor_hidden=tuple(m["actor_hidden"]), actor_final_scale=m["final_scale"])
    agent = make_agent(cell, hyper, substream(m["seed"], "agent-init"))
    assert weights_digest(agent.actor) == m["actor_sha256"]
    assert weights_digest(agent.critic1) == m["critic1_sha256"]
    g = lambda k: z[f"{name}/{k}"]  # noqa: E731
    obj, det = sac.actor_objective(agent.actor, (agent.critic1, agent.critic2), cell, m["zeta"],
                                   g("alloc_rows"), g("j_rows"), g("eps"), m["denom"],
                                   precision=precision, with_details=True)
    tol = TOL[precision]
    for key in ("q1", "q2", "log_pi"):
        want = g(key)
        err = np.max(np.abs(det[key] - want)) / max(np.max(np.abs(want)), 1e-300)
        assert err <= tol, f"{key}: {err:.2e}"
    berr = np.max(np.abs(det["b"] - g("b")) / np.maximum(g("alloc_rows"), 1.0))
    assert berr <= tol, f"b: {berr:.2e}"
    want = float(g("objective"))
    scale = max(abs(want), np.max(np.abs(g("q1"))) * g("j_rows").size / m["denom"])
    assert abs(obj - want) <= tol * scale, (obj, want)


def _agent_golden():
    z = dict(np.load(os.path.join(GOLDEN, "agent_golden.npz")))
    return z, json.loads(str(z["meta_json"]))


def _agent_cell_hyper(m):
    cell = CellConfig(m["total_scs"], m["num_embb"], m["urllc_sc_len"], m["minislots"], 12)
    hyper = AgentHyper(actor_hidden=tuple(m["actor_hidden"]),
                       critic_hidden=tuple(m["critic_hidden"]), batch=m["batch"])
    return cell, hyper


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_load_agent_reference_checkpoint(precision):
    """A directory the reference's save_agent wrote (a TRAINED agent, not
    regenerable from a seed) drives the GPU path: codebooks equal the
    reference's own from the same checkpoint; critic targets within tol."""
    z, m = _agent_golden()
    cell, hyper = _agent_cell_hyper(m)
    agent = sac.load_agent(os.path.join(GOLDEN, "agent_ckpt"), cell, hyper, precision=precision)
    assert weights_digest(agent.actor) == m["actor_sha256"]
    assert weights_digest(agent.target1) == m["target1_sha256"]
    assert agent.adam_actor.t == m["adam_t"]
    st = make_streams(m["streams_seed"], cell.num_branches)
    scheds = [ScheduleVector(a.tolist(), [0] * cell.num_embb) for a in z["agent/alloc"]]
    sto = np.array([build_codebook(agent, s, st, precision=precision).columns for s in scheds])
    det = np.array([build_codebook(agent, s, st, True, precision=precision).columns
                    for s in scheds])
    assert np.array_equal(sto, z["agent/sto_codebook"])
    assert np.array_equal(det, z["agent/det_codebook"])
    arrays = (z["agent/batch_alloc"], z["agent/batch_k"],
              np.zeros(z["agent/batch_k"].shape + (cell.num_embb,)), z["agent/batch_reward"])
    y = sac.critic_targets(agent, arrays, np.random.default_rng(m["targets_rng_seed"]),
                           precision=precision)
    want = z["agent/y"]
    assert np.max(np.abs(y - want)) <= TOL[precision] * np.max(np.abs(want))


def test_mlp_from_checkpoint_equals_published():
    z, m = _agent_golden()
    cell, hyper = _agent_cell_hyper(m)
    agent = sac.load_agent(os.path.join(GOLDEN, "agent_ckpt"), cell, hyper, publish=False)
    a = DeviceMlp.from_checkpoint(os.path.join(GOLDEN, "agent_ckpt", "target1.net"), "fp64")
    b = DeviceMlp(agent.target1, "fp64")
    x = torch.rand((300, 2 * cell.num_embb + 1), dtype=torch.float64, device="cuda")
    assert torch.equal(a.forward(x), b.forward(x))
    a.close()
    b.close()
