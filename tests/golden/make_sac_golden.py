"""Freeze SAC actor-objective vectors and a trained agent checkpoint from
the UNMODIFIED reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_sac_golden.py

1. objective_golden.npz — ``sac.actor_objective_grads`` (sac.py:249-296), the
   forward half: for each configuration an agent from make_agent (weights
   regenerable from the seed, SHA-256 recorded), the (alloc_rows, j_rows,
   eps, denom) block actor_update builds (sac.py:299-317) from a
   replay-batch-shaped input, and the reference's objective.  The
   intermediates (raw logits, log pi, the raw SC demands b, both critics' q)
   are recomputed with the reference's own functions and checked to
   reproduce the objective bit for bit.

2. agent_ckpt/ + agent_golden.npz — a small agent TRAINED by the reference
   (critic_update / actor_update / soft_update on synthetic replay batches,
   so its weights are not regenerable from any seed), written by the
   reference's ``save_agent`` (sac.py:361-371: five PSIMMLP1 networks and
   three PSIMADM1 optimiser states), together with what the reference
   computes with it after ``load_agent`` (sac.py:374-393): stochastic and
   deterministic codebooks of 16 slots (engine.build_codebook) and
   critic_targets on a replay batch.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from punctsim import engine, neural, sac  # noqa: E402
from punctsim.core import CellConfig, ScheduleVector  # noqa: E402
from punctsim.sac import ExperienceRecord  # noqa: E402
from punctsim.scheduler import DEFAULT_MCS_TABLE  # noqa: E402
from punctsim.seeding import substream  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name: (N, E, L, actor_hidden, final_scale, seed, records H)
OBJECTIVE = {
    "cfg2": (780, 10, 195, (256, 256), 0.01, 31, 256),
    "paper": (780, 10, 300, (128,), 0.01, 32, 64),
    "stress": (780, 10, 195, (256, 256), 1.0, 33, 128),
    "cfg1": (780, 4, 300, (256, 256), 0.01, 34, 40),
}


def digest(params) -> str:
    h = hashlib.sha256()
    for w, b in zip(params.weights, params.biases):
        h.update(np.ascontiguousarray(w, "<f8").tobytes())
        h.update(np.ascontiguousarray(b, "<f8").tobytes())
    return h.hexdigest()


def batch_arrays(cell, h, seed):
    scen = substream(seed, "scenario")
    alloc = np.array([engine._synthetic_schedule(cell, DEFAULT_MCS_TABLE, scen).alloc
                      for _ in range(h)], dtype=float)
    krng = np.random.default_rng(seed)
    k = krng.integers(0, cell.num_branches + 1, size=(h, cell.minislots)).astype(np.int64)
    punct = np.zeros((h, cell.minislots, cell.num_embb))
    reward = krng.normal(0.0, 3.0, size=h)
    return alloc, k, punct, reward


def objective_block(name, spec, out, meta):
    n, e, l, hidden, scale, seed, h = spec
    cell = CellConfig(total_scs=n, num_embb=e, urllc_sc_len=l, minislots=7, rb_size=12)
    cap, m = cell.num_branches, cell.minislots
    hyper = sac.AgentHyper(actor_hidden=hidden, actor_final_scale=scale)
    agent = sac.make_agent(cell, hyper, substream(seed, "agent-init"))
    alloc, k, _, _ = batch_arrays(cell, h, seed)
    # the block actor_update builds (sac.py:307-317)
    k_flat = k.reshape(-1)
    sel = np.flatnonzero(k_flat > 0)
    pair_h = np.repeat(np.arange(h), m)
    alloc_rows = alloc[pair_h[sel]]
    j_rows = k_flat[sel]
    eps = np.random.default_rng(seed + 2000).standard_normal((e, sel.size))
    denom = h * m
    objective, _ = sac.actor_objective_grads(agent.actor, (agent.critic1, agent.critic2), cell,
                                             hyper.zeta, alloc_rows, j_rows, eps, denom)
    # the forward, step by step with the reference's own functions (sac.py:265-281)
    x = np.vstack([alloc_rows.T / n, j_rows[None, :].astype(float) / cap])
    raw, _ = neural.forward(agent.actor, x)
    mu, log_sigma = neural.split_head(raw, e)
    a, log_pi, _ = neural.sample_squashed(mu, log_sigma, eps)
    b = neural.action_to_scs(a, alloc_rows.T)
    xc = np.vstack([alloc_rows.T / n, j_rows[None, :].astype(float) / cap, b / n])
    q1, _ = neural.forward(agent.critic1, xc)
    q2, _ = neural.forward(agent.critic2, xc)
    obj2 = float((np.minimum(q1[0], q2[0]) - hyper.zeta * log_pi).sum() / denom)
    assert obj2 == objective, "step-by-step restatement differs from actor_objective_grads"
    p = f"{name}/"
    out[p + "alloc_rows"] = alloc_rows
    out[p + "j_rows"] = j_rows
    out[p + "eps"] = eps
    out[p + "raw"] = raw
    out[p + "log_pi"] = log_pi
    out[p + "b"] = np.ascontiguousarray(b.T)
    out[p + "q1"] = q1[0]
    out[p + "q2"] = q2[0]
    out[p + "objective"] = np.array(objective)
    meta[name] = dict(total_scs=n, num_embb=e, urllc_sc_len=l, minislots=m,
                      actor_hidden=list(hidden), final_scale=scale, seed=seed, rows=int(sel.size),
                      denom=denom, zeta=hyper.zeta, actor_sha256=digest(agent.actor),
                      critic1_sha256=digest(agent.critic1), critic2_sha256=digest(agent.critic2))


def trained_agent(out):
    """A cfg2-geometry agent (actor 128 = the reference default, critics
    64x64) after 12 reference SAC steps, saved with save_agent."""
    cell = CellConfig(total_scs=780, num_embb=10, urllc_sc_len=195, minislots=7, rb_size=12)
    hyper = sac.AgentHyper(actor_hidden=(128,), critic_hidden=(64, 64), batch=32)
    agent = sac.make_agent(cell, hyper, substream(41, "agent-init"))
    rng = np.random.default_rng(41)
    streams = engine.make_streams(41, cell.num_branches)
    scen = substream(41, "scenario")
    buf = []
    for t in range(64):
        sched = engine._synthetic_schedule(cell, DEFAULT_MCS_TABLE, scen)
        book = engine.build_codebook(agent, sched, streams)
        ks = tuple(int(x) for x in rng.integers(0, cell.num_branches + 1, size=7))
        buf.append(ExperienceRecord(alloc=tuple(sched.alloc), k=ks,
                                    punctures=tuple(book.column(x) for x in ks),
                                    reward=float(rng.normal())))
    for step in range(12):
        batch = [buf[i] for i in rng.choice(len(buf), size=32, replace=False)]
        sac.critic_update(agent, batch, streams.target_noise)
        sac.actor_update(agent, batch, streams.actor_noise)
        sac.soft_update(agent)
    ckpt = os.path.join(HERE, "agent_ckpt")
    shutil.rmtree(ckpt, ignore_errors=True)
    sac.save_agent(ckpt, agent)
    loaded = sac.load_agent(ckpt, cell, hyper)
    assert digest(loaded.actor) == digest(agent.actor)
    # what the reference computes with the loaded agent
    scen = substream(42, "scenario")
    scheds = [engine._synthetic_schedule(cell, DEFAULT_MCS_TABLE, scen) for _ in range(16)]
    st = engine.make_streams(42, cell.num_branches)
    sto = np.array([engine.build_codebook(loaded, s, st).columns for s in scheds])
    det = np.array([engine.build_codebook(loaded, s, st, deterministic=True).columns
                    for s in scheds])
    arrays = batch_arrays(cell, 64, 43)
    y = sac.critic_targets(loaded, arrays, np.random.default_rng(44))
    out["agent/alloc"] = np.array([s.alloc for s in scheds], dtype=np.int64)
    out["agent/sto_codebook"] = sto
    out["agent/det_codebook"] = det
    out["agent/y"] = y
    out["agent/batch_alloc"] = arrays[0]
    out["agent/batch_k"] = arrays[1]
    out["agent/batch_reward"] = arrays[3]
    return dict(total_scs=780, num_embb=10, urllc_sc_len=195, minislots=7,
                actor_hidden=[128], critic_hidden=[64, 64], batch=32, streams_seed=42,
                targets_rng_seed=44, actor_sha256=digest(loaded.actor),
                target1_sha256=digest(loaded.target1), adam_t=int(loaded.adam_actor.t))


def main():
    out, meta = {}, {}
    for name, spec in OBJECTIVE.items():
        objective_block(name, spec, out, meta)
        print(name, "rows", meta[name]["rows"])
    out["meta_json"] = np.array(json.dumps(meta))
    path = os.path.join(HERE, "objective_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")
    out = {}
    meta = trained_agent(out)
    out["meta_json"] = np.array(json.dumps(meta))
    path = os.path.join(HERE, "agent_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
