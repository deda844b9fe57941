"""Freeze SAC critic-target vectors from the UNMODIFIED reference (build
container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_critic_golden.py

For each configuration: an agent from make_agent (weights regenerable from
the seed; SHA-256 digests recorded), a replay-batch-shaped input of H
records (allocations from engine._synthetic_schedule, admitted counts k per
mini-slot, rewards), and the reference's sac.critic_targets(agent, arrays,
rng) output y.  The intermediate values of its sampling block (sac.py:
190-205) are recomputed with the reference's own functions and checked to
reproduce y bit for bit: the branch noise eps, raw logits, the raw SC
demands b, the enforced actions (ONE coupled enforce_batch over all rows),
log pi, and the target-critic values q1 / q2.

Output: tests/golden/critic_golden.npz (travels to the GPU box).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from punctsim import engine, enforcer, neural, sac  # noqa: E402
from punctsim.core import CellConfig  # noqa: E402
from punctsim.scheduler import DEFAULT_MCS_TABLE  # noqa: E402
from punctsim.seeding import substream  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "critic_golden.npz")

# name: (N, E, L, actor_hidden, final_scale, seed, records H)
CONFIGS = {
    "cfg2": (780, 10, 195, (256, 256), 0.01, 21, 256),     # H*(M-1) = 1,536 pairs
    "paper": (780, 10, 300, (128,), 0.01, 22, 64),
    "stress": (780, 10, 195, (256, 256), 1.0, 23, 256),
    "cfg1": (780, 4, 300, (256, 256), 0.01, 24, 40),        # < 256 coupled rows
}


def digest(params) -> str:
    h = hashlib.sha256()
    for w, b in zip(params.weights, params.biases):
        h.update(np.ascontiguousarray(w, "<f8").tobytes())
        h.update(np.ascontiguousarray(b, "<f8").tobytes())
    return h.hexdigest()


def block(name, spec, out, meta):
    n, e, l, hidden, scale, seed, h = spec
    cell = CellConfig(total_scs=n, num_embb=e, urllc_sc_len=l, minislots=7, rb_size=12)
    cap, m = cell.num_branches, cell.minislots
    hyper = sac.AgentHyper(actor_hidden=hidden, actor_final_scale=scale)
    agent = sac.make_agent(cell, hyper, substream(seed, "agent-init"))
    scen = substream(seed, "scenario")
    alloc = np.array([engine._synthetic_schedule(cell, DEFAULT_MCS_TABLE, scen).alloc
                      for _ in range(h)], dtype=float)
    krng = np.random.default_rng(seed)
    k = krng.integers(0, cap + 1, size=(h, m)).astype(np.int64)
    punct = np.zeros((h, m, e))
    reward = krng.normal(0.0, 3.0, size=h)
    arrays = (alloc, k, punct, reward)
    y = sac.critic_targets(agent, arrays, np.random.default_rng(seed + 1000))

    # the sampling block, step by step with the reference's own functions
    rng = np.random.default_rng(seed + 1000)
    pair_h = np.repeat(np.arange(h), m)
    pair_tau = np.tile(np.arange(m), h)
    last = pair_tau == m - 1
    nl_idx = np.flatnonzero(~last)
    next_k = k[pair_h[nl_idx], pair_tau[nl_idx] + 1]
    nl_alloc = alloc[pair_h[nl_idx]]
    pos = np.flatnonzero(next_k > 0)
    x = np.vstack([nl_alloc[pos].T / n, next_k[pos][None, :].astype(float) / cap])
    raw, _ = neural.forward(agent.actor, x)
    mu, log_sigma = neural.split_head(raw, e)
    eps = rng.standard_normal(mu.shape)
    a, lp, _ = neural.sample_squashed(mu, log_sigma, eps)
    b = neural.action_to_scs(a, nl_alloc[pos].T)
    dem = next_k[pos] * l
    m_hat, nu, _ = enforcer.kl_project_batch(b.T, nl_alloc[pos], dem.astype(float))
    grants = enforcer.apportion_batch(m_hat, nl_alloc[pos], dem)
    assert np.array_equal(grants, enforcer.enforce_batch(b.T, nl_alloc[pos], dem))
    actions = np.zeros((nl_idx.size, e))
    actions[pos] = grants
    log_pi = np.zeros(nl_idx.size)
    log_pi[pos] = lp
    x_next = np.vstack([nl_alloc.T / n, next_k[None, :].astype(float) / cap, actions.T / n])
    q1, _ = neural.forward(agent.target1, x_next)
    q2, _ = neural.forward(agent.target2, x_next)
    y2 = np.empty(h * m)
    y2[last] = reward[pair_h[last]]
    y2[nl_idx] = hyper.discount * (np.minimum(q1[0], q2[0]) - hyper.zeta * log_pi)
    assert np.array_equal(y, y2), "step-by-step restatement differs from critic_targets"

    p = f"{name}/"
    out[p + "alloc"] = alloc
    out[p + "k"] = k
    out[p + "reward"] = reward
    out[p + "y"] = y
    out[p + "eps"] = eps                 # (E, npos), the draw critic_targets makes
    out[p + "raw"] = raw
    out[p + "b"] = np.ascontiguousarray(b.T)
    out[p + "m_hat"] = m_hat
    out[p + "nu"] = nu
    out[p + "grants"] = grants
    out[p + "log_pi"] = lp
    out[p + "q1"] = q1[0]
    out[p + "q2"] = q2[0]
    meta[name] = dict(total_scs=n, num_embb=e, urllc_sc_len=l, minislots=m, actor_hidden=list(hidden),
                      final_scale=scale, seed=seed, records=h, rng_seed=seed + 1000,
                      rows=int(pos.size), discount=hyper.discount, zeta=hyper.zeta,
                      actor_sha256=digest(agent.actor), target1_sha256=digest(agent.target1),
                      target2_sha256=digest(agent.target2))


def main():
    out, meta = {}, {}
    for name, spec in CONFIGS.items():
        block(name, spec, out, meta)
        print(name, "rows", meta[name]["rows"])
    out["meta_json"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
