"""Freeze golden vectors from the UNMODIFIED reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ``punctsim`` from /root/reference/pkg/src (read-only) and records,
for every configuration in SURVEY.md §8 plus the reference's own desk cell:

  * the schedules (engine._synthetic_schedule on the "scenario" substream),
  * the branch noise each stochastic build_codebook call consumed,
  * the reference's codebooks (deterministic and stochastic),
  * the exact float64 ``b`` the reference fed to enforce_batch, its raw
    actor logits, and kl_project_batch's m_hat / nu / degenerate flags,
  * a SHA-256 of the actor weights (the weights themselves are regenerated
    on any machine from the seed by paper_2506_00167_b200.policy.make_agent;
    the digest proves they are the reference's),

plus a randomized enforcer corpus (coupled groups of rows with zero caps,
zero/tiny/huge masses, fractional caps and degenerate rows) answered by the
reference's kl_project_batch + apportion_batch.

Output: tests/golden/reference_golden.npz.  /root/reference never travels
to the GPU box; only this file does.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

from punctsim import engine, enforcer, neural, sac  # noqa: E402
from punctsim.core import CellConfig  # noqa: E402
from punctsim.scheduler import DEFAULT_MCS_TABLE  # noqa: E402
from punctsim.seeding import substream  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")

# name: (N, E, L, actor_hidden, final_scale, seed, slots)
CONFIGS = {
    "desk":   (96, 4, 24, (16,), 0.01, 7, 64),
    "cfg1":   (780, 4, 300, (256, 256), 0.01, 0, 64),
    "cfg2":   (780, 10, 195, (256, 256), 0.01, 1, 64),
    "paper":  (780, 10, 300, (128,), 0.01, 2, 64),
    "stress": (780, 10, 195, (256, 256), 1.0, 3, 64),
    "cfg5":   (780, 16, 130, (1024, 1024, 1024), 0.01, 4, 12),
}


def weights_digest(actor) -> str:
    h = hashlib.sha256()
    for w, b in zip(actor.weights, actor.biases):
        h.update(np.ascontiguousarray(w, "<f8").tobytes())
        h.update(np.ascontiguousarray(b, "<f8").tobytes())
    return h.hexdigest()


def config_block(name, spec, out, meta):
    n, e, l, hidden, scale, seed, slots = spec
    cell = CellConfig(total_scs=n, num_embb=e, urllc_sc_len=l, minislots=7, rb_size=12)
    cap = cell.num_branches
    hyper = sac.AgentHyper(actor_hidden=hidden, actor_final_scale=scale)
    agent = sac.make_agent(cell, hyper, substream(seed, "agent-init"))
    scen = substream(seed, "scenario")
    schedules = [engine._synthetic_schedule(cell, DEFAULT_MCS_TABLE, scen) for _ in range(slots)]
    alloc = np.array([s.alloc for s in schedules], dtype=np.int32)
    mcs = np.array([s.mcs for s in schedules], dtype=np.int32)

    # noise: stochastic build_codebook consumes one E-draw per branch per call
    streams = engine.make_streams(seed, cap)
    replay = engine.make_streams(seed, cap)
    eps = np.zeros((slots, cap, e))
    books = {"det": [], "sto": []}
    for s, sched in enumerate(schedules):
        for j in range(1, cap + 1):
            eps[s, j - 1] = replay.branch[j].standard_normal(e)
        books["sto"].append(engine.build_codebook(agent, sched, streams, deterministic=False).columns)
        books["det"].append(engine.build_codebook(agent, sched, streams, deterministic=True).columns)
    block_eps = engine.make_streams(seed, cap)
    for j in range(1, cap + 1):   # (S, E) at once == S sequential draws
        assert np.array_equal(block_eps.branch[j].standard_normal((slots, e)), eps[:, j - 1])

    for mode in ("det", "sto"):
        bs, raws, mh, nus, dgs, grs = [], [], [], [], [], []
        for s, sched in enumerate(schedules):
            a_alloc = np.asarray(sched.alloc, dtype=float)
            x = np.empty((e + 1, cap))
            x[:-1, :] = (a_alloc / n)[:, None]
            x[-1, :] = np.arange(1, cap + 1, dtype=float) / cap
            raw, _ = neural.forward(agent.actor, x)
            mu, log_sigma = neural.split_head(raw, e)
            if mode == "det":
                a = np.tanh(mu)
            else:
                a, _, _ = neural.sample_squashed(mu, log_sigma, eps[s].T)
            b = neural.action_to_scs(a, a_alloc[:, None])
            caps = np.tile(a_alloc, (cap, 1))
            dem = np.arange(1, cap + 1) * l
            m_hat, nu, deg = enforcer.kl_project_batch(b.T, caps, dem.astype(float))
            grants = enforcer.apportion_batch(m_hat, caps, dem)
            assert np.array_equal(grants, enforcer.enforce_batch(b.T, caps, dem))
            assert np.array_equal(grants, np.asarray(books[mode][s][1:]))
            bs.append(np.ascontiguousarray(b.T))
            raws.append(raw)
            mh.append(m_hat)
            nus.append(nu)
            dgs.append(deg)
            grs.append(grants)
        out[f"{name}/{mode}/codebook"] = np.array(books[mode], dtype=np.int32)
        out[f"{name}/{mode}/b"] = np.array(bs)
        out[f"{name}/{mode}/raw"] = np.array(raws)
        out[f"{name}/{mode}/m_hat"] = np.array(mh)
        out[f"{name}/{mode}/nu"] = np.array(nus)
        out[f"{name}/{mode}/degenerate"] = np.array(dgs)
    out[f"{name}/alloc"] = alloc
    out[f"{name}/mcs"] = mcs
    out[f"{name}/eps"] = eps
    meta[name] = dict(total_scs=n, num_embb=e, urllc_sc_len=l, minislots=7,
                      actor_hidden=list(hidden), final_scale=scale, seed=seed,
                      slots=slots, cap=cap, weights_sha256=weights_digest(agent.actor))


def enforcer_corpus(out, groups=400, seed=20261018):
    rng = np.random.default_rng(seed)
    bs, cs, ds, gid = [], [], [], []
    for g in range(groups):
        rows = int(rng.integers(1, 13))
        e = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 9, 10, 12, 15, 16, 17, 24, 31, 32]))
        kind = g % 8
        if kind == 7:   # fractional caps
            caps = rng.random((rows, e)) * 30 * (rng.random((rows, e)) > 0.15)
        else:
            caps = rng.integers(0, 60, size=(rows, e)).astype(float)
            caps[rng.random((rows, e)) < 0.15] = 0.0
        b = rng.random((rows, e)) * 50
        if kind == 1:
            b *= 10.0 ** rng.uniform(-200, 6, size=(rows, e))
        elif kind == 2:
            b[rng.random((rows, e)) < 0.5] = 0.0
        elif kind == 3:
            b[rng.random((rows, e)) < 0.4] = 1e-260
        elif kind == 4:
            b = caps * rng.random()          # already proportional
        elif kind == 5:
            b = np.zeros((rows, e))
            b[:, 0] = 1.0                    # single positive user -> degenerate
        elif kind == 6:
            b = np.round(rng.random((rows, e)) * 4) * 2.5   # many exact ties
        total = np.floor(caps.sum(axis=1))
        dem = np.floor(rng.random(rows) * (total + 1)).astype(np.int64)
        dem = np.minimum(dem, total.astype(np.int64))
        if rows > 1:
            dem[0] = 0
        bs.append(b)
        cs.append(caps)
        ds.append(dem)
        gid.append(np.full(rows, g))
    flat_shape = []
    m_all, nu_all, dg_all, gr_all = [], [], [], []
    for b, caps, dem in zip(bs, cs, ds):
        m_hat, nu, deg = enforcer.kl_project_batch(b, caps, dem.astype(float))
        grants = enforcer.apportion_batch(m_hat, caps, dem)
        m_all.append(m_hat)
        nu_all.append(nu)
        dg_all.append(deg)
        gr_all.append(grants)
        flat_shape.append(b.shape)
    # groups have different E: store padded to 32 columns with a width vector
    width = np.array([s[1] for s in flat_shape], dtype=np.int32)
    rows = np.array([s[0] for s in flat_shape], dtype=np.int32)

    def pad(arrs, dtype):
        total = int(rows.sum())
        buf = np.zeros((total, 32), dtype=dtype)
        r0 = 0
        for a in arrs:
            buf[r0:r0 + a.shape[0], :a.shape[1]] = a
            r0 += a.shape[0]
        return buf
    out["enf/rows"] = rows
    out["enf/width"] = width
    out["enf/b"] = pad(bs, np.float64)
    out["enf/caps"] = pad(cs, np.float64)
    out["enf/demand"] = np.concatenate(ds)
    out["enf/m_hat"] = pad(m_all, np.float64)
    out["enf/nu"] = np.concatenate(nu_all)
    out["enf/degenerate"] = np.concatenate(dg_all)
    out["enf/grants"] = pad(gr_all, np.int64)


def main():
    out, meta = {}, {}
    for name, spec in CONFIGS.items():
        config_block(name, spec, out, meta)
        print("config", name, "done", flush=True)
    enforcer_corpus(out)
    out["meta_json"] = np.array(json.dumps(meta, sort_keys=True))
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
