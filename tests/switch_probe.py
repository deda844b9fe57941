"""Helper for tests/test_gpu_switches.py (run in a subprocess, because every
CYR_* A/B switch is read once per process): the codebook paths under the
current environment against the reference golden codebooks.  Prints one JSON
line: rows compared and rows that differ outside the logged near-ties."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import mode_t, projection  # noqa: E402
from paper_2506_00167_b200 import (CodebookEngine, DevicePolicy, ScheduleVector,  # noqa: E402
                                   build_codebook, make_streams, policy_for, substream, tree)
from tests.golden_util import Golden  # noqa: E402


def near_ties(cfg, mode, thr=1e-5):
    m_hat, l = cfg[f"{mode}/m_hat"], cfg.meta["urllc_sc_len"]
    out = set()
    for s in range(m_hat.shape[0]):
        caps = np.tile(cfg["alloc"][s].astype(float), (m_hat.shape[1], 1))
        _, margin = projection.apportion(m_hat[s], caps, np.arange(1, m_hat.shape[1] + 1) * l,
                                         with_margin=True)
        out |= {(s, int(j)) for j in np.flatnonzero(margin < thr)}
    return out


def count(got, cfg, mode):
    want = cfg[f"{mode}/codebook"]
    ties = near_ties(cfg, mode)
    bad = 0
    for s in range(want.shape[0]):
        for j in range(1, want.shape[1]):
            if not np.array_equal(got[s, j], want[s, j]) and (s, j - 1) not in ties:
                bad += 1
    return want.shape[0] * (want.shape[1] - 1), bad


def main():
    golden = Golden.load()
    res = {}
    for name in ("cfg2", "desk", "cfg5"):
        cfg = golden.config(name)
        agent = cfg.agent()
        allocs, eps = cfg["alloc"], cfg["eps"]
        # batch engine (K2 variants + K3), stochastic and deterministic
        pol = DevicePolicy(agent.actor, "fp32")
        eng = CodebookEngine(pol, cfg.cell, max_slots=allocs.shape[0])
        for mode, e in (("sto", eps), ("det", None)):
            books = eng.run(torch.from_numpy(allocs).cuda(),
                            None if e is None else torch.from_numpy(e).cuda())
            eng.check()
            res[f"batch/{name}/{mode}"] = count(books.cpu().numpy(), cfg, mode)
        pol.close()
        # drop-in single slot (resident server or graph path), deterministic
        st = make_streams(0, cfg.cell.num_branches)
        got = np.array([build_codebook(agent, ScheduleVector(a.tolist(), [0] * len(a)), st,
                                       True).columns for a in allocs[:24]])
        res[f"dropin/{name}/det"] = count(np.concatenate([got, cfg["det/codebook"][24:]]), cfg,
                                          "det")
        policy_for(agent).quiesce()
    # Mode T levels (the K3 level mapping switch), cfg1 geometry, fp32
    cfg = golden.config("cfg1")
    from dataclasses import replace
    cell = replace(cfg.cell, minislots=5)
    actor = tree.make_mode_t_actor(cell, (64, 64), substream(11, "mode-t"))
    al = cfg["alloc"][:2].astype(np.int32)
    mcs = np.zeros_like(al)
    ep = cfg["eps"][:2]
    got = tree.build_tree_mode_t(DevicePolicy(actor, "fp32"), cell, torch.from_numpy(al).cuda(),
                                 torch.from_numpy(mcs).cuda(), torch.from_numpy(ep).cuda())
    got = got.cpu().numpy()
    bad = 0
    for s in range(2):
        want, margins = mode_t.mode_t_tree(actor.weights, actor.biases, al[s], mcs[s],
                                           cell.total_scs, cell.urllc_sc_len, 5, ep[s],
                                           details=True)
        diff = (got[s, :, :cell.num_embb] != want).any(axis=1)
        near = min(float(m.min()) for m in margins) < 1e-5
        bad += 0 if near else int(diff.sum())
    res["mode_t/cfg1"] = (int(got.shape[1]) * 2, bad)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
