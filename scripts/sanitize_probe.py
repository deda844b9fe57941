"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the path at a small config, through the C ABI.

    compute-sanitizer --tool racecheck python scripts/sanitize_probe.py [parts]

parts (comma list, default all): server (resident slot server, drop-in
build_codebook), graph (CYR_SLOT_SERVER=0 path is selected by the env of the
whole process), batch (K2 tiled/osplit + K3 warp/lane + K1 tree + leaf score),
modet (Mode-T levels fp32), tc (bf16 tcgen05 narrow + wide), enforce (multi-CTA
coupled enforcement), sac (critic targets / objective sampling).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import (AgentHyper, CellConfig, CodebookEngine, DevicePolicy,  # noqa
                                   ScheduleVector, build_codebook, enforcer, make_agent,
                                   make_streams, sac, substream, tree)


def main():
    parts = set((sys.argv[1] if len(sys.argv) > 1 else
                 "server,batch,modet,tc,enforce,sac").split(","))
    torch.cuda.init()
    cell = CellConfig(780, 10, 195)
    agent = make_agent(cell, AgentHyper(actor_hidden=(256, 256)), substream(0, "agent-init"))
    allocs, eps = synthetic_inputs(cell, 64)
    if "server" in parts or "graph" in parts:
        st = make_streams(1, cell.num_branches)
        for s in range(6):
            sch = ScheduleVector(allocs[s].tolist(), [0] * 10)
            build_codebook(agent, sch, st)
            build_codebook(agent, sch, st, True)
        agent.actor.biases[-1][:] += 0.25  # in-place change: republish path
        build_codebook(agent, ScheduleVector(allocs[0].tolist(), [0] * 10), st)
        from paper_2506_00167_b200 import policy_for
        policy_for(agent).quiesce()
        print("server ok", flush=True)
    if "batch" in parts:
        pol = DevicePolicy(agent.actor, "fp32")
        for slots in (16, 64):
            eng = CodebookEngine(pol, cell, max_slots=slots, with_tree=True)
            eng.run(torch.from_numpy(allocs[:slots]).cuda(), torch.from_numpy(eps[:slots]).cuda())
            eng.check()
        big_a, big_e = synthetic_inputs(cell, 1200)   # lane-mapped K3 (>= 1184 slots)
        eng = CodebookEngine(pol, cell, max_slots=1200)
        eng.run(torch.from_numpy(big_a).cuda(), torch.from_numpy(big_e).cuda())
        eng.check()
        books = eng.codebooks[:8].clone()
        marg = torch.full((8, 10), 0.3, dtype=torch.float64, device="cuda")
        probs = torch.from_numpy(tree.admitted_count_probs(cell)).cuda()
        tree.score_tree(books, cell, torch.from_numpy(allocs[:8]).cuda(), marg, probs)
        torch.cuda.synchronize()
        print("batch ok", flush=True)
    if "modet" in parts:
        c1 = CellConfig(780, 4, 300, minislots=4)
        actor = tree.make_mode_t_actor(c1, (64, 64), substream(2, "mode-t"))
        a1, e1 = synthetic_inputs(c1, 2)
        mcs = np.zeros_like(a1)
        tree.build_tree_mode_t(DevicePolicy(actor, "fp32"), c1, torch.from_numpy(a1).cuda(),
                               torch.from_numpy(mcs).cuda(), torch.from_numpy(e1).cuda())
        torch.cuda.synchronize()
        print("modet ok", flush=True)
    if "tc" in parts:
        pol = DevicePolicy(agent.actor, "bf16_tc")
        a2, e2 = synthetic_inputs(cell, 300)          # 1200 columns: narrow tcgen05 kernel
        eng = CodebookEngine(pol, cell, max_slots=300)
        eng.run(torch.from_numpy(a2).cuda(), torch.from_numpy(e2).cuda())
        eng.check()
        c5 = CellConfig(780, 16, 130, minislots=2)
        actor = tree.make_mode_t_actor(c5, (1024, 1024, 1024), substream(0, "mode-t"))
        a5, e5 = synthetic_inputs(c5, 1)
        tree.build_tree_mode_t(DevicePolicy(actor, "bf16_tc"), c5, torch.from_numpy(a5).cuda(),
                               torch.from_numpy(np.zeros_like(a5)).cuda(),
                               torch.from_numpy(e5).cuda())
        torch.cuda.synchronize()
        print("tc ok", flush=True)
    if "enforce" in parts:
        rng = np.random.default_rng(3)
        rows = 600
        caps = np.tile(allocs[0].astype(float), (rows, 1))
        b = rng.random((rows, 10)) * caps
        dem = rng.integers(1, 5, size=rows) * 195
        enforcer.enforce_batch(b, caps, dem)
        print("enforce ok", flush=True)
    if "sac" in parts:
        h, m = 24, 7
        k = np.random.default_rng(4).integers(0, 5, size=(h, m))
        arrays = (allocs[:h].astype(float), k, np.zeros((h, m, 10)), np.zeros(h))
        sac.critic_targets(agent, arrays, np.random.default_rng(5))
        sel = k.reshape(-1) > 0
        rows = np.repeat(np.arange(h), m)[sel]
        sac.actor_objective(agent.actor, (agent.critic1, agent.critic2), cell, 0.2,
                            allocs[rows], k.reshape(-1)[sel],
                            np.random.default_rng(6).standard_normal((10, int(sel.sum()))), h * m)
        print("sac ok", flush=True)
    torch.cuda.synchronize()
    print("SANITIZE_OK", flush=True)


if __name__ == "__main__":
    main()
