"""Leaf scoring on a real cfg5 Mode-T tree (the bench's sharded entry at N=1)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import CellConfig, DevicePolicy, substream, tree  # noqa: E402

cell = CellConfig(780, 16, 130)
actor = tree.make_mode_t_actor(cell, (1024, 1024, 1024), substream(0, "mode-t"))
allocs, eps = synthetic_inputs(cell, 1, seed=11)
mcs = np.random.default_rng(11).integers(0, 6, size=allocs.shape).astype(np.int32)
al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
pol = DevicePolicy(actor, "bf16_tc")
out = tree.build_tree_mode_t(pol, cell, al, mc, ep)
margins = torch.from_numpy(tree.threshold_margins(mcs)).cuda()
prob = torch.from_numpy(tree.admitted_count_probs(cell)).cuda()
torch.cuda.synchronize()
for rep in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    ok, exp = tree.score_leaf_states(out, cell, al, margins, prob)
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: events {a.elapsed_time(b) * 1e3:.0f} us, host launch {1e6 * (t1 - t0):.0f} us, "
          f"sync {1e6 * (t2 - t1):.0f} us, exp {exp.cpu().numpy()}")
