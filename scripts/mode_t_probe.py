"""Mode-T tree timing (CUDA events around the level loop)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import CellConfig, DevicePolicy, substream, tree  # noqa: E402

GEOMS = {"cfg1": (780, 4, 300, (256, 256)), "cfg2": (780, 10, 195, (256, 256)),
         "cfg5": (780, 16, 130, (1024, 1024, 1024))}

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2")
ap.add_argument("--slots", type=int, default=1)
ap.add_argument("--precision", default="fp32", choices=("fp32", "fp64", "bf16_tc"))
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n, e, l, hidden = GEOMS[a.cfg]
cell = CellConfig(n, e, l)
actor = tree.make_mode_t_actor(cell, hidden, substream(0, "mode-t"))
pol = DevicePolicy(actor, a.precision)
allocs, eps = synthetic_inputs(cell, a.slots)
mcs = np.random.default_rng(0).integers(0, 6, size=allocs.shape).astype(np.int32)
al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
out = tree.build_tree_mode_t(pol, cell, al, mc, ep)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    tree.build_tree_mode_t(pol, cell, al, mc, ep, out=out)
    s1.record()
    torch.cuda.synchronize()
    ts.append(s0.elapsed_time(s1))
cap = cell.num_branches
cols = sum((cap + 1) ** t for t in range(cell.minislots)) * cap * a.slots
sizes = tree.mode_t_sizes(cell, hidden)
flops = 2 * cols * sum(i * o for i, o in zip(sizes[:-1], sizes[1:]))
ms = float(np.median(ts))
print(f"{a.cfg} slots={a.slots} {a.precision}: {ms:.2f} ms/tree-batch, actor columns {cols}, "
      f"{flops / 1e9:.1f} GFLOP -> {flops / ms / 1e9:.1f} TFLOP/s over the whole tree")
