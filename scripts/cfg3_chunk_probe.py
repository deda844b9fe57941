"""cfg3 Mode-T (1024 trees, cfg2 geometry, 2x256) with different tree-batch
sizes, bf16 tcgen05: does a bigger batch amortise the small levels?"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_00167_b200 import CellConfig, DevicePolicy, substream, tree  # noqa: E402

cell = CellConfig(780, 10, 195)
actor = tree.make_mode_t_actor(cell, (256, 256), substream(0, "mode-t"))
total = 1024
allocs, eps = bench.synthetic_inputs(cell, total, seed=12)
mcs = np.random.default_rng(12).integers(0, 6, size=allocs.shape).astype(np.int32)
al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
prec = os.environ.get("PREC", "bf16_tc")
pol = DevicePolicy(actor, prec)
for chunk in [int(x) for x in (sys.argv[1:] or ["32", "64", "128"])]:
    buf = tree.build_tree_mode_t(pol, cell, al[:chunk], mc[:chunk], ep[:chunk])
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for c0 in range(0, total, chunk):
            tree.build_tree_mode_t(pol, cell, al[c0:c0 + chunk], mc[c0:c0 + chunk],
                                   ep[c0:c0 + chunk], out=buf)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{prec} chunk {chunk}: {best:.2f} ms for 1024 trees = {total / (best * 1e-3):.0f} trees/s")
    del buf
    torch.cuda.empty_cache()
