"""CYR_TRACE=1 phase profile of the lane-mapped K3 (tree_level_kernel): run one
Mode-T tree and print the clock64 cycles per warp of each phase, summed over
the lane-mapped levels.  usage: CYR_TRACE=1 python scripts/k3_phase_probe.py cfg5"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import CellConfig, DevicePolicy, _native, substream, tree  # noqa: E402

GEOMS = {"cfg2": (780, 10, 195, (256, 256), 8), "cfg5": (780, 16, 130, (1024, 1024, 1024), 1)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
n, e, l, hidden, slots = GEOMS[name]
cell = CellConfig(n, e, l)
pol = DevicePolicy(tree.make_mode_t_actor(cell, hidden, substream(0, "mode-t")),
                   "bf16_tc" if name == "cfg5" else "fp32")
allocs, eps = synthetic_inputs(cell, slots)
mcs = np.random.default_rng(0).integers(0, 6, size=allocs.shape).astype(np.int32)
al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
tree.build_tree_mode_t(pol, cell, al, mc, ep)
torch.cuda.synchronize()
buf = (ctypes.c_int64 * 64)()
_native.lib().cyr_debug_trace(buf, 64)
vals = [buf[i] for i in range(36, 64)]
warps = max(vals[8], 1)
names = ["head", "setup", "water level", "threshold", "coupled loop", "finish", "HH", "emit"]
tot = sum(vals[:8])
print(f"{name}: {warps} warps, {tot / warps:.0f} cycles per warp")
for k, nm in enumerate(names):
    print(f"  {nm:13s} {vals[k] / warps:9.0f} cycles/warp  {100 * vals[k] / max(tot, 1):5.1f} %")
rows = max(vals[11], 1)
print(f"  per row: {vals[9] / rows:.2f} fill evaluations, {vals[10] / rows:.2f} Huntington-Hill "
      f"exchange steps (phase-1 rows); coupled-bisection iterations per warp {vals[12] / warps:.1f}")
print(f"  per warp (its slowest lane): {vals[13] / warps:.2f} fill evaluations, "
      f"{vals[14] / warps:.2f} exchange steps")
hist = vals[16:28]
print("  fill evaluations per row (1 .. 11, 12+):", hist)
