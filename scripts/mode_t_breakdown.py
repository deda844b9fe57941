"""Per-level K2 / K3 time of a Mode-T tree (events around each launch)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import CellConfig, DevicePolicy, _native, substream, tree  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n, e, l, hidden = {"cfg2": (780, 10, 195, (256, 256)),
                   "cfg5": (780, 16, 130, (1024, 1024, 1024))}[cfg]
cell = CellConfig(n, e, l)
pol = DevicePolicy(tree.make_mode_t_actor(cell, hidden, substream(0, "mode-t")), "fp32")
allocs, eps = synthetic_inputs(cell, 1)
al = torch.from_numpy(allocs).cuda()
ep = torch.from_numpy(eps).cuda()
mc = torch.zeros_like(al)
out = tree.build_tree_mode_t(pol, cell, al, mc, ep)  # warm
lib = _native.lib()
cap, m = cell.num_branches, cell.minislots
R = cap + 1
nodes = tree.num_nodes(cap, m)
ws = torch.empty(lib.cyr_tree_mode_t_workspace_bytes(pol.handle, 1, cap, m), dtype=torch.uint8,
                 device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
# time one level at a time by running M=tau trees and differencing
prev = 0.0
for tau in range(1, m + 1):
    c2 = CellConfig(n, e, l, minislots=tau)
    o2 = torch.empty((1, tree.num_nodes(cap, tau), out.shape[2]), dtype=torch.int16, device="cuda")
    for _ in range(2):
        tree.build_tree_mode_t(pol, c2, al, mc, ep, out=o2)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        tree.build_tree_mode_t(pol, c2, al, mc, ep, out=o2)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 3
    cols = R ** (tau - 1) * cap
    print(f"level {tau}: {cols:7d} columns, +{(t - prev) * 1e3:8.1f} us")
    prev = t
