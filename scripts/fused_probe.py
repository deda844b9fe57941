"""Event-timed actor launches of the bf16 tcgen05 paths (no profiler):
Mode-R batches of S slots (cap 4 -> 4S columns), 2x256 actor, cfg2 cell.
CYR_TC_FUSED=0 selects the previous kernels for comparison."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import (AgentHyper, CellConfig, DevicePolicy, _native,  # noqa: E402
                                   make_agent, substream)

cell = CellConfig(780, 10, 195)
agent = make_agent(cell, AgentHyper(actor_hidden=(256, 256)), substream(0, "agent-init"))
pol = DevicePolicy(agent.actor, "bf16_tc")
lib = _native.lib()
for slots in (int(x) for x in (sys.argv[1:] or ["4096", "65536", "524288"])):
    allocs, _ = synthetic_inputs(cell, min(slots, 4096))
    al = torch.from_numpy(np.resize(allocs, (slots, 10)).astype(np.int32)).cuda()
    raw = torch.empty((slots * 4, 20), dtype=torch.float32, device="cuda")
    st = _native.stream_handle()
    for _ in range(3):
        _native.check(lib.cyr_actor_forward_device(pol.handle, al.data_ptr(), slots, 780, 4,
                                                   raw.data_ptr(), st))
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _native.check(lib.cyr_actor_forward_device(pol.handle, al.data_ptr(), slots, 780, 4,
                                                   raw.data_ptr(), st))
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    cols = slots * 4
    flops = 2.0 * cols * (11 * 256 + 256 * 256 + 256 * 20)
    print(f"fused={os.environ.get('CYR_TC_FUSED', '1')} cols={cols}: {ms * 1e3:.1f} us, "
          f"{flops / ms / 1e9:.0f} TFLOP/s ({flops / ms / 1e9 / 1403.5 * 100:.1f}% of 1403.5)")
