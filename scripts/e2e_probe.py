"""bench.py's e2e loop alone (CodebookStream, two batches in flight, host wall clock)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_00167_b200 import CodebookStream, DevicePolicy  # noqa: E402

cell, agent = bench.make_cell_agent()
allocs, eps = bench.synthetic_inputs(cell, bench.SLOTS)
pol = DevicePolicy(agent.actor, "fp32")
alloc_h = torch.from_numpy(allocs).pin_memory()
eps_h = torch.from_numpy(eps).pin_memory()
outs = [torch.empty((bench.SLOTS, 5, 10), dtype=torch.int32, pin_memory=True) for _ in range(2)]
serve = CodebookStream(pol, cell, max_slots=bench.SLOTS, with_tree=True)


def run(k):
    pending = None
    for i in range(k):
        h = serve.submit(alloc_h, eps_h, outs[i % 2])
        if pending is not None:
            serve.wait(pending)
        pending = h
    serve.wait(pending)
    serve.drain()
    torch.cuda.synchronize()


run(5)
best = []
for _ in range(3):
    t0 = time.perf_counter()
    run(40)
    best.append((time.perf_counter() - t0) / 40)
ms = min(best) * 1e3
print(f"waves={os.environ.get('CYR_TREE_WAVES', '1')} prio={os.environ.get('CYR_STREAM_MAIN_PRIORITY', '0')}: "
      f"{ms * 1e3:.1f} us per batch, {bench.SLOTS / ms * 1e3 / 1e6:.3f} M codebooks/s")
