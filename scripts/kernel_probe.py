"""Per-kernel device times (CUDA events) for the single-slot and batch paths.

    python scripts/kernel_probe.py [--slots 1 1024] [--reps 200] [--precision fp32]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_cell_agent, synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import CodebookEngine, DevicePolicy, _native  # noqa: E402


def timed(fn, reps):
    st = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    for a, b in evs:
        a.record(st)
        fn()
        b.record(st)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in evs]
    return {"p50_us": float(np.median(t)), "min_us": float(np.min(t))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slots", type=int, nargs="+", default=[1, 1024])
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--precision", default="fp32")
    a = ap.parse_args()
    cell, agent = make_cell_agent()
    allocs, eps = synthetic_inputs(cell, max(a.slots))
    pol = DevicePolicy(agent.actor, a.precision)
    lib = _native.lib()
    out = {}
    for s in a.slots:
        eng = CodebookEngine(pol, cell, max_slots=s, with_tree=True)
        al = torch.from_numpy(allocs[:s]).cuda()
        ep = torch.from_numpy(eps[:s]).cuda()
        st = _native.stream_handle()

        def actor():
            _native.check(lib.cyr_actor_forward_device(pol.handle, al.data_ptr(), s, 780, 4,
                                                       eng.raw.data_ptr(), st))

        def codebook():
            _native.check(lib.cyr_codebook_from_raw_device(
                pol.handle, eng.raw.data_ptr(), al.data_ptr(), ep.data_ptr(), s, 780, 195,
                eng.codebooks.data_ptr(), None, None, None, None, eng.status.data_ptr(), st))

        def tree():
            _native.check(lib.cyr_tree_expand_device(eng.codebooks.data_ptr(), s, 10, 4, 7,
                                                     eng.node_state.data_ptr(), st))
        out[s] = {"actor": timed(actor, a.reps), "codebook": timed(codebook, a.reps),
                  "tree": timed(tree, a.reps)}
        eng.check()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
