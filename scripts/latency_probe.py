"""Drop-in single-slot path, for ncu launch lists (cfg2 geometry, fp32).

    python scripts/latency_probe.py [--calls 30] [--tree]
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_cell_agent, synthetic_inputs  # noqa: E402
from paper_2506_00167_b200 import (ScheduleVector, build_codebook, make_streams,  # noqa: E402
                                   set_weight_sync)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=30)
    a = ap.parse_args()
    cell, agent = make_cell_agent()
    allocs, _ = synthetic_inputs(cell, a.calls)
    set_weight_sync("manual")
    streams = make_streams(3, cell.num_branches)
    import time
    host, dev, wall = [], [], []
    scheds = [ScheduleVector(allocs[s], [0] * 10) for s in range(a.calls)]
    for s in range(a.calls):
        t0 = time.perf_counter_ns()
        cb = build_codebook(agent, scheds[s], streams)
        wall.append((time.perf_counter_ns() - t0) / 1e3)
        host.append(cb.gen_ns / 1e3)
        dev.append(cb.device_ns / 1e3)
    print(f"call p50 {np.median(wall):.1f} us p99 {np.percentile(wall, 99):.1f}, "
          f"gen_ns p50 {np.median(host):.1f} us, device p50 {np.median(dev):.1f} us")
    if os.environ.get("CYR_TRACE") == "1":
        import ctypes
        from paper_2506_00167_b200 import _native
        buf = (ctypes.c_int64 * 64)()
        _native.lib().cyr_debug_trace(buf, 64)
        t = list(buf)
        print(f"  SM clock during the kernel: {(t[32 + 15] - t[32]) / max(1, t[15] - t[0]) * 1e3:.0f} MHz")
        names = {0: "start", 1: "input+cluster.sync", 2: "layer1", 3: "layer2", 4: "layer3",
                 8: "k3 head", 9: "kl_setup", 10: "threshold", 11: "phase1 barrier",
                 12: "coupled loop", 13: "finish", 14: "HH", 15: "cb_host written"}
        h = t[48:53]
        if h[0]:
            print("  host: inline copy->SetParams %.2f us, SetParams %.2f, GraphLaunch %.2f, "
                  "sync wait %.2f" % ((h[1] - h[0]) / 1e3, (h[2] - h[1]) / 1e3,
                                      (h[3] - h[2]) / 1e3, (h[4] - h[3]) / 1e3))
        for cl in (1, 8):
            ns = ctypes.c_int64()
            _native.lib().cyr_selftest_launch(cl, 200, ctypes.byref(ns))
            print(f"  empty kernel launch (cluster {cl}): {ns.value / 1e3:.2f} us event-to-event")
        print("  phase-1 end per row warp (us after start):",
              [round((t[16 + w] - t[0]) / 1e3, 2) for w in range(8) if t[16 + w]])
        print("  HH steps per row:", t[40:48], " coupled iterations per row:", t[56:64])
        for l in range(3):
            if t[24 + 2 * l]:
                print(f"  layer {l + 1}: FMA done at {(t[24 + 2 * l] - t[0]) / 1e3:.2f}, "
                      f"exchange done at {(t[25 + 2 * l] - t[0]) / 1e3:.2f}")
        prev = t[0]
        for k in sorted(names):
            if t[k]:
                print(f"  {names[k]:>20s}: +{(t[k] - prev) / 1e3:7.2f} us  (at {(t[k] - t[0]) / 1e3:7.2f})")
                prev = t[k]


if __name__ == "__main__":
    main()
