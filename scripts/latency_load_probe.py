"""Drop-in latency idle and under a concurrent CodebookStream load (bench.py's
_time_calls / _latency_under_load), one process; run twice with
CYR_SLOT_WSM=1/0 to A/B the slot server's shared-memory weights."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_00167_b200 import DevicePolicy, ScheduleVector, make_streams, policy_for  # noqa

cell, agent = bench.make_cell_agent()
allocs, eps = bench.synthetic_inputs(cell, bench.SLOTS)
scheds = [ScheduleVector(a.tolist(), [0] * 10) for a in allocs]
streams = make_streams(7, cell.num_branches)
dev = torch.device("cuda", 0)
pol = DevicePolicy(agent.actor, "fp32")
out = {"wsm": os.environ.get("CYR_SLOT_WSM", "1")}
out["idle"] = bench._time_calls(agent, scheds, streams, 5000)
policy_for(agent).quiesce()
out["load"] = bench._latency_under_load(agent, cell, scheds, streams, pol, allocs, dev, 2000)
policy_for(agent).quiesce()
keep = ("call_p50", "call_p99", "call_max", "device_p50", "device_p99")
print(json.dumps({k: ({kk: round(v[kk], 1) for kk in keep} if isinstance(v, dict) else v)
                  for k, v in out.items()}))
