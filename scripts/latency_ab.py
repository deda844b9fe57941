"""Idle drop-in latency (bench _time_calls, 5000 cfg2 stochastic slots) under
the current environment (e.g. CYR_ACTOR_CLUSTER)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_00167_b200 import ScheduleVector, make_streams, policy_for  # noqa: E402

cell, agent = bench.make_cell_agent()
allocs, _ = bench.synthetic_inputs(cell, 256)
scheds = [ScheduleVector(a.tolist(), [0] * 10) for a in allocs]
r = bench._time_calls(agent, scheds, make_streams(7, 4), 5000)
policy_for(agent).quiesce()
print(os.environ.get("CYR_ACTOR_CLUSTER", "8"), json.dumps({k: round(v, 2) for k, v in r.items()
                                                           if k != "slots"}))
