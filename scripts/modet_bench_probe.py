"""Run only bench.py's Mode-T entries (cfg2, cfg3, cfg5, latency) and print them."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_00167_b200 import CellConfig  # noqa: E402

cell = CellConfig(**bench.GEOM)
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what == "all":
    out = bench.mode_t_all(cell)
elif what == "cfg3":
    out = bench.mode_t_cfg3(cell, bench.HIDDEN)
elif what == "latency":
    out = bench.mode_t_latency()
else:
    out = bench.mode_t_run(cell, bench.HIDDEN, 32)
    out.pop("_slot0")
print(json.dumps(out, indent=1))
