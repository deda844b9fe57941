"""Every CYR_* A/B switch selects a path that is still
parity-correct: the codebooks match the reference golden codebooks (batch
engine, drop-in single slot) and Mode-T trees match the oracle, outside
logged near-ties.  Switches are read once per process, so each combination
runs tests/switch_probe.py in a subprocess."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SWITCHES = [
    {},
    {"CYR_ACTOR_TILED": "0"},          # first-generation per-output batch kernel
    {"CYR_TILED_OSPLIT": "0"},         # tiled kernel without the output split
    {"CYR_TILED16": "0"},              # no 12-warp in-place variant
    {"CYR_ACTOR_GEMM": "0"},           # never the layer-GEMM path
    {"CYR_SLOT_SERVER": "0"},          # per-call fused cluster launch (CUDA graph)
    {"CYR_SLOT_SERVER": "0", "CYR_SLOT_GRAPH": "0"},  # ... without the graph
    {"CYR_ACTOR_CLUSTER": "4"},        # 4-CTA latency cluster
    {"CYR_WARP_LEVEL_ROWS": "0"},      # Mode-T levels always lane-per-row K3
]


@pytest.mark.parametrize("env", SWITCHES, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items())
                         or "default")
def test_switch_paths_match_reference(env):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "switch_probe.py")],
                         env=dict(os.environ, **env), capture_output=True, text=True, cwd=ROOT,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    for what, (rows, bad) in res.items():
        assert rows > 0 and bad == 0, f"{env}: {what}: {bad} of {rows} rows differ"
