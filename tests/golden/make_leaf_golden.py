"""Freeze leaf-scoring vectors from the UNMODIFIED reference (build
container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_leaf_golden.py

For a few golden slots (codebooks from reference_golden.npz, i.e. the
reference's own build_codebook output) every leaf of the arrival tree — one
admitted count per mini-slot — is run through the reference's TTI scoring:
rows = codebook columns (engine.py:230), phy.decode_user with the threshold
DecodabilityModel (margin None -> 1 - code_rate of the user's MCS, and a
fixed margin 0.1), core.compute_reward and core.goodput_scs.

Output: tests/golden/leaf_golden.npz (per-leaf decode bitmask, reward,
goodput per case).
"""

from __future__ import annotations

import itertools
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from punctsim import core, phy  # noqa: E402
from punctsim.scheduler import DEFAULT_MCS_TABLE  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "leaf_golden.npz")
# (config, slot, margin); margin "ldpc": DecodabilityModel("erasure_ldpc",
# code_seed=3) with a clean channel (sc_erasure_prob 0)
CASES = [("cfg1", 0, None), ("cfg1", 5, 0.1), ("paper", 3, None), ("desk", 2, None),
         ("cfg1", 9, None), ("cfg1", 2, "ldpc")]


def main():
    z = np.load(os.path.join(HERE, "reference_golden.npz"))
    meta = json.loads(str(z["meta_json"]))
    out, info = {}, {}
    for i, (name, slot, margin) in enumerate(CASES):
        m = meta[name]
        book = z[f"{name}/sto/codebook"][slot]
        alloc = [int(v) for v in z[f"{name}/alloc"][slot]]
        mcs = [int(v) for v in z[f"{name}/mcs"][slot]]
        sched = core.ScheduleVector(alloc, mcs)
        model = (phy.DecodabilityModel("erasure_ldpc", code_seed=3) if margin == "ldpc"
                 else phy.DecodabilityModel("threshold", margin=margin))
        q = phy.LinkQuality(snr_db=20.0, sc_erasure_prob=0.0)
        rng = np.random.default_rng(0)
        mm, r = m["minislots"], book.shape[0]
        bits, rew, good = [], [], []
        for digits in itertools.product(range(r), repeat=mm):   # BFS leaf order
            rows = [book[k] for k in digits]
            ok = []
            for u in range(len(alloc)):
                per_slot = tuple(int(rows[t][u]) for t in range(mm))
                ok.append(phy.decode_user(model, alloc[u], DEFAULT_MCS_TABLE[mcs[u]], per_slot,
                                          q, mm, rng))
            outcome = core.DecodeOutcome(ok)
            bits.append(sum(1 << u for u, d in enumerate(ok) if d))
            rew.append(core.compute_reward(sched, outcome, m["total_scs"]))
            good.append(core.goodput_scs(sched, outcome))
        out[f"c{i}/bits"] = np.array(bits, dtype=np.int64)
        out[f"c{i}/reward"] = np.array(rew)
        out[f"c{i}/goodput"] = np.array(good, dtype=np.int64)
        info[f"c{i}"] = dict(config=name, slot=slot, margin=margin, leaves=len(bits))
        print(name, slot, margin, len(bits), "leaves")
    out["meta_json"] = np.array(json.dumps(info))
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
