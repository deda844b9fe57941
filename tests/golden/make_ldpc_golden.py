"""Freeze erasure-LDPC vectors from the UNMODIFIED reference (build container
only, decodability model "erasure_ldpc").

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ldpc_golden.py

For codes the reference builds through DecodabilityModel.code_for (every
MCS code rate of DEFAULT_MCS_TABLE, TTI lengths M * n_e of typical
allocations): a SHA-256 of the graph (edge_var, edge_check) and, for a set
of erasure patterns (decode_user's puncture layout, optionally with random
channel erasures), phy.peel_decode's verdict.

Output: tests/golden/ldpc_golden.npz.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from punctsim import phy  # noqa: E402
from punctsim.scheduler import DEFAULT_MCS_TABLE  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ldpc_golden.npz")
M = 7


def main():
    rng = np.random.default_rng(20261018)
    model = phy.DecodabilityModel("erasure_ldpc", code_seed=3)
    out, meta = {}, {}
    case = 0
    for entry in DEFAULT_MCS_TABLE:
        for n_e in (24, 96, 264):
            code = model.code_for(M * n_e, entry.code_rate)
            h = hashlib.sha256()
            h.update(code.edge_var.astype("<i8").tobytes())
            h.update(code.edge_check.astype("<i8").tobytes())
            masks, verdicts = [], []
            for t in range(48):
                per_slot = rng.integers(0, n_e + 1, size=M) if t % 3 else \
                    rng.integers(0, max(1, n_e // 4), size=M)
                erased = np.zeros(code.n, dtype=bool)
                for tau, m in enumerate(per_slot):
                    if m:
                        erased[np.arange(int(m)) * M + tau] = True
                if t % 4 == 1:
                    erased[: M * n_e] |= rng.random(M * n_e) < rng.uniform(0.0, 0.3)
                masks.append(erased)
                verdicts.append(phy.peel_decode(code, erased))
            key = f"c{case}"
            out[key + "/erased"] = np.packbits(np.array(masks), axis=1)
            out[key + "/ok"] = np.array(verdicts)
            meta[key] = dict(n_symbols=M * n_e, code_rate=entry.code_rate, n=code.n, dv=code.dv,
                             dc=code.dc, seed=3, graph_sha256=h.hexdigest())
            case += 1
    out["meta_json"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT, **out)
    ok = np.concatenate([out[f"c{i}/ok"] for i in range(case)])
    print("wrote", OUT, os.path.getsize(OUT), "bytes;", case, "codes,", ok.mean(), "decodable")


if __name__ == "__main__":
    main()
