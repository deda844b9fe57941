"""Freeze PF-scheduler vectors from the UNMODIFIED reference (build container
only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_pf_golden.py

C cells x T consecutive TTIs of scheduler.pf_schedule (state carried
between TTIs like run_tti does): rates from the reference's own link model
((1 - erasure) * bits_per_symbol of select_mcs, engine.py:188-202) plus
exact ties and zero rates; per TTI the allocations and the committed
avg_tput.  Output: tests/golden/pf_golden.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from punctsim import phy, scheduler  # noqa: E402
from punctsim.core import CellConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pf_golden.npz")


def main():
    rng = np.random.default_rng(20261018)
    cells, ttis = 96, 6
    out = {}
    for e in (4, 10, 16):
        cell = CellConfig(total_scs=780, num_embb=e, urllc_sc_len=195, minislots=7, rb_size=12)
        rates = np.empty((ttis, cells, e))
        chan = phy.ChannelParams()
        for c in range(cells):
            dist = rng.uniform(10.0, 400.0, size=e)
            for t in range(ttis):
                shadow = rng.normal(0.0, chan.shadowing_std_db, size=e)
                for u in range(e):
                    snr = phy.snr_from_distance(dist[u], chan) + shadow[u]
                    entry = scheduler.select_mcs(snr)
                    q = phy.erasure_prob(snr, entry.snr_req_db)
                    rates[t, c, u] = (1.0 - q) * entry.bits_per_symbol
            if c % 8 == 0:
                rates[:, c, :] = 2.0                     # exact ties: round robin
            if c % 8 == 1:
                rates[:, c, 0] = 0.0                     # a zero-rate user
        beta = np.where(np.arange(cells) % 3 == 0, 0.01, 0.2)
        allocs = np.zeros((ttis, cells, e), dtype=np.int64)
        avgs = np.zeros((ttis + 1, cells, e))
        for c in range(cells):
            st = scheduler.PfState.cold_start(e, beta=float(beta[c]))
            avgs[0, c] = st.avg_tput
            for t in range(ttis):
                sv = scheduler.pf_schedule(st, rates[t, c], [0] * e, cell)
                allocs[t, c] = sv.alloc
                avgs[t + 1, c] = st.avg_tput
        out[f"e{e}/rates"] = rates
        out[f"e{e}/beta"] = beta
        out[f"e{e}/alloc"] = allocs
        out[f"e{e}/avg"] = avgs
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
