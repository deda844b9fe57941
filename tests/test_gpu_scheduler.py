"""GPU parity for SURVEY.md §8(f) row f4: the batched PF scheduler.

cyr_pf_schedule_device against scheduler.pf_schedule fixtures frozen from
the unmodified reference (tests/golden/make_pf_golden.py): allocations and
the committed PfState are bit-identical over consecutive TTIs, for E = 4,
10, 16, with exact rate ties (round robin) and zero-rate users.
"""

import os

import numpy as np
import pytest
import torch

from paper_2506_00167_b200 import CellConfig, scheduler

pytestmark = pytest.mark.gpu

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "pf_golden.npz"))


@pytest.mark.parametrize("e", [4, 10, 16])
def test_pf_batch_bit_exact_over_ttis(e):
    rates, beta, alloc, avg = (Z[f"e{e}/{k}"] for k in ("rates", "beta", "alloc", "avg"))
    cell = CellConfig(780, e, 195)
    for b in np.unique(beta):
        cells = np.flatnonzero(beta == b)
        state = torch.from_numpy(np.ascontiguousarray(avg[0, cells])).cuda()
        for t in range(rates.shape[0]):
            r = torch.from_numpy(np.ascontiguousarray(rates[t, cells])).cuda()
            got = scheduler.pf_schedule_batch(state, r, cell, float(b)).cpu().numpy()
            assert np.array_equal(got, alloc[t, cells]), (e, b, t)
            assert np.array_equal(state.cpu().numpy(), avg[t + 1, cells]), (e, b, t)


def test_pf_drop_in_single_cell():
    rates, beta, alloc, avg = (Z[f"e10/{k}"] for k in ("rates", "beta", "alloc", "avg"))
    cell = CellConfig(780, 10, 195)
    st = scheduler.PfState.cold_start(10, beta=float(beta[5]))
    for t in range(rates.shape[0]):
        sv = scheduler.pf_schedule(st, rates[t, 5], list(range(10)), cell)
        assert list(sv.alloc) == list(alloc[t, 5]) and np.array_equal(st.avg_tput, avg[t + 1, 5])
    with pytest.raises(ValueError):
        scheduler.pf_schedule(st, -rates[0, 5], [0] * 10, cell)
    with pytest.raises(ValueError):
        scheduler.pf_schedule(st, rates[0, 5][:4], [0] * 10, cell)
