"""Proportional-fair eMBB scheduler on the GPU.

The codebook path's input s(t) — each eMBB user's SC allocation — comes from
``punctsim.scheduler.pf_schedule`` (scheduler.py:79-106), a greedy per-RB
loop.  For an O-DU batch of cells the loop runs on the GPU, one warp per
cell (``cyr_pf_schedule_device``), bit-identical to the reference, so a
batch can go PF -> actor -> enforcement -> arrival tree without leaving the
device.

* ``PfState`` / ``pf_schedule``: the reference's single-cell API (same
  arguments, exceptions and in-place state update);
* ``pf_schedule_batch``: C cells of device tensors, state updated in place.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import ScheduleVector

EWMA_BETA = 0.01   # scheduler.py:16
AVG_FLOOR = 1e-6   # scheduler.py:17


@dataclass
class PfState:
    """Smoothed per-user throughput in SCs/TTI (scheduler.py:66-76)."""

    avg_tput: np.ndarray
    beta: float = EWMA_BETA

    @classmethod
    def cold_start(cls, num_users: int, beta: float = EWMA_BETA) -> "PfState":
        return cls(avg_tput=np.full(num_users, AVG_FLOOR), beta=beta)


def pf_schedule_batch(avg_tput, inst_rate, cell, beta: float = EWMA_BETA, alloc=None,
                      stream=None):
    """C cells at once on the current stream.  avg_tput: CUDA float64 (C, E),
    updated in place (the PfState commit); inst_rate: CUDA float64 (C, E).
    Returns alloc int32 (C, E)."""
    import torch
    if avg_tput.dtype != torch.float64 or inst_rate.dtype != torch.float64:
        raise ValueError("avg_tput and inst_rate must be float64")
    if tuple(avg_tput.shape) != tuple(inst_rate.shape) or avg_tput.dim() != 2:
        raise ValueError("inst_rate length mismatch")
    if not avg_tput.is_contiguous():
        raise ValueError("avg_tput must be contiguous (updated in place)")
    c, e = avg_tput.shape
    if alloc is None:
        alloc = torch.empty((c, e), dtype=torch.int32, device=avg_tput.device)
    status = torch.zeros(1, dtype=torch.int32, device=avg_tput.device)
    _native.check(_native.lib().cyr_pf_schedule_device(
        avg_tput.data_ptr(), inst_rate.contiguous().data_ptr(), c, e, float(beta), cell.num_rbs,
        cell.rb_size, alloc.data_ptr(), status.data_ptr(), _native.stream_handle(stream)),
        "pf_schedule")
    code = int(status.item())
    if code:
        raise ValueError("rates must be non-negative")
    return alloc


def pf_schedule(state: PfState, inst_rate, mcs_indices, cell) -> ScheduleVector:
    """Drop-in for scheduler.pf_schedule (scheduler.py:79-106): grants all
    RBs greedily by rate/avg on the GPU, then commits the EWMA update into
    ``state`` (mutated, like the reference)."""
    import torch
    rates = np.asarray(inst_rate, dtype=float)
    if rates.shape != (cell.num_embb,):
        raise ValueError("inst_rate length mismatch")
    if np.any(rates < 0):
        raise ValueError("rates must be non-negative")
    avg = torch.from_numpy(np.ascontiguousarray(state.avg_tput, dtype=np.float64)[None, :]).cuda()
    rd = torch.from_numpy(rates[None, :].copy()).cuda()
    alloc = pf_schedule_batch(avg, rd, cell, state.beta)[0].cpu().numpy()
    state.avg_tput = avg[0].cpu().numpy()
    if int(alloc.sum()) != cell.total_scs:
        raise AssertionError("PF must grant the whole band")
    return ScheduleVector(alloc=[int(a) for a in alloc], mcs=list(mcs_indices))
