"""GPU feasibility enforcer with the reference's batch API.

``kl_project_batch``, ``apportion_batch`` and ``enforce_batch`` take and
return numpy arrays like ``punctsim/enforcer.py:49-207`` and raise the same
exceptions in the same order (shape mismatch / negative input -> ValueError,
demand above capacity -> InfeasibleDemandError), but compute on the GPU
through the C ABI (K3 core):

* one call == one coupled bisection (the stop test spans every bisecting
  row of the call, enforcer.py:90-92), any number of rows (one CTA up to
  256, a two-pass multi-CTA call above);
* results are bit-identical to the reference for identical float64 inputs
  (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._native import InfeasibleDemandError

__all__ = ["InfeasibleDemandError", "kl_project_batch", "apportion_batch", "enforce_batch"]

def _validate_projection(b, caps, demand):
    b = np.ascontiguousarray(b, dtype=np.float64)
    caps = np.ascontiguousarray(caps, dtype=np.float64)
    demand = np.asarray(demand, dtype=np.float64)
    if b.ndim != 2 or b.shape != caps.shape or demand.shape != (b.shape[0],):
        raise ValueError("shape mismatch")
    if (b < 0).any() or (caps < 0).any() or (demand < 0).any():
        raise ValueError("b, caps and demand must be non-negative")
    if (demand > caps.sum(axis=1) + 1e-9).any():
        raise _native.infeasible_error_class()("demand exceeds total capacity")
    return b, caps, demand


def _run(b, caps, demand_i64, want_grants=True):
    import torch
    rows, users = b.shape
    dev = torch.device("cuda")
    bd = torch.from_numpy(b).to(dev)
    cd = torch.from_numpy(caps).to(dev)
    dd = torch.from_numpy(demand_i64).to(dev)
    m = torch.empty((rows, users), dtype=torch.float64, device=dev)
    nu = torch.empty(rows, dtype=torch.float64, device=dev)
    dg = torch.empty(rows, dtype=torch.uint8, device=dev)
    gr = torch.empty((rows, users), dtype=torch.int64, device=dev)
    mg = torch.empty(rows, dtype=torch.float64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(_native.lib().cyr_enforce_batch_device(
        bd.data_ptr(), cd.data_ptr(), dd.data_ptr(), rows, users, m.data_ptr(), nu.data_ptr(),
        dg.data_ptr(), gr.data_ptr(), mg.data_ptr(), st.data_ptr(), _native.stream_handle()),
        "enforce_batch")
    code = int(st.item())
    if code:
        _native.check(code, "enforce_batch")
    return (m.cpu().numpy(), nu.cpu().numpy(), dg.cpu().numpy().astype(bool),
            gr.cpu().numpy(), mg.cpu().numpy())


def kl_project_batch(b, caps, demand):
    """(m_hat (R,E), nu (R,), degenerate (R,)) — enforcer.py:49-115."""
    import torch
    b, caps, demand = _validate_projection(b, caps, demand)
    rows, users = b.shape
    if rows == 0:
        return np.zeros_like(b), np.zeros(0), np.zeros(0, dtype=bool)
    dev = torch.device("cuda")
    bd, cd = torch.from_numpy(b).to(dev), torch.from_numpy(caps).to(dev)
    dd = torch.from_numpy(np.ascontiguousarray(demand)).to(dev)
    m = torch.empty((rows, users), dtype=torch.float64, device=dev)
    nu = torch.empty(rows, dtype=torch.float64, device=dev)
    dg = torch.empty(rows, dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(_native.lib().cyr_kl_project_batch_device(
        bd.data_ptr(), cd.data_ptr(), dd.data_ptr(), rows, users, m.data_ptr(), nu.data_ptr(),
        dg.data_ptr(), st.data_ptr(), _native.stream_handle()), "kl_project_batch")
    code = int(st.item())
    if code:
        _native.check(code, "kl_project_batch")
    return m.cpu().numpy(), nu.cpu().numpy(), dg.cpu().numpy().astype(bool)


def apportion_batch(m_hat, caps, demand) -> np.ndarray:
    """Integer Huntington-Hill rounding — enforcer.py:118-165."""
    import torch
    m_hat = np.ascontiguousarray(m_hat, dtype=np.float64)
    caps = np.ascontiguousarray(caps, dtype=np.float64)
    demand = np.asarray(demand)
    if m_hat.ndim != 2 or m_hat.shape != caps.shape:
        raise ValueError("shape mismatch")
    if np.any(demand < 0):
        raise ValueError("demand must be non-negative")
    if np.any(demand > caps.sum(axis=1)):
        raise _native.infeasible_error_class()("demand exceeds total capacity")
    rows, users = m_hat.shape
    want = np.zeros(rows, dtype=np.int64)
    want[:] = np.asarray(demand, dtype=np.int64)
    if rows == 0 or not want.any():
        return np.zeros((rows, users), dtype=np.int64)
    dev = torch.device("cuda")
    md = torch.from_numpy(m_hat).to(dev)
    cd = torch.from_numpy(caps).to(dev)
    wd = torch.from_numpy(want).to(dev)
    gr = torch.empty((rows, users), dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(_native.lib().cyr_apportion_batch_device(
        md.data_ptr(), cd.data_ptr(), wd.data_ptr(), rows, users, gr.data_ptr(), None,
        st.data_ptr(), _native.stream_handle()), "apportion_batch")
    code = int(st.item())
    if code:
        _native.check(code, "apportion_batch")
    return gr.cpu().numpy()


def enforce_batch(b, caps, demands, with_details: bool = False):
    """Project then round, one coupled call — enforcer.py:201-207."""
    demands = np.asarray(demands, dtype=np.int64)
    b, caps, _ = _validate_projection(b, caps, demands.astype(np.float64))
    if np.any(demands > caps.sum(axis=1)):
        raise _native.infeasible_error_class()("demand exceeds total capacity")
    if b.shape[0] == 0:
        grants = np.zeros(b.shape, dtype=np.int64)
        return (grants, {}) if with_details else grants
    m, nu, dg, grants, margin = _run(b, caps, demands)
    if with_details:
        return grants, dict(m_hat=m, nu=nu, degenerate=dg, margin=margin)
    return grants
