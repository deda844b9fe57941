"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — float64 restatement of
the reference feasibility enforcer.

Reference: ``/root/reference/pkg/src/punctsim/enforcer.py``
  * constants            enforcer.py:21-25
  * kl_project_batch     enforcer.py:49-115
  * apportion_batch      enforcer.py:118-165
  * enforce_batch        enforcer.py:201-207

Numerics that must be reproduced bit for bit (and that the CUDA kernel
reproduces):
  * every row sum is numpy's contiguous-row reduction, i.e. ``0.0 +
    pairwise8(row)`` (``pairwise8`` below restates it; verified against
    ``np.sum`` in tests/test_oracle.py);
  * the bisection stop test is taken over ALL bisecting rows of one call —
    rows that converged early keep bisecting until the slowest row converges
    (enforcer.py:90-97);
  * ``mid = sqrt(lo) * sqrt(hi)``; ``m_hat = min(cap, b / nu)``.
"""

from __future__ import annotations

import numpy as np

MASS_FLOOR = 1e-250       # enforcer.py:25
REL_WIDTH = 1e-13         # enforcer.py:22
MAX_ITERS = 200           # enforcer.py:21


class InfeasibleDemand(ValueError):
    """demand > total capacity (enforcer.py:28-29)."""


def pairwise8(values) -> float:
    """numpy's pairwise float64 summation for one contiguous run (n <= 128
    branch is all the hot path needs; larger n recurses on 8-aligned halves)."""
    v = [float(x) for x in values]
    n = len(v)
    if n < 8:
        acc = 0.0
        for x in v:
            acc += x
        return acc
    if n > 128:
        half = n // 2
        half -= half % 8
        return pairwise8(v[:half]) + pairwise8(v[half:])
    lanes = v[:8]
    whole = n - n % 8
    for base in range(8, whole, 8):
        for j in range(8):
            lanes[j] += v[base + j]
    acc = ((lanes[0] + lanes[1]) + (lanes[2] + lanes[3])) + \
          ((lanes[4] + lanes[5]) + (lanes[6] + lanes[7]))
    for x in v[whole:]:
        acc += x
    return acc


def project(b, caps, demand):
    """Continuous KL projection of a coupled batch of rows.

    Returns ``(m_hat (R,E), nu (R,), degenerate (R,), iterations)``; the
    iteration count is shared by all bisecting rows of the call.
    """
    b = np.asarray(b, dtype=np.float64)
    caps = np.asarray(caps, dtype=np.float64)
    demand = np.asarray(demand, dtype=np.float64)
    if b.ndim != 2 or caps.shape != b.shape or demand.shape != (b.shape[0],):
        raise ValueError("shape mismatch")
    if (b < 0).any() or (caps < 0).any() or (demand < 0).any():
        raise ValueError("b, caps and demand must be non-negative")
    if (demand > caps.sum(axis=1) + 1e-9).any():
        raise InfeasibleDemand("demand exceeds total capacity")

    rows = b.shape[0]
    m_hat = np.zeros_like(b)
    nu = np.zeros(rows)
    usable = (b > MASS_FLOOR) & (caps > 0)
    usable_cap = np.where(usable, caps, 0.0).sum(axis=1)
    wanted = demand > 0
    degenerate = wanted & (usable_cap < demand - 1e-12)
    bisect = np.flatnonzero(wanted & ~degenerate)

    iterations = 0
    if bisect.size:
        bb, cc, dd = b[bisect], caps[bisect], demand[bisect]
        ratio = np.where(usable[bisect], bb / np.maximum(cc, 1e-300), np.inf)
        hi = bb.sum(axis=1) / dd
        lo = np.minimum(ratio.min(axis=1), hi)
        while iterations < MAX_ITERS:
            if np.all(hi - lo <= REL_WIDTH * hi):
                break
            mid = np.sqrt(lo) * np.sqrt(hi)
            filled = np.minimum(cc, bb / mid[:, None]).sum(axis=1)
            above = filled >= dd
            lo = np.where(above, mid, lo)
            hi = np.where(above, hi, mid)
            iterations += 1
        level = np.sqrt(lo) * np.sqrt(hi)
        m_hat[bisect] = np.minimum(cc, bb / level[:, None])
        nu[bisect] = level

    for r in np.flatnonzero(degenerate):
        # cap every usable user; spread the slack over the others by capacity
        keep = usable[r]
        row = np.where(keep, caps[r], 0.0)
        slack = demand[r] - row.sum()
        spare = np.where(~keep, caps[r], 0.0).sum()
        if spare > 0 and slack > 0:
            row = np.where(~keep, caps[r] * slack / spare, row)
        m_hat[r] = row
    return m_hat, nu, degenerate, iterations


def _seat_table(m_hat, caps):
    """Flattened seat list of a batch: owner (row*E+user), seat index, phase,
    priority.  Phases: 0 first seat of a positive user, 1 its later seats,
    2/3 the same for zero-mass users (enforcer.py:147-157)."""
    rows, users = m_hat.shape
    per_user = np.ceil(caps).astype(np.int64).ravel()
    owner = np.repeat(np.arange(rows * users, dtype=np.int64), per_user)
    first_pos = np.cumsum(per_user) - per_user
    seat = np.arange(owner.size, dtype=np.int64) - np.repeat(first_pos, per_user)
    mass = m_hat.ravel()[owner]
    opening = seat == 0
    phase = np.where(mass > 0, 0, 2) + np.where(opening, 0, 1)
    a = seat.astype(np.float64)
    prio = np.where(opening, mass, mass / np.sqrt(np.maximum(a * (a + 1.0), 1.0)))
    return per_user, owner, seat, phase, prio


def apportion(m_hat, caps, demand, with_margin: bool = False):
    """Huntington-Hill integer rounding: per row, the top-``demand`` seats of
    the order (phase asc, priority desc, user asc, seat asc).

    With ``with_margin`` also returns, per row, the relative priority gap
    between the last granted and first refused seat when both sit in the
    same positive phase (0 or 1); +inf when the boundary is a phase change or
    nothing is refused.  That gap is the near-tie score used by the parity
    tests.
    """
    m_hat = np.asarray(m_hat, dtype=np.float64)
    caps = np.asarray(caps, dtype=np.float64)
    want = np.asarray(demand).astype(np.int64)
    if m_hat.ndim != 2 or m_hat.shape != caps.shape:
        raise ValueError("shape mismatch")
    if (np.asarray(demand) < 0).any():
        raise ValueError("demand must be non-negative")
    if (np.asarray(demand) > caps.sum(axis=1)).any():
        raise InfeasibleDemand("demand exceeds total capacity")
    rows, users = m_hat.shape
    grants = np.zeros((rows, users), dtype=np.int64)
    margin = np.full(rows, np.inf)
    if rows == 0 or not want.any():
        return (grants, margin) if with_margin else grants

    per_user, owner, seat, phase, prio = _seat_table(m_hat, caps)
    order = np.lexsort((seat, owner % users, -prio, phase, owner // users))
    seats_in_row = per_user.reshape(rows, users).sum(axis=1)
    row_start = np.cumsum(seats_in_row) - seats_in_row
    rank = np.arange(owner.size) - np.repeat(row_start, seats_in_row)
    taken = order[rank < np.repeat(want, seats_in_row)]
    np.add.at(grants.ravel(), owner[taken], 1)

    if with_margin:
        for r in range(rows):
            k = int(want[r])
            if k <= 0 or k >= seats_in_row[r]:
                continue
            last = order[row_start[r] + k - 1]
            nxt = order[row_start[r] + k]
            if phase[last] == phase[nxt] and phase[last] in (0, 1) and prio[last] > 0:
                margin[r] = (prio[last] - prio[nxt]) / prio[last]
        return grants, margin
    return grants


def enforce(b, caps, demands, with_details: bool = False):
    """enforce_batch restated (enforcer.py:201-207): project, then round."""
    demands = np.asarray(demands, dtype=np.int64)
    m_hat, nu, degenerate, iters = project(b, caps, demands.astype(np.float64))
    grants, margin = apportion(m_hat, caps, demands, with_margin=True)
    if with_details:
        return grants, dict(m_hat=m_hat, nu=nu, degenerate=degenerate,
                            iterations=iters, margin=margin)
    return grants
