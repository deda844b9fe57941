"""Boundary value types of the codebook hot path.

These mirror the reference's hot-path boundary so a
caller of ``punctsim`` can hand the same objects to this package:

* ``CellConfig``      — ``punctsim/core.py:13-49`` (``num_branches`` = ⌊N/L⌋,
  ``core.py:42-45``).
* ``ScheduleVector``  — ``punctsim/core.py:52-74``.
* ``PuncturingVector``— ``punctsim/core.py:77-101``.

Duck typing is deliberate: every public entry point of this package only
reads ``total_scs / num_embb / urllc_sc_len / minislots / num_branches``
from a cell and ``alloc`` from a schedule, so reference objects work too.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class CellConfig:
    """Static cell geometry: N subcarriers, E eMBB users, L SCs per URLLC
    packet, M mini-slots per slot, resource-block size (``core.py:13-40``)."""

    total_scs: int = 780
    num_embb: int = 10
    urllc_sc_len: int = 300
    minislots: int = 7
    rb_size: int = 12

    def __post_init__(self):
        if self.total_scs <= 0:
            raise ValueError("total_scs must be positive")
        if self.num_embb < 1:
            raise ValueError("num_embb must be >= 1")
        if not 0 < self.urllc_sc_len < self.total_scs:
            raise ValueError("urllc_sc_len must lie in (0, total_scs)")
        if self.minislots < 1:
            raise ValueError("minislots must be >= 1")
        if self.rb_size < 1 or self.total_scs % self.rb_size:
            raise ValueError("rb_size must divide total_scs")

    @property
    def num_branches(self) -> int:
        """cap = ⌊N/L⌋: the most URLLC packets one mini-slot can absorb."""
        return self.total_scs // self.urllc_sc_len

    @property
    def num_rbs(self) -> int:
        return self.total_scs // self.rb_size


@dataclass(frozen=True)
class ScheduleVector:
    """Per-slot eMBB allocation s(t): SC count and MCS index per user."""

    alloc: tuple
    mcs: tuple

    def __init__(self, alloc, mcs):
        alloc = tuple(int(v) for v in alloc)
        mcs = tuple(int(v) for v in mcs)
        if len(alloc) != len(mcs):
            raise ValueError("alloc and mcs must have equal length")
        if min(alloc, default=0) < 0:
            raise ValueError("allocations must be non-negative")
        object.__setattr__(self, "alloc", alloc)
        object.__setattr__(self, "mcs", mcs)

    def __len__(self):
        return len(self.alloc)

    @property
    def total(self) -> int:
        return sum(self.alloc)


@dataclass(frozen=True)
class PuncturingVector:
    """SCs taken from each eMBB user in one mini-slot."""

    punct: tuple

    def __init__(self, punct):
        punct = tuple(int(v) for v in punct)
        if min(punct, default=0) < 0:
            raise ValueError("puncture counts must be non-negative")
        object.__setattr__(self, "punct", punct)

    def __len__(self):
        return len(self.punct)

    @property
    def total(self) -> int:
        return sum(self.punct)

    def check_against(self, schedule) -> None:
        if len(self.punct) != len(schedule.alloc):
            raise ValueError("puncture vector length mismatch")
        if any(m > n for m, n in zip(self.punct, schedule.alloc)):
            raise ValueError("puncture count exceeds user allocation")
