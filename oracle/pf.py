"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — restatement of the
proportional-fair scheduler, scheduler.py:79-106:

  avg = max(state.avg_tput, 1e-6); granted = 0
  per RB: provisional = max((1-beta)*avg + beta*granted, 1e-6)
          winner = argmax(rates / provisional) (first maximum); granted += rb
  state.avg_tput = max((1-beta)*avg + beta*granted, 1e-6)
"""

from __future__ import annotations

import numpy as np

AVG_FLOOR = 1e-6


def pf_schedule(avg_tput, rates, beta: float, num_rbs: int, rb_size: int):
    """(alloc int64 (E,), new avg_tput (E,)) for one cell."""
    rates = np.asarray(rates, dtype=float)
    granted = np.zeros(rates.size)
    avg = np.maximum(np.asarray(avg_tput, dtype=float), AVG_FLOOR)
    for _ in range(num_rbs):
        provisional = np.maximum((1 - beta) * avg + beta * granted, AVG_FLOOR)
        winner = int(np.argmax(rates / provisional))
        granted[winner] += rb_size
    new_avg = np.maximum((1 - beta) * avg + beta * granted, AVG_FLOOR)
    return granted.astype(np.int64), new_avg
