"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — float64 restatement of
the actor evaluation on a slot's branch columns.

Reference:
  * column-stable GEMM, narrow batches zero-padded to width 8   neural.py:25-32
  * forward: ReLU hidden layers, identity output               neural.py:66-84
  * split_head: mu = raw[:E], log-sigma clipped to [-20, 2]    neural.py:144-150
  * sample_squashed: a = tanh(mu + exp(log_sigma) * eps)       neural.py:153-165
  * deterministic branch: a = tanh(mu)                         sac.py:349-350
  * branch input x[:E] = alloc / N, x[E] = j / cap             sac.py:344-346
  * action_to_scs: b = (a + 1) * 0.5 * alloc                   neural.py:181-183

The GEMM is OpenBLAS dgemm through numpy (not bit-reproducible across BLAS
builds), so logits are compared by tolerance; everything after the logits is
elementwise IEEE float64 and reproducible.
"""

from __future__ import annotations

import numpy as np

LOG_SIGMA_MIN = -20.0
LOG_SIGMA_MAX = 2.0
MIN_GEMM_WIDTH = 8


def _gemm(w, x):
    width = x.shape[1]
    if width == 0 or width >= MIN_GEMM_WIDTH:
        return w @ x
    padded = np.zeros((x.shape[0], MIN_GEMM_WIDTH))
    padded[:, :width] = x
    return (w @ padded)[:, :width]


def forward(weights, biases, x):
    """x: (in, columns) float64 -> raw logits (out, columns)."""
    act = np.asarray(x, dtype=np.float64)
    depth = len(weights)
    for layer, (w, b) in enumerate(zip(weights, biases)):
        z = _gemm(w, act) + b[:, None]
        act = z if layer == depth - 1 else np.maximum(z, 0.0)
    return act


def branch_inputs(alloc, total_scs: int, cap: int):
    """(E+1, cap) actor input for branches j = 1..cap of one slot."""
    alloc = np.asarray(alloc, dtype=np.float64)
    x = np.empty((alloc.size + 1, cap))
    x[:-1, :] = (alloc / total_scs)[:, None]
    x[-1, :] = np.arange(1, cap + 1, dtype=np.float64) / cap
    return x


def head(raw, num_users: int, eps=None):
    """Squashed action a (E, cols) from raw logits; eps (E, cols) or None."""
    if raw.shape[0] != 2 * num_users:
        raise ValueError("head expects 2*E rows")
    mu = raw[:num_users]
    log_sigma = np.clip(raw[num_users:], LOG_SIGMA_MIN, LOG_SIGMA_MAX)
    if eps is None:
        return np.tanh(mu)
    return np.tanh(mu + np.exp(log_sigma) * eps)


def to_subcarriers(a, alloc):
    return (a + 1.0) * 0.5 * np.asarray(alloc, dtype=np.float64)[:, None]
