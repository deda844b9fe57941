"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py) — float64 restatement of
the SAC critic targets.

Reference: punctsim.sac.critic_targets (sac.py:167-214)
  * pairs (record h, mini-slot tau); terminal pairs take the reward   sac.py:180-186
  * next-mini-slot branch k = k[h, tau+1]; rows with k > 0 sample      sac.py:188-194
    x = [alloc/N, k/cap], forward, split_head                          sac.py:195-198
    eps = rng.standard_normal((E, npos))                               sac.py:199
    a, log pi = sample_squashed (log-density with tanh Jacobian)       sac.py:200, neural.py:153-165
    b = action_to_scs(a, alloc); ONE coupled enforce_batch over rows   sac.py:201-205
  * x_next = [alloc/N, k/cap, actions/N]; q = min(target1, target2)    sac.py:207-212
  * y = discount * (q_min - zeta * log pi)                             sac.py:213
"""

from __future__ import annotations

import numpy as np

from . import mlp, projection

SQUASH_EPS = 1e-6


def log_prob(raw, num_users: int, eps):
    """(a (E, cols), log pi (cols,)) of sample_squashed (neural.py:153-165)."""
    mu = raw[:num_users]
    log_sigma = np.clip(raw[num_users:], mlp.LOG_SIGMA_MIN, mlp.LOG_SIGMA_MAX)
    a = np.tanh(mu + np.exp(log_sigma) * eps)
    lp = (-log_sigma - 0.5 * np.log(2.0 * np.pi) - 0.5 * np.square(eps)
          - np.log(1.0 - np.square(a) + SQUASH_EPS))
    return a, lp.sum(axis=0)


def critic_targets(actor, target1, target2, cell, discount, zeta, arrays, rng, details=None):
    """actor / target1 / target2: (weights, biases); cell: geometry with
    total_scs, urllc_sc_len, num_branches."""
    alloc, k, _, reward = arrays
    h, m = k.shape
    e = alloc.shape[1]
    n, cap, l = cell.total_scs, cell.num_branches, cell.urllc_sc_len
    pair_h = np.repeat(np.arange(h), m)
    pair_tau = np.tile(np.arange(m), h)
    y = np.empty(h * m)
    last = pair_tau == m - 1
    y[last] = reward[pair_h[last]]
    nl_idx = np.flatnonzero(~last)
    next_k = k[pair_h[nl_idx], pair_tau[nl_idx] + 1]
    nl_alloc = alloc[pair_h[nl_idx]]
    actions = np.zeros((nl_idx.size, e))
    log_pi = np.zeros(nl_idx.size)
    pos = np.flatnonzero(next_k > 0)
    if pos.size:
        x = np.vstack([nl_alloc[pos].T / n, next_k[pos][None, :].astype(float) / cap])
        raw = mlp.forward(*actor, x)
        eps = rng.standard_normal((e, pos.size))
        a, lp = log_prob(raw, e, eps)
        b = (a + 1.0) * 0.5 * nl_alloc[pos].T
        grants = projection.enforce(b.T, nl_alloc[pos], next_k[pos] * l)
        actions[pos] = grants
        log_pi[pos] = lp
        if details is not None:
            details.update(raw=raw, b=b.T, grants=grants, log_pi=lp, pos=pos)
    x_next = np.vstack([nl_alloc.T / n, next_k[None, :].astype(float) / cap, actions.T / n])
    q1 = mlp.forward(*target1, x_next)
    q2 = mlp.forward(*target2, x_next)
    y[nl_idx] = discount * (np.minimum(q1[0], q2[0]) - zeta * log_pi)
    return y
