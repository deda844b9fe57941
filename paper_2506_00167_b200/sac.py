"""SAC critic targets on the GPU.

``critic_targets(agent, arrays, rng)`` mirrors ``punctsim.sac.critic_targets``
(sac.py:167-214): the Near-RT update runs the same actor + feasibility
enforcement as the codebook path, but on H*(M-1) next-mini-slot columns at
once (1,536 at the default batch of 256) with ONE coupled enforcement call
across all of them (sac.py:202-205).  Here:

* the branch noise is drawn on the host from ``rng`` with the reference's
  own call (``rng.standard_normal((E, npos))``, sac.py:199), so the stream
  advances identically;
* actor forward (K2, per-column allocation rows), split_head /
  sample_squashed / log-density, action_to_scs and the coupled enforcement
  (K3, the multi-CTA call above 256 rows) run in one C-ABI call,
  ``cyr_policy_actions_device``;
* the target critics run on the GPU (``cyr_mlp_forward_device``);
* the target combination discount * (min(q1, q2) - zeta * log pi) is an
  elementwise device op.

Enforced actions are bit-exact with the reference except rows whose
Huntington-Hill boundary is a near-tie under fp32 logits (logged by the
tests); the float targets match within the tolerance stated in the tests.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .device import DevicePolicy, mlp_for, policy_for


def policy_actions(policy: DevicePolicy, cell, alloc_rows, k_rows, eps_rows=None, stream=None):
    """Enforced actions of arbitrary (allocation row, k) columns.

    alloc_rows: CUDA int32 (R, E); k_rows: CUDA int32 (R,) in 1..cap;
    eps_rows: CUDA float64 (R, E) or None (deterministic mean).  Returns
    (grants int64 (R, E), log_pi float64 (R,)) CUDA tensors — the block of
    sac.py:190-205 with all R rows in one coupled enforce_batch call.
    """
    import torch
    rows, users = int(alloc_rows.shape[0]), int(alloc_rows.shape[1])
    dev = alloc_rows.device
    grants = torch.empty((rows, users), dtype=torch.int64, device=dev)
    log_pi = torch.zeros(rows, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    if rows:
        _native.check(_native.lib().cyr_policy_actions_device(
            policy.handle, alloc_rows.contiguous().data_ptr(), k_rows.contiguous().data_ptr(),
            None if eps_rows is None else eps_rows.contiguous().data_ptr(), rows,
            cell.total_scs, cell.urllc_sc_len, grants.data_ptr(), log_pi.data_ptr(), None,
            status.data_ptr(), _native.stream_handle(stream)), "policy actions")
        code = int(status.item())
        if code:
            _native.check(code, "policy actions")
    return grants, log_pi


def critic_targets(agent, arrays, rng: np.random.Generator, *, precision: str | None = None,
                   with_details: bool = False):
    """Entropy-regularised one-step targets for every (record, mini-slot),
    as sac.critic_targets (sac.py:167-214), computed on the GPU."""
    import torch
    cell, cfg = agent.cell, agent.cfg
    alloc, k, _, reward = arrays
    alloc = np.asarray(alloc, dtype=float)
    k = np.asarray(k, dtype=np.int64)
    reward = np.asarray(reward, dtype=float)
    h, m = k.shape
    e = alloc.shape[1]
    n_total = cell.total_scs
    cap = cell.num_branches

    pair_h = np.repeat(np.arange(h), m)
    pair_tau = np.tile(np.arange(m), h)
    y = np.empty(h * m)
    last = pair_tau == m - 1
    y[last] = reward[pair_h[last]]

    nl_idx = np.flatnonzero(~last)
    next_k = k[pair_h[nl_idx], pair_tau[nl_idx] + 1]
    nl_alloc = alloc[pair_h[nl_idx]]
    pos = np.flatnonzero(next_k > 0)
    dev = torch.device("cuda")
    actions = torch.zeros((nl_idx.size, e), dtype=torch.float64, device=dev)
    log_pi = torch.zeros(nl_idx.size, dtype=torch.float64, device=dev)
    details = {}
    if pos.size:
        if np.any(nl_alloc != np.round(nl_alloc)) or np.any(nl_alloc < 0):
            raise ValueError("allocations must be non-negative integers")
        eps = rng.standard_normal((e, pos.size))           # sac.py:199, same draw
        policy = policy_for(agent, precision)
        al = torch.from_numpy(nl_alloc[pos].astype(np.int32)).to(dev)
        kk = torch.from_numpy(next_k[pos].astype(np.int32)).to(dev)
        ep = torch.from_numpy(np.ascontiguousarray(eps.T)).to(dev)
        grants, lp = policy_actions(policy, cell, al, kk, ep)
        idx = torch.from_numpy(pos).to(dev)
        actions[idx] = grants.to(torch.float64)
        log_pi[idx] = lp
        if with_details:
            details.update(grants=grants.cpu().numpy(), log_pi=lp.cpu().numpy(), pos=pos)

    # x_next = [alloc/N, k/cap, actions/N] (sac.py:207-209), one column per pair
    x = torch.empty((nl_idx.size, 2 * e + 1), dtype=torch.float64, device=dev)
    x[:, :e] = torch.from_numpy(nl_alloc).to(dev) / n_total
    x[:, e] = torch.from_numpy(next_k.astype(float)).to(dev) / cap
    x[:, e + 1:] = actions / n_total
    mlp_prec = "fp64" if (precision or "") == "fp64" else None
    q1 = mlp_for(agent.target1, mlp_prec).forward(x)[:, 0].to(torch.float64)
    q2 = mlp_for(agent.target2, mlp_prec).forward(x)[:, 0].to(torch.float64)
    q_min = torch.minimum(q1, q2)
    y[nl_idx] = (cfg.discount * (q_min - cfg.zeta * log_pi)).cpu().numpy()
    if with_details:
        details.update(q1=q1.cpu().numpy(), q2=q2.cpu().numpy())
        return y, details
    return y


def load_agent(directory, cell, cfg, precision: str | None = None, publish: bool = True):
    """sac.load_agent (sac.py:374-393): the five PSIMMLP1 networks and three
    PSIMADM1 optimiser states of an agent directory written by the
    reference's ``save_agent``, with the reference's checks and errors.
    ``publish``: the actor goes to the device as the codebook policy
    (``policy_for``) and the target critics as device MLPs (``mlp_for``),
    so ``build_codebook`` / ``critic_targets`` start without a first-call
    upload."""
    from .policy import load_agent_host
    agent = load_agent_host(directory, cell, cfg)
    if publish:
        policy_for(agent, precision)
        mlp_prec = "fp64" if (precision or "") == "fp64" else None
        mlp_for(agent.target1, mlp_prec)
        mlp_for(agent.target2, mlp_prec)
    return agent


class _ActorOnly:
    __slots__ = ("actor",)

    def __init__(self, actor):
        self.actor = actor


def policy_samples(policy: DevicePolicy, cell, alloc_rows, k_rows, eps_rows=None, stream=None):
    """The sampling half of actor_objective_grads (sac.py:265-270) on the
    GPU: actor on (allocation row, k) columns, tanh-Gaussian sample with its
    log-density, action_to_scs — no feasibility projection.
    alloc_rows CUDA int32 (R, E), k_rows CUDA int32 (R,), eps_rows CUDA
    float64 (R, E) or None.  Returns (b float64 (R, E), log_pi float64 (R,))."""
    import torch
    rows, users = int(alloc_rows.shape[0]), int(alloc_rows.shape[1])
    dev = alloc_rows.device
    b = torch.empty((rows, users), dtype=torch.float64, device=dev)
    log_pi = torch.zeros(rows, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    if rows:
        _native.check(_native.lib().cyr_policy_sample_device(
            policy.handle, alloc_rows.contiguous().data_ptr(), k_rows.contiguous().data_ptr(),
            None if eps_rows is None else eps_rows.contiguous().data_ptr(), rows,
            cell.total_scs, cell.urllc_sc_len, b.data_ptr(), log_pi.data_ptr(),
            status.data_ptr(), _native.stream_handle(stream)), "policy samples")
        code = int(status.item())
        if code:
            _native.check(code, "policy samples")
    return b, log_pi


def actor_objective(actor, critics, cell, zeta: float, alloc_rows, j_rows, eps, denom: int, *,
                    precision: str | None = None, with_details: bool = False):
    """The forward of sac.actor_objective_grads (sac.py:249-296) on the GPU:
    actor on (alloc_rows, j_rows), the sampled head with log pi, the raw SC
    demands b = action_to_scs(a) (NOT projected: the critics see b), both
    critics on [alloc/N, j/cap, b/N], and

        objective = sum(min(q1, q2) - zeta * log_pi) / denom.

    Same arguments as the reference (eps is (E, R) as actor_update draws
    it).  Returns the objective (float); gradients stay with the reference
    trainer (SAC training is out of scope)."""
    import torch
    e = cell.num_embb
    n_total = cell.total_scs
    cap = cell.num_branches
    alloc_rows = np.asarray(alloc_rows, dtype=float)
    j_rows = np.asarray(j_rows)
    rows = int(j_rows.size)
    if np.any(alloc_rows != np.round(alloc_rows)) or np.any(alloc_rows < 0):
        raise ValueError("allocations must be non-negative integers")
    dev = torch.device("cuda")
    policy = policy_for(_ActorOnly(actor), precision)
    al = torch.from_numpy(alloc_rows.astype(np.int32)).to(dev)
    kk = torch.from_numpy(j_rows.astype(np.int32)).to(dev)
    ep = torch.from_numpy(np.ascontiguousarray(np.asarray(eps, dtype=float).T)).to(dev)
    b, log_pi = policy_samples(policy, cell, al, kk, ep)
    xc = torch.empty((rows, 2 * e + 1), dtype=torch.float64, device=dev)
    xc[:, :e] = al.to(torch.float64) / n_total
    xc[:, e] = kk.to(torch.float64) / cap
    xc[:, e + 1:] = b / n_total
    mlp_prec = "fp64" if (precision or "") == "fp64" else None
    q1 = mlp_for(critics[0], mlp_prec).forward(xc)[:, 0].to(torch.float64)
    q2 = mlp_for(critics[1], mlp_prec).forward(xc)[:, 0].to(torch.float64)
    objective = float((torch.minimum(q1, q2) - zeta * log_pi).sum().item() / denom)
    if with_details:
        return objective, {"b": b.cpu().numpy(), "log_pi": log_pi.cpu().numpy(),
                           "q1": q1.cpu().numpy(), "q2": q2.cpu().numpy()}
    return objective
