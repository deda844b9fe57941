"""GPU parity for SURVEY.md §8(f) row f1: SAC critic targets.

sac.critic_targets (sac.py:167-214) on the GPU (paper_2506_00167_b200.sac)
against fixtures frozen from the unmodified reference
(tests/golden/make_critic_golden.py):

  * K3 alone on the reference's exact float64 b: ONE coupled enforcement of
    all rows (up to 1,233 here, > one CTA) — grants, m_hat, nu bit-exact;
  * the whole target computation through the C ABI
    (cyr_policy_actions_device + cyr_mlp_forward_device): the host draws the
    same noise as the reference; enforced actions bit-exact except rows the
    reference marks near-tie (HH boundary gap < 1e-5 fp32 / 1e-9 fp64);
    log pi and y within |d| <= TOL * max|.| (TOL 1e-4 fp32, 1e-9 fp64) on
    every pair whose action matched.
"""

import numpy as np
import pytest
import torch

from oracle import projection
from paper_2506_00167_b200 import enforcer, sac
from tests.golden_util import critic_cases

pytestmark = pytest.mark.gpu

NEAR_TIE = {"fp32": 1e-5, "fp64": 1e-9}
TOL = {"fp32": 1e-4, "fp64": 1e-9}
CASES = {c.name: c for c in critic_cases()}


@pytest.mark.parametrize("name", sorted(CASES))
def test_coupled_enforcement_on_reference_b(name):
    case = CASES[name]
    b = case["b"]
    m = case.meta
    k = case["k"]
    h, mm = k.shape
    pair_h = np.repeat(np.arange(h), mm)
    pair_tau = np.tile(np.arange(mm), h)
    nl = np.flatnonzero(pair_tau != mm - 1)
    next_k = k[pair_h[nl], pair_tau[nl] + 1]
    pos = np.flatnonzero(next_k > 0)
    caps = case["alloc"][pair_h[nl]][pos]
    dem = next_k[pos] * m["urllc_sc_len"]
    got, info = enforcer.enforce_batch(b, caps, dem, with_details=True)
    assert np.array_equal(got, case["grants"])
    assert np.array_equal(info["m_hat"], case["m_hat"])
    assert np.array_equal(info["nu"], case["nu"])


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_critic_targets_match_reference(name, precision):
    case = CASES[name]
    agent = case.agent()
    y, det = sac.critic_targets(agent, case.arrays(), case.rng(), precision=precision,
                                with_details=True)
    want_y, grants_ref = case["y"], case["grants"]
    got = det["grants"]
    assert got.shape == grants_ref.shape
    # near-tie rows (reference HH margin) may round differently under fp32 logits
    m = case.meta
    k = case["k"]
    h, mm = k.shape
    pair_h = np.repeat(np.arange(h), mm)
    pair_tau = np.tile(np.arange(mm), h)
    nl = np.flatnonzero(pair_tau != mm - 1)
    next_k = k[pair_h[nl], pair_tau[nl] + 1]
    pos = np.flatnonzero(next_k > 0)
    caps = case["alloc"][pair_h[nl]][pos]
    _, margin = projection.apportion(case["m_hat"], caps, next_k[pos] * m["urllc_sc_len"],
                                     with_margin=True)
    differ = (got != grants_ref).any(axis=1)
    bad = np.flatnonzero(differ & (margin >= NEAR_TIE[precision]))
    assert bad.size == 0, f"non-near-tie rows differ: {bad[:10]}"
    if differ.any():
        print(f"[near-tie] critic {name}/{precision}: {int(differ.sum())} of {differ.size} rows")
    lp_ok = ~differ
    lp_scale = max(1.0, float(np.abs(case["log_pi"]).max()))
    assert np.abs(det["log_pi"][lp_ok] - case["log_pi"][lp_ok]).max() <= TOL[precision] * lp_scale
    # y on pairs whose action matched
    same_pair = np.ones(y.size, dtype=bool)
    same_pair[nl[pos[differ]]] = False
    scale = max(1.0, float(np.abs(want_y).max()))
    err = np.abs(y[same_pair] - want_y[same_pair]).max()
    assert err <= TOL[precision] * scale, f"max |dy| {err}"
    terminal = pair_tau == mm - 1
    assert np.array_equal(y[terminal], want_y[terminal])


def test_policy_actions_rejects_bad_k():
    case = CASES["cfg1"]
    agent = case.agent()
    from paper_2506_00167_b200 import policy_for
    pol = policy_for(agent, "fp32")
    al = torch.from_numpy(case["alloc"][:4].astype(np.int32)).cuda()
    kk = torch.tensor([1, 0, 2, 1], dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        sac.policy_actions(pol, case.cell, al, kk)
