"""CPU: pin the oracle against the reference's golden vectors and KATs.

The oracle (oracle/) is the checker for every GPU parity test, so it must
itself reproduce the reference bit for bit.  Fixtures come from the
unmodified reference (tests/golden/make_golden.py); the known-answer tests
are the reference's own (pkg/tests/test_enforcer.py:20-105,
pkg/tests/test_engine.py:81-99).
"""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import arrival_tree, mlp, mode_t, projection, slot


def test_pairwise8_is_numpys_row_sum():
    rng = np.random.default_rng(3)
    for n in list(range(1, 40)) + [64, 127, 128, 129, 200, 300]:
        x = rng.random((5, n)) * 10.0 ** rng.uniform(-8, 8, (5, n))
        got = x.sum(axis=1)
        for r in range(5):
            assert projection.pairwise8(x[r]) == got[r]
        assert projection.pairwise8(x[0]) == x[0].sum()


@pytest.mark.parametrize("name", ["desk", "cfg1", "cfg2", "paper", "stress", "cfg5"])
@pytest.mark.parametrize("mode", ["det", "sto"])
def test_oracle_codebooks_bit_exact(golden, name, mode):
    cfg = golden.config(name)
    agent = cfg.agent()  # asserts the weight digest equals the reference's
    eps = None if mode == "det" else cfg["eps"]
    books, infos = slot.batch_codebooks(agent.actor.weights, agent.actor.biases, cfg["alloc"],
                                        cfg.meta["total_scs"], cfg.meta["urllc_sc_len"], eps,
                                        details=True)
    assert np.array_equal(books, cfg[f"{mode}/codebook"])
    for s, info in enumerate(infos):
        assert np.array_equal(info["b"], cfg[f"{mode}/b"][s])
        assert np.array_equal(info["m_hat"], cfg[f"{mode}/m_hat"][s])
        assert np.array_equal(info["nu"], cfg[f"{mode}/nu"][s])
        assert np.array_equal(info["degenerate"], cfg[f"{mode}/degenerate"][s])


def test_oracle_enforcer_corpus_bit_exact(golden):
    groups = 0
    for b, caps, dem, m_hat, nu, deg, grants in golden.enforcer_groups():
        got, info = projection.enforce(b, caps, dem, with_details=True)
        assert np.array_equal(got, grants)
        assert np.array_equal(info["m_hat"], m_hat)
        assert np.array_equal(info["nu"], nu)
        assert np.array_equal(info["degenerate"], deg)
        groups += 1
    assert groups == 400


# ---- the reference's own known-answer tests (pkg/tests/test_enforcer.py)
def _proj(b, caps, d):
    m, nu, deg, _ = projection.project(np.atleast_2d(np.asarray(b, float)),
                                       np.atleast_2d(np.asarray(caps, float)),
                                       np.asarray([d], float))
    return m[0], deg[0]


def _seats(m, caps, d):
    return list(projection.apportion(np.atleast_2d(m), np.atleast_2d(np.asarray(caps, float)),
                                     np.asarray([d]))[0])


def test_kat_worked_example():
    m, _ = _proj([8.0, 4.0, 4.0], [5, 10, 10], 12)
    assert np.allclose(m, [5.0, 3.5, 3.5], atol=1e-9)
    assert _seats(m, [5, 10, 10], 12) == [5, 4, 3]


def test_kat_degenerate_spreads_slack():
    m, deg = _proj([1.0, 0.0, 0.0], [2, 4, 2], 8)
    assert deg and m[0] == 2.0 and np.allclose(m, [2.0, 4.0, 2.0], atol=1e-9)
    m, _ = _proj([1.0, 0.0, 0.0], [2, 6, 2], 6)
    assert m[0] == 2.0 and abs(m[1] - 3.0) < 1e-9 and abs(m[2] - 1.0) < 1e-9


def test_kat_ties_caps_and_errors():
    assert _seats(np.array([2.0, 2.0, 2.0]), [4, 4, 4], 2) == [1, 1, 0]
    assert _seats(np.array([5.0, 0.1]), [3, 4], 6) == [3, 3]
    with pytest.raises(projection.InfeasibleDemand):
        _proj([1.0, 1.0], [3, 3], 7)
    with pytest.raises(ValueError):
        projection.apportion(np.array([[1.0, 1.0]]), np.array([[3.0, 3.0]]), np.array([-1]))


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 5).flatmap(lambda e: st.tuples(
    st.lists(st.floats(0.0, 50.0), min_size=e, max_size=e),
    st.lists(st.integers(1, 30), min_size=e, max_size=e),
    st.floats(0.0, 1.0))))
def test_oracle_feasibility_property(args):
    b, caps, frac = args
    demand = int(round(frac * sum(caps)))
    m, _ = _proj(b, caps, demand)
    assert abs(m.sum() - demand) < 1e-6 * max(demand, 1)
    assert np.all(m >= -1e-12) and np.all(m <= np.asarray(caps) + 1e-9)
    seats = _seats(m, caps, demand)
    assert sum(seats) == demand and all(0 <= s <= c for s, c in zip(seats, caps))


def test_codebook_column_contract(golden):
    # test_engine.py:81-99: col 0 zero, col j sums to j*L, 0 <= m <= n
    for name in golden.names:
        cfg = golden.config(name)
        l = cfg.meta["urllc_sc_len"]
        for mode in ("det", "sto"):
            books = cfg[f"{mode}/codebook"]
            assert (books[:, 0] == 0).all()
            for j in range(1, books.shape[1]):
                assert (books[:, j].sum(axis=1) == j * l).all()
            assert (books >= 0).all() and (books <= cfg["alloc"][:, None, :]).all()


def test_tree_oracle_structure():
    book = np.array([[0, 0, 0], [1, 2, 0], [3, 0, 5]])
    states = arrival_tree.node_states(book, 3)
    assert states.shape == (3 + 9 + 27, 3)
    # node of path (2, 1): level 2, index 2*3+1 = 7 -> offset 3 + 7
    assert list(states[3 + 7]) == [4, 2, 5]
    arr = arrival_tree.node_arrivals(2, 3)
    assert arr[3 + 7] == 3 and arr.max() == 6


def test_head_matches_reference_formula():
    raw = np.array([[0.5], [-0.5], [-30.0], [5.0]])
    a = mlp.head(raw, 2)
    assert np.array_equal(a, np.tanh(raw[:2]))
    eps = np.array([[0.7], [-1.1]])
    a = mlp.head(raw, 2, eps)
    assert np.array_equal(a, np.tanh(raw[:2] + np.exp(np.array([[-20.0], [2.0]])) * eps))


@pytest.mark.parametrize("name,minislots", [("desk", 3), ("cfg1", 4)])
def test_mode_t_oracle_bridge_equals_mode_r(golden, name, minislots):
    """A Mode-T actor with zero node-state columns is the reference actor at
    every node, so the Mode-T tree equals the Mode-R tree of the reference's
    own codebook (golden, from punctsim)."""
    from paper_2506_00167_b200.tree import bridge_actor
    cfg = golden.config(name)
    agent = cfg.agent()
    bridged = bridge_actor(agent.actor)
    for s in range(3):
        for mode in ("det", "sto"):
            eps = None if mode == "det" else cfg["eps"][s]
            got = mode_t.mode_t_tree(bridged.weights, bridged.biases, cfg["alloc"][s],
                                     cfg["mcs"][s], cfg.meta["total_scs"],
                                     cfg.meta["urllc_sc_len"], minislots, eps)
            want = arrival_tree.node_states(cfg[f"{mode}/codebook"][s], minislots)
            assert np.array_equal(got, want)


# ------------------------------------------------- SAC critic targets (f1)
def test_critic_oracle_matches_reference_golden():
    """oracle.critic restates sac.critic_targets bit for bit (fixtures from
    the unmodified reference, tests/golden/make_critic_golden.py), including
    the coupled enforcement of > 256 rows in one call."""
    from oracle import critic
    from tests.golden_util import critic_cases
    cases = critic_cases()
    assert max(c.meta["rows"] for c in cases) > 1000
    for case in cases:
        agent = case.agent()
        details = {}
        y = critic.critic_targets((agent.actor.weights, agent.actor.biases),
                                  (agent.target1.weights, agent.target1.biases),
                                  (agent.target2.weights, agent.target2.biases),
                                  case.cell, case.meta["discount"], case.meta["zeta"],
                                  case.arrays(), case.rng(), details)
        assert np.array_equal(y, case["y"]), case.name
        assert np.array_equal(details["grants"], case["grants"]), case.name
        assert np.array_equal(details["log_pi"], case["log_pi"]), case.name


# ------------------------------------------------- leaf scoring (f2)
def test_leaf_score_oracle_matches_reference_golden(golden):
    """oracle.leaf_score restates the reference's threshold decode + reward
    for every leaf (fixtures: tests/golden/make_leaf_golden.py)."""
    import json
    import os
    from oracle import leaf_score
    from paper_2506_00167_b200 import tree
    path = os.path.join(os.path.dirname(__file__), "golden", "leaf_golden.npz")
    z = np.load(path)
    info = json.loads(str(z["meta_json"]))
    for key, case in info.items():
        if case["margin"] == "ldpc":
            continue  # erasure_ldpc: test_ldpc_leaf_oracle_matches_reference_golden
        cfg = golden.config(case["config"])
        s = case["slot"]
        book = cfg["sto/codebook"][s]
        margin = tree.threshold_margins(cfg["mcs"][s], case["margin"])
        prob = tree.admitted_count_probs(cfg.cell)
        bits, reward, er, eg, el = leaf_score.score_leaves(book, cfg["alloc"][s], margin, prob,
                                                           cfg.meta["minislots"],
                                                           cfg.meta["total_scs"])
        assert np.array_equal(bits, z[f"{key}/bits"]), key
        assert np.array_equal(reward, z[f"{key}/reward"]), key
        good = z[f"{key}/goodput"]
        assert abs(eg - float(np.sum(_leaf_weights(prob) * good))) <= 1e-9 * max(1.0, abs(eg))
        assert abs(prob.sum(axis=1) - 1.0).max() < 1e-12
        assert er <= 0.0 and el >= 0.0


def _leaf_weights(prob):
    w = np.ones(1)
    for row in prob:
        w = (w[:, None] * row[None, :]).ravel()
    return w


# ------------------------------------------------- PF scheduler (f4)
def test_pf_oracle_matches_reference_golden():
    """oracle.pf restates scheduler.pf_schedule bit for bit over consecutive
    TTIs (fixtures: tests/golden/make_pf_golden.py)."""
    import os
    from oracle import pf
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "pf_golden.npz"))
    for e in (4, 10, 16):
        rates, beta, alloc, avg = (z[f"e{e}/{k}"] for k in ("rates", "beta", "alloc", "avg"))
        for c in range(rates.shape[1]):
            state = avg[0, c]
            for t in range(rates.shape[0]):
                a, state = pf.pf_schedule(state, rates[t, c], float(beta[c]), 65, 12)
                assert np.array_equal(a, alloc[t, c]) and np.array_equal(state, avg[t + 1, c])


# ------------------------------------------------- erasure LDPC (f2)
def _ldpc_cases():
    import json
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "ldpc_golden.npz"))
    meta = json.loads(str(z["meta_json"]))
    return z, meta


def test_ldpc_graphs_and_oracle_match_reference_golden():
    """paper_2506_00167_b200.phy builds the reference's graphs bit for bit
    (same seeded construction), and oracle.ldpc.peel_decode reproduces
    phy.peel_decode on every frozen pattern."""
    import hashlib
    from oracle import ldpc
    from paper_2506_00167_b200 import phy
    z, meta = _ldpc_cases()
    model = phy.DecodabilityModel(code_seed=3)
    for key, m in meta.items():
        code = model.code_for(m["n_symbols"], m["code_rate"])
        h = hashlib.sha256()
        h.update(code.edge_var.astype("<i8").tobytes())
        h.update(code.edge_check.astype("<i8").tobytes())
        assert (code.n, code.dv, code.dc) == (m["n"], m["dv"], m["dc"])
        assert h.hexdigest() == m["graph_sha256"], key
        erased = np.unpackbits(z[key + "/erased"], axis=1)[:, :code.n].astype(bool)
        got = [ldpc.peel_decode(code.edge_var, code.edge_check, code.n_checks, e) for e in erased]
        assert got == list(z[key + "/ok"]), key


def test_ldpc_leaf_oracle_matches_reference_golden(golden):
    """Every leaf of a cfg1 slot under the erasure_ldpc model (clean
    channel): the oracle peel on our graphs reproduces decode_user."""
    import json
    import os
    from oracle import leaf_score, ldpc
    from paper_2506_00167_b200 import phy, tree
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "leaf_golden.npz"))
    info = json.loads(str(z["meta_json"]))
    key = [k for k, c in info.items() if c["margin"] == "ldpc"][0]
    case = info[key]
    cfg = golden.config(case["config"])
    s = case["slot"]
    book, alloc, mcs = cfg["sto/codebook"][s], cfg["alloc"][s], cfg["mcs"][s]
    m = cfg.meta["minislots"]
    model = phy.DecodabilityModel(code_seed=3)
    rates = np.asarray(tree.MCS_CODE_RATES)[mcs]
    cum = leaf_score.leaf_states(book, m)
    r = book.shape[0]
    digits = np.stack(np.unravel_index(np.arange(r ** m), (r,) * m), axis=1)
    bits = np.zeros(r ** m, dtype=np.int64)
    for e in range(alloc.size):
        n_e = int(alloc[e])
        if n_e <= 0:
            bits |= 1 << e
            continue
        code = model.code_for(m * n_e, float(rates[e]))
        pats, inv = np.unique(book[digits, e], axis=0, return_inverse=True)
        ok = np.array([ldpc.peel_decode(code.edge_var, code.edge_check, code.n_checks,
                                        phy.puncture_mask(code, p, m)) for p in pats])
        bits |= ok[inv.ravel()].astype(np.int64) << e
    assert np.array_equal(bits, z[key + "/bits"])
    assert cum.shape[0] == r ** m
