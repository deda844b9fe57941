"""GPU parity for the erasure-LDPC decodability model:
cyr_ldpc_peel_device against phy.peel_decode verdicts frozen from the
unmodified reference (tests/golden/make_ldpc_golden.py), and against the
oracle on random patterns."""

import json
import os

import numpy as np
import pytest

from oracle import ldpc
from paper_2506_00167_b200 import phy

pytestmark = pytest.mark.gpu

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "ldpc_golden.npz"))
META = json.loads(str(Z["meta_json"]))


@pytest.mark.parametrize("key", sorted(META))
def test_peel_batch_matches_reference(key):
    m = META[key]
    code = phy.DecodabilityModel(code_seed=3).code_for(m["n_symbols"], m["code_rate"])
    erased = np.unpackbits(Z[key + "/erased"], axis=1)[:, :code.n].astype(bool)
    got = phy.peel_decode_batch(code, erased)
    assert np.array_equal(got, Z[key + "/ok"])


def test_peel_batch_random_patterns_and_puncture_masks():
    rng = np.random.default_rng(7)
    model = phy.DecodabilityModel(code_seed=11)
    code = model.code_for(7 * 180, 1 / 2)
    masks = [phy.puncture_mask(code, rng.integers(0, 181, size=7), 7) for _ in range(100)]
    masks += [rng.random(code.n) < p for p in np.linspace(0.0, 0.6, 100)]
    masks = np.array(masks)
    got = phy.peel_decode_batch(code, masks)
    want = [ldpc.peel_decode(code.edge_var, code.edge_check, code.n_checks, e) for e in masks]
    assert list(got) == want
    assert got[0:1].dtype == bool and got.any() and not got.all()
    with pytest.raises(ValueError):
        phy.peel_decode_batch(code, masks[:, :-1])


def test_leaf_decode_ldpc_matches_reference(golden):
    """Tree leaves under erasure_ldpc (clean channel) on the GPU: the per-leaf
    decode bitmask equals the reference's decode_user (leaf_golden.npz)."""
    from paper_2506_00167_b200 import tree
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "leaf_golden.npz"))
    info = json.loads(str(z["meta_json"]))
    key = [k for k, c in info.items() if c["margin"] == "ldpc"][0]
    case = info[key]
    cfg = golden.config(case["config"])
    s = case["slot"]
    rates = np.asarray(tree.MCS_CODE_RATES)[cfg["mcs"][s]]
    ok = phy.leaf_decode_ldpc(cfg["sto/codebook"][s], cfg["alloc"][s], rates,
                              cfg.meta["minislots"], phy.DecodabilityModel(code_seed=3))
    bits = (ok.astype(np.int64) << np.arange(ok.shape[1])[None, :]).sum(axis=1)
    assert np.array_equal(bits, z[key + "/bits"])
