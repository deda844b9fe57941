"""GPU: the optional bf16 tcgen05 actor (precision "bf16_tc").

Not a parity path: bf16 operands change logits at the 1e-3 level, so
decisions are compared as an AGREEMENT RATE (BASELINE configs[4]: "fp32
SIMT vs bf16 tcgen05 path with decision-agreement rate") — against the fp32
path AND against the reference (golden codebooks frozen from punctsim; the
Mode-T oracle for trees).  Gates sit just below the
measured rates (a packing/swizzle bug that scrambles a few percent of the
decisions fails them).  The logits must be close to fp32 and the integer
outputs must satisfy every feasibility contract.
"""

import json
import os

import numpy as np
import pytest
import torch

from paper_2506_00167_b200 import CodebookEngine, DevicePolicy, _native, tree

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(cfg, slots, seed=0):
    from bench import synthetic_inputs
    return synthetic_inputs(cfg.cell, slots, seed=seed)


def _logits(pol, cell, allocs):
    s = allocs.shape[0]
    cap = cell.num_branches
    raw = torch.empty((s * cap, 2 * cell.num_embb), dtype=torch.float32, device="cuda")
    al = torch.from_numpy(allocs).cuda()
    _native.check(_native.lib().cyr_actor_forward_device(
        pol.handle, al.data_ptr(), s, cell.total_scs, cap, raw.data_ptr(), _native.stream_handle()))
    torch.cuda.synchronize()
    return raw.double().cpu().numpy()


@pytest.mark.parametrize("name", ["cfg2", "stress", "cfg1", "cfg5"])
def test_tc_logits_close_to_fp32(golden, name):
    cfg = golden.config(name)
    agent = cfg.agent()
    allocs, _ = _inputs(cfg, 512)           # 512 slots x cap columns >= 1024: tensor-core path
    fp32 = _logits(DevicePolicy(agent.actor, "fp32"), cfg.cell, allocs)
    tc = _logits(DevicePolicy(agent.actor, "bf16_tc"), cfg.cell, allocs)
    scale = np.abs(fp32).max(axis=1, keepdims=True)
    worst = float((np.abs(tc - fp32) / scale).max())
    print(f"[bf16_tc] {name}: worst |dlogit|/max|col| = {worst:.2e}")
    assert worst < 3e-2
    assert not np.array_equal(tc, fp32)     # it really ran the bf16 path


def _record(key, value):
    path = os.path.join(ROOT, "gpurun_out", "bf16_agreement.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    data = {}
    if os.path.exists(path):
        data = json.load(open(path))
    data[key] = value
    json.dump(data, open(path, "w"), indent=1)


@pytest.mark.parametrize("name", ["cfg2", "stress"])
def test_tc_codebook_agreement_and_feasibility(golden, name):
    cfg = golden.config(name)
    agent = cfg.agent()
    slots = 1024
    allocs, eps = _inputs(cfg, slots, seed=5)
    books = {}
    for prec in ("fp32", "bf16_tc"):
        eng = CodebookEngine(DevicePolicy(agent.actor, prec), cfg.cell, max_slots=slots)
        out = eng.run(torch.from_numpy(allocs).cuda(), torch.from_numpy(eps).cuda())
        eng.check()
        books[prec] = out.cpu().numpy()
    tc = books["bf16_tc"]
    l = cfg.meta["urllc_sc_len"]
    assert (tc[:, 0] == 0).all()
    for j in range(1, tc.shape[1]):
        assert (tc[:, j].sum(axis=1) == j * l).all()
    assert (tc >= 0).all() and (tc <= allocs[:, None, :]).all()
    rows = (books["fp32"][:, 1:] == tc[:, 1:]).all(axis=2)
    rate = float(rows.mean())
    print(f"[bf16_tc] {name}: codebook-row agreement with fp32 = {rate:.4f}")
    _record(f"mode_r/{name}", rate)
    # measured 0.9993 (cfg2) / 0.925 (stress, final-scale 1.0: trained-like logits)
    assert rate >= (0.995 if name == "cfg2" else 0.90)


@pytest.mark.parametrize("name,floor", [("cfg2", 0.99), ("cfg1", 0.99), ("stress", 0.88),
                                        ("cfg5", 0.99)])
def test_tc_codebooks_agree_with_reference(golden, name, floor):
    """bf16 tcgen05 codebooks on the reference's own golden inputs (tiled to
    >= 1024 branch columns so the tensor-core path runs) against the
    codebooks the unmodified reference produced for them."""
    cfg = golden.config(name)
    agent = cfg.agent()
    allocs, eps, want = cfg["alloc"], cfg["eps"], cfg["sto/codebook"]
    reps = -(-1024 // (allocs.shape[0] * cfg.cell.num_branches))
    al = np.tile(allocs, (reps, 1)).astype(np.int32)
    ep = np.tile(eps, (reps, 1, 1))
    eng = CodebookEngine(DevicePolicy(agent.actor, "bf16_tc"), cfg.cell, max_slots=al.shape[0])
    got = eng.run(torch.from_numpy(al).cuda(), torch.from_numpy(ep).cuda())
    eng.check()
    got = got.cpu().numpy()[:allocs.shape[0]]
    rate = float((got[:, 1:] == want[:, 1:]).all(axis=2).mean())
    print(f"[bf16_tc] {name}: codebook-row agreement with the reference = {rate:.4f}")
    _record(f"mode_r_vs_reference/{name}", rate)
    assert rate >= floor


def test_tc_mode_t_agreement(golden):
    cfg = golden.config("cfg2")
    from paper_2506_00167_b200 import substream
    actor = tree.make_mode_t_actor(cfg.cell, (256, 256), substream(0, "mode-t"))
    slots = 2
    allocs, eps = _inputs(cfg, slots, seed=9)
    mcs = np.random.default_rng(1).integers(0, 6, size=allocs.shape).astype(np.int32)
    al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
    states = {}
    for prec in ("fp32", "bf16_tc"):
        states[prec] = tree.build_tree_mode_t(DevicePolicy(actor, prec), cfg.cell, al, mc,
                                              ep).cpu().numpy()
    e = cfg.meta["num_embb"]
    same = (states["fp32"][:, :, :e] == states["bf16_tc"][:, :, :e]).all(axis=2)
    rate = float(same.mean())
    leaves = tree.level_offsets(4, 7)[-1]
    leaf_rate = float(same[:, leaves:].mean())
    print(f"[bf16_tc] mode-T cfg2: node agreement {rate:.4f}, leaves {leaf_rate:.4f}")
    _record("mode_t/cfg2_nodes", rate)
    _record("mode_t/cfg2_leaves", leaf_rate)
    # levels with < 1024 columns (2 slots: levels 1-4) run fp32 SIMT and agree exactly
    four = tree.level_offsets(4, 7)[4]
    assert same[:, :four].all()
    assert rate >= 0.97 and leaf_rate >= 0.97   # measured 0.984 / 0.983
    # against the Mode-T oracle (the reference's actor, head and enforcer per
    # node, float64): levels 1..5 of slot 0 (level 5 runs the tensor cores)
    from oracle import mode_t
    want = mode_t.mode_t_tree(actor.weights, actor.biases, allocs[0], mcs[0],
                              cfg.cell.total_scs, cfg.cell.urllc_sc_len, 7, eps[0],
                              stop_level=5)
    n = want.shape[0]
    ora = float((states["bf16_tc"][0, :n, :e] == want).all(axis=1).mean())
    print(f"[bf16_tc] mode-T cfg2 levels 1-5: agreement with the oracle {ora:.4f}")
    _record("mode_t_vs_oracle/cfg2_levels1_5", ora)
    assert ora >= 0.97


def test_tc_wide_mode_t_cfg5(golden):
    """cfg5's 3 x 1024 actor runs the per-layer tensor-core GEMMs (HBM
    activation images) at every level; compare its Mode-T tree with fp32
    SIMT."""
    cfg = golden.config("cfg5")
    from paper_2506_00167_b200 import substream
    actor = tree.make_mode_t_actor(cfg.cell, (1024, 1024, 1024), substream(0, "mode-t"))
    allocs, eps = _inputs(cfg, 1, seed=11)
    mcs = np.random.default_rng(2).integers(0, 6, size=allocs.shape).astype(np.int32)
    al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
    states = {}
    for prec in ("fp32", "bf16_tc"):
        states[prec] = tree.build_tree_mode_t(DevicePolicy(actor, prec), cfg.cell, al, mc,
                                              ep).cpu().numpy()
    e = cfg.meta["num_embb"]
    same = (states["fp32"][:, :, :e] == states["bf16_tc"][:, :, :e]).all(axis=2)
    rate = float(same.mean())
    print(f"[bf16_tc] mode-T cfg5: node agreement {rate:.4f}")
    _record("mode_t/cfg5_nodes", rate)
    assert rate >= 0.995   # measured 1.0
    from oracle import mode_t
    want = mode_t.mode_t_tree(actor.weights, actor.biases, allocs[0], mcs[0],
                              cfg.cell.total_scs, cfg.cell.urllc_sc_len, 7, eps[0],
                              stop_level=3)
    n = want.shape[0]
    ora = float((states["bf16_tc"][0, :n, :e] == want).all(axis=1).mean())
    print(f"[bf16_tc] mode-T cfg5 levels 1-3: agreement with the oracle {ora:.4f}")
    _record("mode_t_vs_oracle/cfg5_levels1_3", ora)
    assert ora >= 0.99
    # every child satisfies the per-level column contract against its parent
    l = cfg.meta["urllc_sc_len"]
    st = states["bf16_tc"][0, :, :e].astype(np.int64)
    offs = tree.level_offsets(6, 7)
    for t in range(1, 7):
        child = st[offs[t]:offs[t] + 7 ** (t + 1)].reshape(-1, 7, e)
        parent = st[offs[t - 1]:offs[t - 1] + 7 ** t]
        grants = child - parent[:, None, :]
        assert (grants[:, 0] == 0).all()
        for k in range(1, 7):
            assert (grants[:, k].sum(axis=1) == k * l).all()


def test_fused_tc_mlp_equals_layer_path(golden):
    """The fused persistent tcgen05 MLP (bf16 operands in SMEM and TMEM, fp32
    accumulation) against the previous one-CTA / layer-by-layer kernels
    (CYR_TC_FUSED=0, read once per process, hence a subprocess): same bf16
    operands, same K order per accumulator, so the logits must be equal to
    fp32 rounding of the bias add."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r);"
        "from tests.golden_util import Golden; from tests.test_gpu_tc import _inputs, _logits;"
        "from paper_2506_00167_b200 import DevicePolicy;"
        "cfg = Golden.load().config('cfg2'); a, _ = _inputs(cfg, 2000);"
        "x = _logits(DevicePolicy(cfg.agent().actor, 'bf16_tc'), cfg.cell, a);"
        "np.save(sys.argv[1], x)" % ROOT)
    outs = {}
    for flag in ("1", "0"):
        path = os.path.join(ROOT, "gpurun_out", f"fused_{flag}.npy")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        env = dict(os.environ, CYR_TC_FUSED=flag)
        subprocess.run([sys.executable, "-c", code, path], env=env, check=True, cwd=ROOT)
        outs[flag] = np.load(path)
    scale = np.abs(outs["0"]).max(axis=1, keepdims=True)
    worst = float((np.abs(outs["1"] - outs["0"]) / scale).max())
    print(f"[bf16_tc] fused vs layer path: worst |dlogit|/max|col| = {worst:.2e}")
    assert worst < 1e-6


@pytest.mark.parametrize("users,slots", [(3, 1601), (7, 1111)])
def test_fused_tc_ragged_odd_users_equals_layer_path(users, slots):
    """The fused MLP's generic paths: a user count without a specialised
    feature row (E not in 4 / 10 / 16), an odd logit count (2E = 6 or 14) and
    a ragged last block whose logits are not a 16-byte multiple (the word-copy
    fallback of the head output instead of the bulk copy).  Against the
    layer path (CYR_TC_FUSED=0) in a subprocess, as above."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r);"
        "from tests.test_gpu_tc import _logits; from bench import synthetic_inputs;"
        "from paper_2506_00167_b200 import AgentHyper, CellConfig, DevicePolicy, make_agent, substream;"
        "cell = CellConfig(780, %d, 260);"
        "agent = make_agent(cell, AgentHyper(actor_hidden=(256, 256)), substream(3, 'ragged'));"
        "a, _ = synthetic_inputs(cell, %d);"
        "x = _logits(DevicePolicy(agent.actor, 'bf16_tc'), cell, a);"
        "np.save(sys.argv[1], x)" % (ROOT, users, slots))
    outs = {}
    for flag in ("1", "0"):
        path = os.path.join(ROOT, "gpurun_out", f"ragged_{users}_{flag}.npy")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        env = dict(os.environ, CYR_TC_FUSED=flag)
        subprocess.run([sys.executable, "-c", code, path], env=env, check=True, cwd=ROOT)
        outs[flag] = np.load(path)
    cap = 780 // 260
    last = (slots * cap) % 128  # columns in the ragged last block
    assert (last * 2 * users * 4) % 16 != 0  # its logits miss the bulk-copy granularity
    assert outs["1"].shape == (slots * cap, 2 * users)
    scale = np.abs(outs["0"]).max(axis=1, keepdims=True)
    worst = float((np.abs(outs["1"] - outs["0"]) / scale).max())
    assert worst < 1e-6, worst


def test_fused_tc_mode_t_generic_users_equals_layer_path():
    """Mode-T features through the fused MLP's generic (per-element) feature
    path: E = 7 (no specialised row), cap 3; the node records of the whole
    tree equal the layer path's (CYR_TC_FUSED=0), both bf16 tcgen05."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r);"
        "from bench import synthetic_inputs;"
        "from paper_2506_00167_b200 import CellConfig, DevicePolicy, substream, tree;"
        "cell = CellConfig(780, 7, 260);"
        "actor = tree.make_mode_t_actor(cell, (256, 256), substream(5, 'mode-t'));"
        "a, e = synthetic_inputs(cell, 2, seed=4);"
        "m = np.random.default_rng(2).integers(0, 6, size=a.shape).astype(np.int32);"
        "al, mc, ep = (torch.from_numpy(x).cuda() for x in (a, m, e));"
        "s = tree.build_tree_mode_t(DevicePolicy(actor, 'bf16_tc'), cell, al, mc, ep);"
        "np.save(sys.argv[1], s.cpu().numpy())" % ROOT)
    outs = {}
    for flag in ("1", "0"):
        path = os.path.join(ROOT, "gpurun_out", f"modet_generic_{flag}.npy")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        env = dict(os.environ, CYR_TC_FUSED=flag)
        subprocess.run([sys.executable, "-c", code, path], env=env, check=True, cwd=ROOT)
        outs[flag] = np.load(path)
    assert outs["1"].shape == outs["0"].shape
    assert np.array_equal(outs["1"], outs["0"])
