"""The drop-in through the reference's OWN objects and callers.

The unmodified ``punctsim`` (pip-installed into baseline/_ref)
is patched as INTEGRATION.md §1 shows (``integration.patch_punctsim``) and
driven through its own entry points:

* acceptance check 08 (pkg/tests/test_acceptance.py:419-429): ``compare``
  runs produce a byte-identical metrics.csv — here pure reference vs patched;
* ``run --train`` (engine.run_tti, engine.py:215-259, with SAC updates
  mutating agent.actor in place every TTI, so the drop-in must follow
  in-place weight changes) — metrics.csv byte-identical, with and without the
  GPU critic targets;
* ``engine.acl_pretrain`` (engine.py:314-369): identical reward histories;
* errors: the reference's ``InfeasibleDemandError`` class catches ours.
"""

import os
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def punctsim():
    if not os.path.isdir(os.path.join(REF, "punctsim")):
        pytest.skip("punctsim is not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import punctsim
    import punctsim.cli
    import punctsim.engine
    import punctsim.enforcer
    import punctsim.sac
    assert torch.cuda.is_available()
    return punctsim


@pytest.fixture
def patched(punctsim):
    from paper_2506_00167_b200.integration import patch_punctsim
    undos = []

    def apply(**kw):
        undos.append(patch_punctsim(punctsim, **kw))

    yield apply
    for u in reversed(undos):
        u()


def _cli(punctsim, argv, out):
    rc = punctsim.cli.main(argv + ["--out", str(out)])
    assert rc == 0
    return (out / "metrics.csv").read_bytes()


TRAIN_CFG = """cell.urllc_sc_len = 195
agent.batch = 16
agent.actor_hidden = 256, 256
traffic.per_ue_prob = 0.2
"""


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_acceptance_08_compare_byte_identical(punctsim, patched, tmp_path, precision):
    argv = ["compare", "--ttis", "60", "--seed", "7"]
    want = _cli(punctsim, argv, tmp_path / "ref")
    patched(precision=precision)
    got = _cli(punctsim, argv, tmp_path / "b200")
    assert len(want) > 0 and got == want
    # the reference's timing artefact is still written, from our gen_ns
    rows = (tmp_path / "b200" / "timing.csv").read_text().splitlines()
    assert rows[0] == "tti,policy,gen_ns,per_branch_us" and len(rows) == 61


@pytest.mark.parametrize("precision,gpu_targets", [("fp32", False), ("fp64", False),
                                                   ("fp64", True)])
def test_run_train_byte_identical(punctsim, patched, tmp_path, precision, gpu_targets):
    """60+ TTIs of run_tti with training: stochastic branch noise from the
    reference's generators, an actor that Adam mutates in place every TTI
    once the replay buffer holds a batch (16 records), cfg2 geometry."""
    cfg = tmp_path / "train.cfg"
    cfg.write_text(TRAIN_CFG)
    argv = ["run", "--config", str(cfg), "--train", "--ttis", "80", "--seed", "3"]
    want = _cli(punctsim, argv, tmp_path / "ref")
    patched(precision=precision, critic_targets=gpu_targets)
    got = _cli(punctsim, argv, tmp_path / "b200")
    assert got == want


def test_acl_pretrain_identical(punctsim, patched):
    from punctsim.core import CellConfig
    from punctsim.engine import CurriculumStage, acl_pretrain
    from punctsim.phy import DecodabilityModel
    from punctsim.sac import AgentHyper, make_agent
    from punctsim.seeding import substream
    cell = CellConfig(total_scs=96, num_embb=4, urllc_sc_len=24, minislots=7, rb_size=12)
    hyper = AgentHyper(actor_hidden=(64, 64), critic_hidden=(64, 64), batch=32)
    stages = (CurriculumStage(1, 20, 40), CurriculumStage(5, 10, 40))

    def run():
        agent = make_agent(cell, hyper, substream(9, "agent-init"))
        hist = acl_pretrain(agent, DecodabilityModel("threshold", margin=0.25), stages,
                            master_seed=9)
        return [np.asarray(h) for h in hist], agent

    want, ref_agent = run()
    patched(precision="fp64")
    got, agent = run()
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    for a, b in zip(agent.actor.weights, ref_agent.actor.weights):
        assert np.array_equal(a, b)


def test_reference_exception_class_catches_ours(punctsim):
    from punctsim.core import CellConfig, ScheduleVector
    from punctsim.engine import make_streams
    from punctsim.sac import AgentHyper, make_agent
    from punctsim.seeding import substream
    from paper_2506_00167_b200 import InfeasibleDemandError, build_codebook, enforcer
    cell = CellConfig(total_scs=96, num_embb=4, urllc_sc_len=24, minislots=7, rb_size=12)
    agent = make_agent(cell, AgentHyper(actor_hidden=(64,)), substream(0, "agent-init"))
    sched = ScheduleVector([12, 24, 24, 0], [0] * 4)     # 4*24 > 60: partial grid
    with pytest.raises(punctsim.enforcer.InfeasibleDemandError):
        build_codebook(agent, sched, make_streams(0, cell.num_branches), True)
    with pytest.raises(InfeasibleDemandError):
        build_codebook(agent, sched, make_streams(0, cell.num_branches), True)
    with pytest.raises(punctsim.enforcer.InfeasibleDemandError):   # test_enforcer.py:55-59
        enforcer.kl_project_batch(np.array([[1.0, 1.0]]), np.array([[1.0, 1.0]]),
                                  np.array([3.0]))
