"""GPU runtime contract of the drop-in path (include/cyrus_b200.h "Threading"):

* two host threads calling build_codebook on ONE agent get exactly the
  codebooks a sequential run gives (the reference's numpy path is reentrant
  for a shared, read-only agent);
* "check" weight sync: in-place changes of the host weights (Adam,
  neural.py:122-141) and replaced arrays are served on the next call, with
  the compare done in C while the device computes;
* library-internal device-wide synchronisation does not wait for a resident
  slot server's idle timeout (20 ms).
"""

import threading
import time

import numpy as np
import pytest
import torch

from oracle import slot
from paper_2506_00167_b200 import (DevicePolicy, ScheduleVector, build_codebook, make_streams,
                                   policy_for, publish, set_weight_sync)
from paper_2506_00167_b200.device import DeviceMlp, quiesce_all

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _check_mode():
    set_weight_sync("check")
    yield
    set_weight_sync("check")


def _schedules(cfg, n):
    allocs = cfg["alloc"]
    return [ScheduleVector(allocs[i % len(allocs)].tolist(), [0] * cfg.meta["num_embb"])
            for i in range(n)]


def test_concurrent_threads_one_agent(golden):
    cfg = golden.config("cfg2")
    agent = cfg.agent()
    scheds = _schedules(cfg, 40)
    threads_n = 4

    def run(seed, out):
        streams = make_streams(100 + seed, cfg.cell.num_branches)
        out.extend(build_codebook(agent, s, streams).columns for s in scheds)

    want = []
    for t in range(threads_n):
        cols = []
        run(t, cols)
        want.append(cols)
    got = [[] for _ in range(threads_n)]
    ths = [threading.Thread(target=run, args=(t, got[t])) for t in range(threads_n)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    for t in range(threads_n):
        assert got[t] == want[t], f"thread {t}: codebooks differ from the sequential run"
    policy_for(agent).quiesce()


@pytest.mark.parametrize("deterministic", [True, False])
def test_in_place_updates_are_served(golden, deterministic):
    """cfg2 geometry (the resident slot server path): the C-side compare
    runs while the cluster computes; a stale answer is recomputed."""
    cfg = golden.config("cfg2")
    agent = cfg.agent()
    n, l = cfg.meta["total_scs"], cfg.meta["urllc_sc_len"]
    sched = _schedules(cfg, 1)[0]

    def oracle_book(seed):
        eps = None
        if not deterministic:
            st = make_streams(seed, cfg.cell.num_branches)
            eps = np.stack([st.branch[j].standard_normal(cfg.meta["num_embb"])
                            for j in range(1, cfg.cell.num_branches + 1)])
        return tuple(map(tuple, slot.slot_codebook(agent.actor.weights, agent.actor.biases,
                                                   sched.alloc, n, l, eps).tolist()))

    def gpu_book(seed):
        return build_codebook(agent, sched, make_streams(seed, cfg.cell.num_branches),
                              deterministic).columns

    assert gpu_book(1) == oracle_book(1)
    rng = np.random.default_rng(5)
    for step in range(4):       # Adam-like in-place steps, then a call each
        agent.actor.weights[-1] *= 1.0 + 40.0 * rng.random()
        agent.actor.biases[-1][:] = rng.normal(0.0, 2.0, agent.actor.biases[-1].size)
        assert gpu_book(2 + step) == oracle_book(2 + step)
    # a replaced array object (not in place) is caught by identity
    agent.actor.weights[0] = agent.actor.weights[0] * -1.0
    assert gpu_book(9) == oracle_book(9)
    # "manual": the published copy is trusted until publish()
    set_weight_sync("manual")
    old = gpu_book(10)
    agent.actor.biases[-1][:] = -agent.actor.biases[-1]
    assert gpu_book(10) == old
    publish(agent)
    assert gpu_book(10) == oracle_book(10)
    policy_for(agent).quiesce()


def test_device_sync_does_not_wait_for_server_idle(golden):
    """A weight update of another object (the target critics after every
    soft update, sac.critic_targets) while the actor's slot server is
    resident: the library stops the server instead of waiting up to
    CYR_SLOT_SERVER_IDLE_MS for it."""
    cfg = golden.config("cfg2")
    agent = cfg.agent()
    sched = _schedules(cfg, 1)[0]
    streams = make_streams(0, cfg.cell.num_branches)
    critic = DeviceMlp(agent.target1, "fp32")
    torch.cuda.synchronize()  # torch's own lazy CUDA init stays out of the timed sync below
    for _ in range(5):
        build_codebook(agent, sched, streams)            # server resident now
        t0 = time.perf_counter()
        critic.update(agent.target1)                     # device-wide sync inside
        ms = (time.perf_counter() - t0) * 1e3
        assert ms < 10.0, f"update waited {ms:.1f} ms (slot-server idle wait)"
    build_codebook(agent, sched, streams)
    quiesce_all()
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    assert (time.perf_counter() - t0) * 1e3 < 5.0
    critic.close()


def test_policy_destroy_while_another_server_runs(golden):
    cfg = golden.config("cfg2")
    a1, a2 = cfg.agent(), cfg.agent()
    sched = _schedules(cfg, 1)[0]
    streams = make_streams(0, cfg.cell.num_branches)
    # one untimed create/destroy first: the first policy teardown on a fresh
    # box carries one-off driver costs (~1 s seen once) unrelated to servers
    DevicePolicy(a2.actor, "fp32").close()
    build_codebook(a1, sched, streams)
    extra = DevicePolicy(a2.actor, "fp32")
    t0 = time.perf_counter()
    extra.close()
    assert (time.perf_counter() - t0) * 1e3 < 10.0
    # the first policy's server was told to leave; its next call relaunches it
    assert build_codebook(a1, sched, make_streams(3, cfg.cell.num_branches)).columns == \
        build_codebook(a1, sched, make_streams(3, cfg.cell.num_branches)).columns
    policy_for(a1).quiesce()


def test_replaced_branch_generator_is_used(golden):
    """The C fast path checks that every streams.branch[j] is still the
    generator it cached; a replaced generator is picked up (its draws)."""
    cfg = golden.config("cfg2")
    agent = cfg.agent()
    sched = _schedules(cfg, 1)[0]
    a = make_streams(1, cfg.cell.num_branches)
    b = make_streams(1, cfg.cell.num_branches)
    assert build_codebook(agent, sched, a).columns == build_codebook(agent, sched, b).columns
    other = make_streams(9, cfg.cell.num_branches)
    a.branch[2] = other.branch[2]
    b.branch[2] = make_streams(9, cfg.cell.num_branches).branch[2]
    assert build_codebook(agent, sched, a).columns == build_codebook(agent, sched, b).columns
    policy_for(agent).quiesce()
