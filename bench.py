"""Benchmark of the RT O-DU codebook hot path (driver contract: ONE JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], "batch of 1024 independent slots on 1
B200, throughput mode"; per rank at N>1, configs[3]-style cells sharded by
rank with one NCCL all-gather of the codebooks per step):
  * cell N=780 subcarriers, E=10 eMBB users, L=195 -> cap 4 packets per
    mini-slot, M=7 mini-slots (numerology 3); actor 2x256 (random init,
    make_agent on substream(0, "agent-init")), fp32 SIMT, stochastic head;
  * synthetic schedules (engine._synthetic_schedule's generator: uniform
    random RB owners, 65 RBs of 12 SCs) and per-branch noise;
  * one step = K2 actor + K3 codebook for 1024 slots + K1 Mode-R arrival
    tree (97,655 packed 20-byte node records per slot, 2.0 GB written).
value = codebooks/s over all ranks (each codebook carries its full arrival
tree).  The single-slot latency against the 125 us numerology-3 budget (the
first half of BASELINE's metric) is measured in the same run through the
drop-in build_codebook call and reported under "latency_us".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("codebook-gen latency per slot (µs vs 125 µs budget); "
          "codebooks/sec at 1/2/4/8 GPUs")
UNIT = "codebooks/s"
GEOM = dict(total_scs=780, num_embb=10, urllc_sc_len=195, minislots=7, rb_size=12)
HIDDEN = (256, 256)
SLOTS = 1024
BUDGET_US = 125.0
HBM_FALLBACK_GBS = 6650.0
WRITE_PEAK_GBS = 6990.0  # measured pure-write ceiling (profiles/r01_write_patterns.txt)
L2_FLUSH_BYTES = 256 << 20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def synthetic_inputs(cell, slots, seed=0):
    """Schedules as engine._synthetic_schedule draws them (engine.py:296-302)
    and the per-branch noise of ``slots`` consecutive stochastic calls."""
    from paper_2506_00167_b200 import draw_branch_noise, make_streams, substream
    rng = substream(seed, "scenario")
    allocs = np.empty((slots, cell.num_embb), dtype=np.int32)
    for s in range(slots):
        owners = rng.integers(0, cell.num_embb, size=cell.num_rbs)
        allocs[s] = np.bincount(owners, minlength=cell.num_embb) * cell.rb_size
        rng.integers(0, 6, size=cell.num_embb)  # MCS draw (keeps the stream aligned)
    eps = draw_branch_noise(make_streams(seed, cell.num_branches), cell.num_branches,
                            cell.num_embb, slots)
    return allocs, eps


def make_cell_agent():
    from paper_2506_00167_b200 import AgentHyper, CellConfig, make_agent, substream
    cell = CellConfig(**GEOM)
    agent = make_agent(cell, AgentHyper(actor_hidden=HIDDEN), substream(0, "agent-init"))
    return cell, agent


# ------------------------------------------------------------- CPU baseline
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_punctsim():
    """The UNMODIFIED reference package (``punctsim``), pip-installed into
    baseline/_ref, or None when it is not there.  Nothing
    from the product package is imported on this path."""
    if not os.path.isdir(os.path.join(REF_DIR, "punctsim")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import punctsim.core
        import punctsim.engine
        import punctsim.sac
        import punctsim.scheduler
        import punctsim.seeding
        return punctsim
    except Exception as exc:  # reported by the caller as the port fallback
        log(f"punctsim not importable from {REF_DIR}: {exc}")
        return None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_world(ps, hidden=HIDDEN):
    """The reference's own objects for the bench workload: CellConfig,
    make_agent on substream(0, "agent-init") (sac.py:114-127)."""
    cell = ps.core.CellConfig(**GEOM)
    agent = ps.sac.make_agent(cell, ps.sac.AgentHyper(actor_hidden=hidden),
                              ps.seeding.substream(0, "agent-init"))
    return cell, agent


def ref_schedules(ps, cell, slots, seed):
    """engine._synthetic_schedule (engine.py:296-302) on substream(seed,
    "scenario"): the same schedules synthetic_inputs() hands the GPU."""
    rng = ps.seeding.substream(seed, "scenario")
    return [ps.engine._synthetic_schedule(cell, ps.scheduler.DEFAULT_MCS_TABLE, rng)
            for _ in range(slots)]


_REF: dict = {}


def _ref_pool_init():
    try:  # one process per core, each with single-threaded BLAS
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _ref_worker(job):
    """Slots [lo, hi) of rank block ``seed`` through the reference's own
    ``punctsim.engine.build_codebook`` (engine.py:97-116), stochastic, with
    the branch streams advanced to slot lo first (one (lo, E) draw per branch
    equals lo sequential E-draws)."""
    seed, lo, hi = job
    ps, agent = _REF["ps"], _REF["agent"]
    scheds = _REF["scheds"][seed]
    cap, e = agent.cell.num_branches, agent.cell.num_embb
    streams = ps.engine.make_streams(seed, cap)
    if lo:
        for j in range(1, cap + 1):
            streams.branch[j].standard_normal((lo, e))
    books = np.empty((hi - lo, cap + 1, e), dtype=np.int32)
    t0 = time.perf_counter()
    for s in range(lo, hi):
        books[s - lo] = ps.engine.build_codebook(agent, scheds[s], streams).columns
    return time.perf_counter() - t0, books


def _port_worker(job):
    """Fallback when punctsim is absent: the oracle port (float64 numpy
    restatement of the same path, test infrastructure)."""
    from oracle import slot
    seed, lo, hi = job
    w, b, allocs, eps, n, l = _REF["port"][seed]
    t0 = time.perf_counter()
    books = slot.batch_codebooks(w, b, allocs[lo:hi], n, l, eps[lo:hi]).astype(np.int32)
    return time.perf_counter() - t0, books


class ReferenceCpu:
    """The reference's CPU path on the host cores: ``punctsim`` from
    baseline/_ref (kind "reference") or, when it is missing, the oracle port
    (kind "port").  One forked process per core; ``run()`` builds every
    slot of ``blocks`` rank blocks (block r = the inputs rank r's GPU arm
    uses, seed r) and returns (wall s, codebooks (blocks*slots, cap+1, E)).
    The reference has no arrival tree: only the codebooks are charged to
    it (ours also writes the Mode-R tree, so the comparison is conservative).
    """

    def __init__(self, blocks=1, slots=SLOTS, cores=None):
        import multiprocessing as mp
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        self.ps = load_punctsim()
        self.kind = "reference" if self.ps is not None else "port"
        self.blocks, self.slots = blocks, slots
        self.cores = max(1, cores or os.cpu_count() or 1)
        if self.ps is not None:
            cell, agent = ref_world(self.ps)
            _REF.update(ps=self.ps, agent=agent,
                        scheds={r: ref_schedules(self.ps, cell, slots, r) for r in range(blocks)})
            worker = _ref_worker
        else:
            cell, agent = make_cell_agent()
            port = {}
            for r in range(blocks):
                allocs, eps = synthetic_inputs(cell, slots, seed=r)
                port[r] = (agent.actor.weights, agent.actor.biases, allocs, eps,
                           cell.total_scs, cell.urllc_sc_len)
            _REF.update(port=port)
            worker = _port_worker
        per_block = max(1, self.cores // blocks)
        self.jobs = []
        for r in range(blocks):
            for c in np.array_split(np.arange(slots), min(per_block, slots)):
                if len(c):
                    self.jobs.append((r, int(c[0]), int(c[-1]) + 1))
        self.worker = worker
        self.pool = mp.get_context("fork").Pool(min(self.cores, len(self.jobs)),
                                                initializer=_ref_pool_init)

    def run(self):
        t0 = time.perf_counter()
        res = self.pool.map(self.worker, self.jobs, chunksize=1)
        wall = time.perf_counter() - t0
        return wall, np.concatenate([r[1] for r in res])

    def close(self):
        self.pool.terminate()
        self.pool.join()

    def describe(self):
        what = ("punctsim.engine.build_codebook (unmodified reference, baseline/_ref)"
                if self.kind == "reference" else
                "oracle port (float64 numpy restatement; punctsim not installed)")
        return (f"{self.blocks * self.slots} slots per step (cfg2 geometry, stochastic) through "
                f"{what}, {min(self.cores, len(self.jobs))} processes with single-threaded BLAS; "
                "codebooks only (the reference has no arrival tree)")


def _single_core_child(q, ps_dir):
    os.sched_setaffinity(0, {min(os.sched_getaffinity(0))})
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    ps = load_punctsim()
    cell, agent = ref_world(ps)
    scheds = ref_schedules(ps, cell, 64, 0)
    streams = ps.engine.make_streams(0, cell.num_branches)
    for s in range(8):
        ps.engine.build_codebook(agent, scheds[s], streams)
    ns = [ps.engine.build_codebook(agent, scheds[s], streams).gen_ns for s in range(64)]
    q.put(ns)


def single_core_reference():
    """The reference on ONE core: (1) its own timing recipe, acceptance
    check 10 (pkg/tests/test_acceptance.py:454-467: ``compare --ttis 60
    --seed 3`` with OPENBLAS_NUM_THREADS=1, per-branch us from timing.csv,
    N=780/E=10/L=300); (2) the bench geometry's per-slot gen_ns."""
    import csv
    import multiprocessing as mp
    import tempfile
    if load_punctsim() is None:
        return None
    out = {"cpu_model": cpu_model()}
    cpu0 = min(os.sched_getaffinity(0))
    with tempfile.TemporaryDirectory() as tmp:
        env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1",
                   PYTHONPATH=REF_DIR)
        res = subprocess.run([sys.executable, "-m", "punctsim", "compare", "--ttis", "60",
                              "--seed", "3", "--out", tmp], env=env, capture_output=True,
                             text=True, preexec_fn=lambda: os.sched_setaffinity(0, {cpu0}))
        if res.returncode == 0:
            with open(os.path.join(tmp, "timing.csv"), newline="") as fh:
                per_branch = np.array([float(r["per_branch_us"]) for r in csv.DictReader(fh)])
            out["acceptance10_per_branch_us"] = {
                "median": float(np.median(per_branch)),
                "p90": float(np.percentile(per_branch, 90)),
                "max": float(per_branch.max()), "ttis": int(per_branch.size),
                "recipe": "punctsim compare --ttis 60 --seed 3, OPENBLAS_NUM_THREADS=1, one "
                          "core (test_acceptance.py:454-467); N=780/E=10/L=300, actor 1x128"}
    q = mp.get_context("fork").Queue()
    p = mp.get_context("fork").Process(target=_single_core_child, args=(q, REF_DIR))
    p.start()
    ns = q.get(timeout=300)
    p.join()
    out["cfg2_slot_us"] = {"p50": float(np.median(ns)) / 1e3,
                           "p99": float(np.percentile(ns, 99)) / 1e3, "slots": len(ns),
                           "what": "punctsim build_codebook gen_ns, bench geometry (cfg2, 2x256, "
                                   "stochastic), one core, single-threaded BLAS"}
    return out


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [r for r in rows if r[2].isdigit() and int(r[2]) > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(statistics.median(float(r[0]) for r in busy)),
                "sm_max_mhz": float(max(float(r[1]) for r in rows)),
                "reasons": reasons, "samples": len(busy)}


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json (of measured)"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback (of fallback)"


def measured_peak_bf16():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops_sustained"])
    except (OSError, KeyError, ValueError):
        return 2250.0  # nominal dense bf16 (B200_PROFILING.md)


_FMA_PEAK: dict = {}


def fp32_fma_peak():
    """(TFLOP/s, source): the fp32 FMA peak MEASURED on this GPU
    (cyr_selftest_fma_peak: FFMA2 chains on every SM, event-timed; SURVEY
    §8(d) asks to measure it), the spec figure if the measurement fails."""
    if "v" not in _FMA_PEAK:
        import ctypes
        from paper_2506_00167_b200 import _native
        v = ctypes.c_double(0.0)
        try:
            _native.check(_native.lib().cyr_selftest_fma_peak(20000, ctypes.byref(v)))
            _FMA_PEAK["v"] = (v.value, "measured: FFMA2 microbenchmark on this GPU "
                                       "(cyr_selftest_fma_peak; spec 148 x 128 x 2 x 1965 MHz = "
                                       "74.4)")
        except Exception:  # reported, never fatal
            _FMA_PEAK["v"] = (148 * 128 * 2 * 1965e6 / 1e12,
                              "spec: 148 SMs x 128 FP32 lanes x 2 x 1965 MHz")
    return _FMA_PEAK["v"]


def committed_traffic():
    """dram read+write bytes per K1 launch from the committed ncu --set full
    capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_tree_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


# --------------------------------------------------------------- reference
def run_reference(args, rank, world):
    """``--impl reference``: the reference's own CPU path on the host cores
    for the same workload (world x 1024 slots per step), rank 0 only.  This
    process imports nothing from paper_2506_00167_b200."""
    if rank != 0:
        return 0
    ref = ReferenceCpu(blocks=world)
    try:
        for _ in range(args.warmup):
            ref.run()
        walls = [ref.run()[0] for _ in range(args.steps)]
    finally:
        ref.close()
    wall = float(np.mean(walls))
    total = SLOTS * world
    value = total / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(world),
        "precision": "float64 numpy (reference)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(ref.cores, len(ref.jobs)),
                         "kind": ref.kind, "sample": ref.describe(), "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_block(world):
    """Identical for both arms (the driver compares them)."""
    return {"workload": "cfg3: 1024 independent slots per rank (N=780, E=10, L=195, cap 4, "
                        "M=7), actor 2x256 random-init, stochastic; GPU arm also writes the "
                        "Mode-R arrival tree" + (", NCCL codebook all-gather" if world > 1 else ""),
            "slots_per_rank": SLOTS, "global_batch": SLOTS * world, "cells": SLOTS * world,
            "actor": "2x256", "parallelism": f"cell-sharded x{world}",
            "l2": "GPU arm: flushed (256 MiB write) between timed steps; CPU arm: n/a"}


# -------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2506_00167_b200 import CodebookEngine, DevicePolicy, _native

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cell, agent = make_cell_agent()
    allocs, eps = synthetic_inputs(cell, SLOTS, seed=rank)
    pol = DevicePolicy(agent.actor, args.precision)
    eng = CodebookEngine(pol, cell, max_slots=SLOTS, with_tree=not args.no_tree, device=dev)
    alloc_d = torch.from_numpy(allocs).to(dev)
    eps_d = torch.from_numpy(eps).to(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    lib = _native.lib()
    st = stream.cuda_stream

    def allgather(local):
        out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=dev)
        dist.all_gather_into_tensor(out, local)   # NCCL over NVLink: the one exchange
        return out

    def step(events=None, split_k2=False):
        """K2 -> K3 (-> K1) for all slots (+ all-gather); events = (start,
        tree_start, tree_end, end, actor_end) recorded on the launching stream
        (actor_end only with split_k2: every event between two kernels costs
        the step a launch gap, so the timed steps record only the four the
        step time and K1's roofline need; K2 / K3 are split in a separate
        pass)."""
        if events:
            events[0].record(stream)
        _native.check(lib.cyr_actor_forward_device(pol.handle, alloc_d.data_ptr(), SLOTS,
                                                   cell.total_scs, cell.num_branches,
                                                   eng.raw.data_ptr(), st))
        if events and split_k2:
            events[4].record(stream)
        _native.check(lib.cyr_codebook_from_raw_device(
            pol.handle, eng.raw.data_ptr(), alloc_d.data_ptr(), eps_d.data_ptr(), SLOTS,
            cell.total_scs, cell.urllc_sc_len, eng.codebooks.data_ptr(), None, None, None, None,
            eng.status.data_ptr(), st))
        if events:
            events[1].record(stream)
        if not args.no_tree:
            _native.check(lib.cyr_tree_expand_device(eng.codebooks.data_ptr(), SLOTS, eng.users,
                                                     eng.cap, cell.minislots,
                                                     eng.node_state.data_ptr(), st))
        if events:
            events[2].record(stream)
        if world > 1:
            allgather(eng.codebooks)
        if events:
            events[3].record(stream)

    launches_per_step = 2 + (0 if args.no_tree else 1)
    for _ in range(args.warmup):
        step()
    eng.check()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    with ClockSampler(local_rank) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(i)                      # L2 flush between timed steps (untimed)
            step(evs[i])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        eng.check()
        step_ms = [e[0].elapsed_time(e[3]) for e in evs]
        tree_ms = [e[1].elapsed_time(e[2]) for e in evs]
        # K2 / K3 split (kernels list only), outside the timed steps
        evk = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
        for i in range(args.steps):
            flush.fill_(i)
            step(evk[i], split_k2=True)
        torch.cuda.synchronize()
        actor_ms = float(np.mean([e[0].elapsed_time(e[4]) for e in evk]))
        k3_ms = float(np.mean([e[4].elapsed_time(e[1]) for e in evk]))

        # ---- e2e through the public serving API (CodebookStream) with host
        # buffers: every step uploads its schedules + noise from pinned host
        # memory, runs K2/K3/K1 and downloads its codebooks; two steps in
        # flight (double-buffered device sets, K1 on its own stream)
        from paper_2506_00167_b200 import CodebookStream
        alloc_h = torch.from_numpy(allocs).pin_memory()
        eps_h = torch.from_numpy(eps).pin_memory()
        outs = [torch.empty((SLOTS, cell.num_branches + 1, cell.num_embb), dtype=torch.int32,
                            pin_memory=True) for _ in range(2)]
        serve = CodebookStream(pol, cell, max_slots=SLOTS, with_tree=not args.no_tree,
                               device=dev)

        def serve_steps(k):
            pending = None
            for i in range(k):
                h = serve.submit(alloc_h, eps_h, outs[i % 2])
                if pending is not None:
                    serve.wait(pending)
                    if world > 1:
                        allgather(pending.engine.codebooks)
                        torch.cuda.synchronize()
                pending = h
            serve.wait(pending)
            if world > 1:
                allgather(pending.engine.codebooks)
            serve.drain()
            torch.cuda.synchronize()

        serve_steps(3)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        serve_steps(args.steps)
        e2e = [(time.perf_counter() - t0) / args.steps]

        # ---- single-slot latency through the drop-in build_codebook
        lat = latency_run(agent, cell, allocs, args.latency_slots, pol, dev)
        try:
            strong = cfg4_strong(pol, cell, world, rank, dev)
        except Exception as exc:  # reported, never fatal for the headline
            strong = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        mode_t = mode_t_all(cell) if (rank == 0 and not args.no_mode_t) else None
        sharded = None
        if not args.no_mode_t:
            try:
                sharded = mode_t_sharded(world, rank, dev)
            except Exception as exc:  # reported, never fatal for the headline
                sharded = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    mean_ms = float(np.mean(step_ms))
    mean_e2e = float(np.mean(e2e))
    if world > 1:
        t = torch.tensor([mean_ms, mean_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mean_ms, mean_e2e = float(t[0]), float(t[1])
    if rank != 0:
        return 0

    total = SLOTS * world
    peak, peak_src = measured_peak_hbm()
    roofline = None
    if not args.no_tree:
        nodes = eng.nodes
        tree_bytes = SLOTS * (nodes * eng.stride * 2 + (cell.num_branches + 1) * cell.num_embb * 4)
        tree_ms = float(np.mean(tree_ms))
        achieved = tree_bytes / (tree_ms * 1e-3) / 1e9
        traffic = committed_traffic()
        roofline = {"kernel": "K1 tree_kernel (Mode-R node states)", "bound": "hbm",
                    "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "peak_source": peak_src, "algorithmic_bytes_per_launch": tree_bytes,
                    "kernel_ms": tree_ms, "share_of_step": tree_ms / mean_ms,
                    "traffic": None if traffic is None else traffic.get("bytes_per_launch"),
                    "traffic_source": None if traffic is None else traffic.get("source"),
                    # K1 only writes: the pure-write ceiling measured on this pool
                    # (scripts/micro/write_patterns.cu, incompressible 3.2 GB, best
                    # store pattern; profiles/r01_write_patterns.txt)
                    "write_peak": WRITE_PEAK_GBS,
                    "frac_of_write_peak": achieved / WRITE_PEAK_GBS}

    # every kernel of the step against its bound (live CUDA-event times)
    sizes = [cell.num_embb + 1, *HIDDEN, 2 * cell.num_embb]
    k2_flops = 2.0 * SLOTS * cell.num_branches * sum(i * o for i, o in zip(sizes[:-1], sizes[1:]))
    fma_peak, fma_src = fp32_fma_peak()
    k3_bytes = SLOTS * (cell.num_branches * 2 * cell.num_embb * 4 + cell.num_embb * 4
                        + cell.num_branches * cell.num_embb * 8
                        + (cell.num_branches + 1) * cell.num_embb * 4)
    kernels = [
        {"kernel": "K2 actor_osplit_kernel (fp32 SIMT tiled, output-split warps, 4096 branch columns)", "bound": "fma",
         "ms": actor_ms, "achieved": k2_flops / (actor_ms * 1e-3) / 1e12, "peak": fma_peak,
         "unit": "TFLOP/s", "frac": k2_flops / (actor_ms * 1e-3) / 1e12 / fma_peak,
         "peak_source": fma_src,
         "work": f"{k2_flops / 1e6:.0f} MFLOP (2 * sum in*out per column)"},
        {"kernel": "K3 codebook_kernel (fp64 head + exact projection + Huntington-Hill)",
         "bound": "latency", "ms": k3_ms,
         "achieved": k3_bytes / (k3_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
         "frac": k3_bytes / (k3_ms * 1e-3) / 1e9 / peak,
         "work": f"{k3_bytes / 1e6:.2f} MB in/out; one warp per row, ~46 dependent fp64 "
                 "sqrt steps per coupled call: latency-bound, not bandwidth-bound"},
    ]
    if roofline:
        kernels.append({k: roofline[k] for k in ("kernel", "bound", "achieved", "peak", "unit",
                                                 "frac")} | {"ms": roofline["kernel_ms"]})

    cpu = None
    other_prec = None
    if world == 1:
        # the same step with the other actor precisions: fp64 (logits within
        # 1e-15 of the reference: settles the fp32 headline's precision) and
        # the optional bf16 tcgen05 actor; their codebooks' agreement with the
        # reference rides on the CPU leg
        other_prec, books_by = {}, {}
        for prec in ("fp64", "bf16_tc"):
            pol_x = DevicePolicy(agent.actor, prec)
            eng_x = CodebookEngine(pol_x, cell, max_slots=SLOTS, with_tree=not args.no_tree,
                                   device=dev)
            for _ in range(3):
                eng_x.run(alloc_d, eps_d)
            eng_x.check()
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(10)]
            for e0, e1 in ev:
                flush.fill_(7)
                e0.record(stream)
                eng_x.run(alloc_d, eps_d, stream=stream)
                e1.record(stream)
            torch.cuda.synchronize()
            ms = float(np.mean([e0.elapsed_time(e1) for e0, e1 in ev]))
            books_by[prec] = eng_x.codebooks[:SLOTS].clone()
            other_prec[prec] = {"ms_per_step": ms, "value": SLOTS / (ms * 1e-3), "unit": UNIT,
                                "steps": 10, "what": "the headline step (K2 -> K3 -> K1, 1024 "
                                                     "slots, L2 flushed) with this actor"}
            pol_x.close()
        cpu = cpu_leg(eng.codebooks, agent, cell, allocs, eps, books_by)
    line = {
        "metric": METRIC, "value": total / (mean_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32", "data": "synthetic",
        "config": config_block(world),
        "precision": f"{args.precision} actor / fp64 projection",
        "e2e": {"value": total / mean_e2e, "unit": UNIT,
                "h2d_bytes_per_step": int(allocs.nbytes + eps.nbytes),
                "d2h_bytes_per_step": int(SLOTS * (cell.num_branches + 1) * cell.num_embb * 4),
                "note": "CodebookStream (public serving API), host wall clock over all "
                        "steps: per step pinned H2D of schedules+noise, K2/K3/K1, D2H of "
                        "the codebooks (node states stay in HBM); two steps in flight; each "
                        + (f"step writes {SLOTS * eng.nodes * eng.stride * 2 / 1e9:.1f} GB "
                           "(16x L2), no separate flush" if not args.no_tree else
                           "step has no tree (--no-tree)")},
        "latency_us": lat,
        "mode_t": mode_t,
        "mode_t_sharded": sharded,
        "cfg4_strong": strong,
        "roofline": roofline,
        "kernels": kernels,
        "cpu_baseline": None if cpu is None else cpu[0],
        "parity": None if cpu is None else cpu[1],
        "other_precisions": other_prec,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_leg(gpu_books, agent, cell, allocs, eps, other_books=None, reps=3):
    """rank 0, N=1: the reference's CPU path (ReferenceCpu) on all host cores
    over this step's 1024 slots, timed over ``reps`` passes, and its
    codebooks compared with the GPU's (the timed steps' output).  Mismatched
    rows are classified with the oracle's Huntington-Hill boundary margin
    (allowed only below 1e-5 under fp32 logits)."""
    ref = ReferenceCpu(blocks=1)
    try:
        ref.run()  # warm the workers
        runs = [ref.run() for _ in range(reps)]
    finally:
        ref.close()
    wall = float(np.mean([r[0] for r in runs]))
    want = runs[-1][1]
    got = gpu_books[:SLOTS].cpu().numpy()
    diff = (got != want).any(axis=2)          # (slots, cap+1) rows
    near = 0
    if diff.any():
        from oracle import slot
        for s in np.flatnonzero(diff.any(axis=1)):
            _, info = slot.slot_codebook(agent.actor.weights, agent.actor.biases, allocs[s],
                                         cell.total_scs, cell.urllc_sc_len, eps[s], details=True)
            for j in np.flatnonzero(diff[s]):
                near += int(j >= 1 and info["margin"][j - 1] < 1e-5)
    cpu = {"value": SLOTS / wall, "unit": UNIT, "cores": min(ref.cores, len(ref.jobs)),
           "kind": ref.kind, "sample": ref.describe() + f"; mean of {reps} passes",
           "cpu_model": cpu_model(), "single_core": single_core_reference()}
    parity = {"against": ref.kind, "slots": int(got.shape[0]),
              "rows": int(diff.size - got.shape[0]), "mismatched": int(diff.sum()),
              "near_tie_logged": near, "mismatched_outside_near_tie": int(diff.sum()) - near,
              "rule": "codebook rows bit-exact except rows whose reference HH margin < 1e-5"}
    for label, books in (other_books or {}).items():
        b = books[:SLOTS].cpu().numpy()
        parity[f"{label}_row_agreement_vs_reference"] = float(
            (b[:, 1:] == want[:, 1:]).all(axis=2).mean())
    return cpu, parity


def mode_t_run(cell, hidden, slots, reps=3, fp32_reps=None):
    """North-star Mode T (actor on every arrival-tree node state): tree-batch
    time for fp32 SIMT and the bf16 tcgen05 path, and their node-decision
    agreement (BASELINE configs[4] for the cfg5 geometry)."""
    import torch
    from paper_2506_00167_b200 import DevicePolicy, substream, tree
    actor = tree.make_mode_t_actor(cell, hidden, substream(0, "mode-t"))
    allocs, eps = synthetic_inputs(cell, slots, seed=11)
    mcs = np.random.default_rng(11).integers(0, 6, size=allocs.shape).astype(np.int32)
    al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
    out, states = {}, {}
    cols = sum((cell.num_branches + 1) ** t for t in range(cell.minislots)) * cell.num_branches
    sizes = tree.mode_t_sizes(cell, hidden)
    flops = 2.0 * cols * slots * sum(i * o for i, o in zip(sizes[:-1], sizes[1:]))
    for prec in ("fp32", "bf16_tc"):
        n = (fp32_reps or reps) if prec == "fp32" else reps
        pol = DevicePolicy(actor, prec)
        st = tree.build_tree_mode_t(pol, cell, al, mc, ep)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            tree.build_tree_mode_t(pol, cell, al, mc, ep, out=st)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        states[prec] = st.cpu().numpy()[:, :, :cell.num_embb]
        eff = flops / (ms * 1e-3) / 1e12
        peak = fp32_fma_peak()[0] if prec == "fp32" else measured_peak_bf16()
        out[prec] = {"ms_per_tree_batch": ms, "trees_per_s": slots / (ms * 1e-3),
                     "actor_tflops_effective": eff,
                     "effective_frac_of_peak": eff / peak,
                     "peak": peak, "peak_source": fp32_fma_peak()[1]
                     if prec == "fp32" else "MEASURED_PEAKS.json bf16 sustained",
                     "note": "whole tree time (actor + K3 + features) over actor FLOPs"}
        pol.close()
    same = (states["fp32"] == states["bf16_tc"]).all(axis=2)
    out["_slot0"] = {k: v[0] for k, v in states.items()}
    out.update({"actor": "x".join(str(h) for h in hidden), "slots": slots,
                "cell": {"N": cell.total_scs, "E": cell.num_embb, "L": cell.urllc_sc_len,
                         "cap": cell.num_branches, "M": cell.minislots},
                "nodes_per_tree": int(same.shape[1]), "actor_columns_per_tree": cols,
                "node_agreement_bf16_vs_fp32": float(same.mean())})
    return out


def mode_t_sharded(world, rank, dev, reps=3):
    """One BASELINE configs[4] Mode-T tree (cfg5: E=16, cap 6, 3x1024 actor,
    bf16 tcgen05) split across the ranks by subtrees of level 3 (343
    subtrees; levels <= 3 replicated); each rank scores its leaves and ONE
    all-gather over NCCL assembles the per-leaf summaries (SURVEY §8(e):
    node records stay on their GPU).  Times are CUDA events, max over
    ranks.  At N > 1 rank 0 also builds the whole tree alone and checks the
    assembled one against it."""
    import torch
    import torch.distributed as dist
    from paper_2506_00167_b200 import CellConfig, DevicePolicy, substream, tree
    cell = CellConfig(780, 16, 130)
    cap, m = cell.num_branches, cell.minislots
    actor = tree.make_mode_t_actor(cell, (1024, 1024, 1024), substream(0, "mode-t"))
    allocs, eps = synthetic_inputs(cell, 1, seed=11)
    mcs = np.random.default_rng(11).integers(0, 6, size=allocs.shape).astype(np.int32)
    al, mc, ep = (torch.from_numpy(x).to(dev) for x in (allocs, mcs, eps))
    level = 3 if world > 1 else 0
    first, count = tree.shard_extent(cap, m, level, world, rank)
    lf, lc = tree.shard_leaf_range(cap, m, level, first, count)
    margins = torch.from_numpy(tree.threshold_margins(mcs)).to(dev)
    prob = torch.from_numpy(tree.admitted_count_probs(cell)).to(dev)
    pol = DevicePolicy(actor, "bf16_tc")
    out = tree.build_tree_mode_t(pol, cell, al, mc, ep, shard=(level, first, count))

    def summarise():
        # node records stay on this GPU; the per-leaf decode bitmasks and the
        # partial expectations travel
        ok, exp = tree.score_leaf_states(out, cell, al, margins, prob, lf, lc)
        if world > 1:
            return tree.gather_leaf_summary(exp, ok, cell.total_scs)
        return exp, ok, int(exp.numel() * 8 + ok.numel() * 4)

    summary = summarise()
    torch.cuda.synchronize()
    build, gather = [], []
    stream = torch.cuda.current_stream()
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e[0].record(stream)
        tree.build_tree_mode_t(pol, cell, al, mc, ep, out=out, shard=(level, first, count))
        e[1].record(stream)
        summary = summarise()
        e[2].record(stream)
        torch.cuda.synchronize()
        build.append(e[0].elapsed_time(e[1]))
        gather.append(e[1].elapsed_time(e[2]))
    t = torch.tensor([np.mean(build), np.mean(gather), np.mean(build) + np.mean(gather)],
                     dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res = {"cell": {"N": 780, "E": 16, "L": 130, "cap": cap, "M": m}, "actor": "1024x1024x1024",
           "precision": "bf16_tc", "shard_level": level, "subtrees": (cap + 1) ** level,
           "ranks": world, "ms_build_max": float(t[0]), "ms_gather_max": float(t[1]),
           "ms_per_tree": float(t[2]), "trees_per_s": 1e3 / float(t[2]),
           "gather": "per-leaf decode bitmasks + partial E[r]/E[goodput]/E[lost] (node "
                     "records stay on their GPU)",
           "gathered_bytes_per_rank": int(summary[2]),
           "whole_tree_record_bytes": int(out.numel() * out.element_size())}
    if world > 1 and rank == 0:
        whole = tree.build_tree_mode_t(pol, cell, al, mc, ep)
        ok_w, exp_w = tree.score_leaf_states(whole, cell, al, margins, prob)
        res["summary_matches_whole_tree"] = bool(
            torch.equal(summary[1], ok_w) and torch.allclose(summary[0], exp_w, rtol=1e-12))
    pol.close()
    return res


def mode_t_cpu(cell, hidden, sample_levels, gpu_slot0=None, seed=11):
    """The Mode-T oracle (float64 numpy: the reference's actor, head and
    enforcer per node) on a sampled subtree — levels 1..sample_levels of
    slot 0 of the same tree the GPU built — timed and scaled by parents (one
    coupled enforcement and cap actor columns each) to the full tree.  Mode
    T has no reference implementation; this is the port's cost (SURVEY
    §8(d)).  With ``gpu_slot0`` ({precision: node states}) the sampled
    nodes are also compared: fp32 must match outside subtrees under a
    near-tie decision (margin < 1e-5); bf16 reports its agreement."""
    from oracle import mode_t
    from paper_2506_00167_b200 import substream, tree
    actor = tree.make_mode_t_actor(cell, hidden, substream(0, "mode-t"))
    allocs, eps = synthetic_inputs(cell, 1, seed=seed)
    mcs = np.random.default_rng(seed).integers(0, 6, size=allocs.shape).astype(np.int32)
    r = cell.num_branches + 1
    sample_parents = sum(r ** t for t in range(sample_levels))
    full_parents = sum(r ** t for t in range(cell.minislots))
    t0 = time.perf_counter()
    want, margins = mode_t.mode_t_tree(actor.weights, actor.biases, allocs[0], mcs[0],
                                       cell.total_scs, cell.urllc_sc_len, cell.minislots, eps[0],
                                       details=True, stop_level=sample_levels)
    wall = time.perf_counter() - t0
    per_parent = wall / sample_parents
    out = {"sample": f"levels 1..{sample_levels} of slot 0 ({sample_parents} parents, "
                     f"{sample_parents * cell.num_branches} actor columns), one process",
           "sample_s": wall, "per_parent_ms": per_parent * 1e3,
           "est_s_per_tree_one_core": per_parent * full_parents,
           "est_trees_per_s_all_cores": (os.cpu_count() or 1) / (per_parent * full_parents),
           "cores": os.cpu_count() or 1, "kind": "port (estimate: per-parent cost x parents)"}
    if gpu_slot0:
        taint, t = np.zeros(1, dtype=bool), []
        for lvl in margins:                  # nodes whose path crosses a near-tie
            child = np.repeat(taint, r).reshape(-1, r)
            child[:, 1:] |= lvl < 1e-5
            taint = child.ravel()
            t.append(taint)
        taint = np.concatenate(t)
        n = want.shape[0]
        par = {"nodes_checked": int(n), "near_tie_nodes": int(taint.sum())}
        for prec, st in gpu_slot0.items():
            diff = (st[:n, :want.shape[1]] != want).any(axis=1)
            if prec == "fp32":
                par["fp32_mismatched"] = int(diff.sum())
                par["fp32_mismatched_outside_near_tie"] = int((diff & ~taint).sum())
            else:
                par[f"{prec}_agreement_vs_oracle"] = float(1.0 - diff.mean())
        out["parity"] = par
    return out


def mode_t_cfg3(cell, hidden, total=SLOTS, chunk=128):
    """BASELINE configs[2] in Mode T: 1024 independent slots, each with its
    full north-star tree (actor on every node state), processed as
    ``total / chunk`` tree batches back to back (the deepest level of one
    128-slot batch is 8M actor columns).  Bigger batches amortise the small,
    latency-bound levels (scripts/cfg3_chunk_probe.py, bf16: 32 / 64 / 128 /
    256 slots per batch = 17.8 / 19.3 / 20.2 / 20.7k trees/s; fp32: 32 / 128
    = 3.42 / 3.57k).  Throughput per precision, CUDA events."""
    import torch
    from paper_2506_00167_b200 import DevicePolicy, substream, tree
    actor = tree.make_mode_t_actor(cell, hidden, substream(0, "mode-t"))
    allocs, eps = synthetic_inputs(cell, total, seed=12)
    mcs = np.random.default_rng(12).integers(0, 6, size=allocs.shape).astype(np.int32)
    al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
    cols = sum((cell.num_branches + 1) ** t for t in range(cell.minislots)) * cell.num_branches
    sizes = tree.mode_t_sizes(cell, hidden)
    flops = 2.0 * cols * total * sum(i * o for i, o in zip(sizes[:-1], sizes[1:]))
    out = {"slots": total, "chunk_slots": chunk, "actor": "x".join(map(str, hidden)),
           "nodes_per_slot": int(tree.num_nodes(cell.num_branches, cell.minislots)),
           "actor_gflop": flops / 1e9}
    for prec in ("bf16_tc", "fp32"):
        pol = DevicePolicy(actor, prec)
        buf = tree.build_tree_mode_t(pol, cell, al[:chunk], mc[:chunk], ep[:chunk])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for c0 in range(0, total, chunk):
            tree.build_tree_mode_t(pol, cell, al[c0:c0 + chunk], mc[c0:c0 + chunk],
                                   ep[c0:c0 + chunk], out=buf)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        eff = flops / (ms * 1e-3) / 1e12
        peak = fp32_fma_peak()[0] if prec == "fp32" else measured_peak_bf16()
        out[prec] = {"ms_for_1024_trees": ms, "trees_per_s": total / (ms * 1e-3),
                     "actor_tflops_effective": eff, "effective_frac_of_peak": eff / peak}
        pol.close()
    return out


def mode_t_latency(reps=60):
    """One slot's whole Mode-T tree (cfg1: 3,279 nodes; cfg2: 97,655 nodes),
    fp32 actor, against the 125 us numerology-3 budget: host-observed (call
    to tree on the device, synchronised) and CUDA-event device time."""
    import torch
    from paper_2506_00167_b200 import CellConfig, DevicePolicy, substream, tree
    out = {"budget_us": BUDGET_US}
    for name, cell in (("cfg1", CellConfig(780, 4, 300)), ("cfg2", CellConfig(780, 10, 195))):
        actor = tree.make_mode_t_actor(cell, HIDDEN, substream(0, "mode-t"))
        allocs, eps = synthetic_inputs(cell, reps, seed=13)
        mcs = np.random.default_rng(13).integers(0, 6, size=allocs.shape).astype(np.int32)
        al, mc, ep = (torch.from_numpy(x).cuda() for x in (allocs, mcs, eps))
        for prec in ("fp32", "bf16_tc"):
            pol = DevicePolicy(actor, prec)
            buf = tree.build_tree_mode_t(pol, cell, al[:1], mc[:1], ep[:1])
            ws = torch.empty(max(1, pol_ws(pol, cell)), dtype=torch.uint8, device="cuda")
            torch.cuda.synchronize()
            host, dev = [], []
            for r in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter_ns()
                a.record()
                tree.build_tree_mode_t(pol, cell, al[r:r + 1], mc[r:r + 1], ep[r:r + 1], out=buf,
                                       workspace=ws)
                b.record()
                b.synchronize()
                host.append((time.perf_counter_ns() - t0) / 1e3)
                dev.append(a.elapsed_time(b) * 1e3)
            out[f"{name}_{prec}"] = {"host_p50": float(np.median(host)),
                                     "host_p99": float(np.percentile(host, 99)),
                                     "device_p50": float(np.median(dev)),
                                     "nodes": int(tree.num_nodes(cell.num_branches, 7))}
            pol.close()
    out["note"] = ("Mode T has no reference counterpart; bf16_tc runs the tensor cores only on "
                   "levels of >= 1024 actor columns (cfg2 levels 6-7)")
    return out


def pol_ws(pol, cell, slots=1):
    from paper_2506_00167_b200 import _native
    return _native.lib().cyr_tree_mode_t_workspace_bytes(pol.handle, slots, cell.num_branches,
                                                         cell.minislots)


def mode_t_all(cell):
    """cfg2 geometry (32 slots per tree batch), cfg3 (1024 slots), the cfg5
    large tree (configs[4]) and single-slot tree latency."""
    from paper_2506_00167_b200 import CellConfig
    cfg5 = CellConfig(780, 16, 130)
    out = {"cfg2": mode_t_run(cell, HIDDEN, 32),
           "cfg5": mode_t_run(cfg5, (1024, 1024, 1024), 1, reps=3, fp32_reps=1)}
    out["cfg3"] = mode_t_cfg3(cell, HIDDEN)
    out["latency"] = mode_t_latency()
    out["cfg2"]["cpu"] = mode_t_cpu(cell, HIDDEN, 4, out["cfg2"].pop("_slot0"))
    out["cfg5"]["cpu"] = mode_t_cpu(cfg5, (1024, 1024, 1024), 3, out["cfg5"].pop("_slot0"))
    return out


def _latency_stats(call_ns, gen_ns, dev_ns):
    c, g, d = (np.asarray(x, dtype=np.float64) / 1e3 for x in (call_ns, gen_ns, dev_ns))
    return {"call_p50": float(np.percentile(c, 50)), "call_p99": float(np.percentile(c, 99)),
            "call_max": float(c.max()),
            "host_p50": float(np.percentile(g, 50)), "host_p99": float(np.percentile(g, 99)),
            "host_max": float(g.max()),
            "device_p50": float(np.percentile(d, 50)), "device_p99": float(np.percentile(d, 99)),
            "slots": int(c.size)}


def _time_calls(agent, scheds, streams, n, det=False):
    from paper_2506_00167_b200 import build_codebook
    for s in range(20):
        build_codebook(agent, scheds[s % len(scheds)], streams, det)
    call, gen, dev = [], [], []
    clock = time.perf_counter_ns
    for s in range(n):
        t0 = clock()
        cb = build_codebook(agent, scheds[s % len(scheds)], streams, det)
        call.append(clock() - t0)
        gen.append(cb.gen_ns)
        dev.append(cb.device_ns)
    return _latency_stats(call, gen, dev)


def latency_run(agent, cell, allocs, n, pol_batch=None, dev=None):
    """Per-slot latency of the drop-in build_codebook against the 125 us
    budget.  ``call`` = the whole Python call as a caller sees it, in the
    DEFAULT weight-sync mode ("check": host weights compared with the
    published copy on every call — in C, overlapped with the device work);
    ``host`` = gen_ns (the reference's own timer span, engine.py:103-111);
    ``device`` = %globaltimer from request seen to codebook stored."""
    from paper_2506_00167_b200 import (AgentHyper, CellConfig, ScheduleVector, make_agent,
                                       make_streams, policy_for, set_weight_sync, substream)
    scheds = [ScheduleVector(allocs[s].tolist(), [0] * cell.num_embb) for s in range(len(allocs))]
    out = {"budget_us": BUDGET_US}
    set_weight_sync("check")
    streams = make_streams(7, cell.num_branches)
    out["stochastic"] = _time_calls(agent, scheds, streams, n)
    out["deterministic"] = _time_calls(agent, scheds, streams, n, det=True)
    policy_for(agent).quiesce()
    set_weight_sync("manual")
    out["stochastic_manual_sync"] = _time_calls(agent, scheds, streams, n)
    policy_for(agent).quiesce()
    set_weight_sync("check")
    # in-place weight change before every call (a training loop's worst
    # case): the stale answer is detected in C and recomputed
    st = _time_calls_updating(agent, scheds, streams, max(200, n // 20))
    out["stochastic_weights_changing"] = st
    policy_for(agent).quiesce()
    # republish cost alone (cyr_policy_update: device-wide quiesce, raw copy,
    # on-device pack of every layout), the 2x256 fp32 actor
    ups = []
    for _ in range(50):
        t0 = time.perf_counter_ns()
        policy_for(agent).update(agent.actor)
        ups.append((time.perf_counter_ns() - t0) / 1e3)
    out["republish_us"] = {"p50": float(np.median(ups)), "max": float(np.max(ups)),
                           "what": "DevicePolicy.update (cyr_policy_update), 2x256 fp32 actor, "
                                   "idle device"}
    if pol_batch is not None:
        out["stochastic_under_batch_load"] = _latency_under_load(agent, cell, scheds, streams,
                                                                 pol_batch, allocs, dev,
                                                                 max(1000, n // 5))
        policy_for(agent).quiesce()
    # BASELINE configs[0]: the reference's CPU-runnable cell (E=4, cap 2)
    cell1 = CellConfig(780, 4, 300)
    agent1 = make_agent(cell1, AgentHyper(actor_hidden=HIDDEN), substream(0, "agent-init"))
    allocs1, _ = synthetic_inputs(cell1, 64)
    scheds1 = [ScheduleVector(a.tolist(), [0] * 4) for a in allocs1]
    out["cfg1_stochastic"] = _time_calls(agent1, scheds1, make_streams(7, cell1.num_branches), n)
    out["cfg1_stochastic"]["cell"] = "N=780, E=4, L=300 (cap 2), actor 2x256"
    policy_for(agent1).quiesce()
    out["cell"] = "cfg2 (N=780, E=10, L=195, cap 4), actor 2x256, unless noted"
    out["path"] = ("drop-in build_codebook -> one C call -> resident slot-server cluster kernel "
                   "(mapped mailbox, no launch per call); call = Python call time in the "
                   "default 'check' weight-sync mode; host = gen_ns; device = %globaltimer "
                   "from request seen to codebook stored")
    return out


def _time_calls_updating(agent, scheds, streams, n):
    from paper_2506_00167_b200 import build_codebook
    call, gen, dev = [], [], []
    w = agent.actor.biases[-1]
    saved = w.copy()
    for s in range(n):
        w[0] = w[0]  # same value: no republish (bitwise compare)
        if s % 2:
            w[0] = np.nextafter(w[0], np.inf)  # a real in-place change every other call
        t0 = time.perf_counter_ns()
        cb = build_codebook(agent, scheds[s % len(scheds)], streams)
        call.append(time.perf_counter_ns() - t0)
        gen.append(cb.gen_ns)
        dev.append(cb.device_ns)
    w[:] = saved
    r = _latency_stats(call, gen, dev)
    r["note"] = "the actor's last bias changes in place before every other call"
    return r


def _latency_under_load(agent, cell, scheds, streams, pol_batch, allocs, dev, n):
    """Drop-in latency while a CodebookStream serving loop (1024-slot
    batches with Mode-R trees, two in flight) runs on the same GPU from a
    second host thread."""
    import threading
    import torch
    from paper_2506_00167_b200 import CodebookStream
    serve = CodebookStream(pol_batch, cell, max_slots=SLOTS, with_tree=True, device=dev)
    alloc_h = torch.from_numpy(allocs).pin_memory()
    eps_h = torch.from_numpy(synthetic_inputs(cell, SLOTS)[1]).pin_memory()
    outs = [torch.empty((SLOTS, cell.num_branches + 1, cell.num_embb), dtype=torch.int32,
                        pin_memory=True) for _ in range(2)]
    stop = threading.Event()
    batches = [0]

    def load():
        torch.cuda.set_device(dev)
        pending = None
        i = 0
        while not stop.is_set():
            h = serve.submit(alloc_h, eps_h, outs[i % 2])
            if pending is not None:
                serve.wait(pending)
                batches[0] += 1
            pending = h
            i += 1
        serve.wait(pending)
        serve.drain()

    th = threading.Thread(target=load)
    th.start()
    time.sleep(0.2)
    t0 = time.perf_counter()
    r = _time_calls(agent, scheds, streams, n)
    wall = time.perf_counter() - t0
    b0 = batches[0]
    stop.set()
    th.join()
    r["load"] = {"batches_during": b0, "batch_codebooks_per_s": b0 * SLOTS / wall,
                 "what": "CodebookStream 1024-slot batches + trees, second host thread"}
    return r


def cfg4_strong(pol, cell, world, rank, dev, steps=20):
    """BASELINE configs[3] literally: ONE 256-cell O-DU batch split across the
    ranks (strong scaling: 256 / N cells per GPU) with the NCCL all-gather of
    the codebooks; K2 -> K3 -> K1 per rank, CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2506_00167_b200 import CodebookEngine, sharding
    cells = 256
    allocs, eps = synthetic_inputs(cell, cells, seed=4)
    lo, hi = sharding.shard_bounds(cells, world, rank)
    eng = CodebookEngine(pol, cell, max_slots=max(1, hi - lo), with_tree=True, device=dev)
    al = torch.from_numpy(allocs[lo:hi]).to(dev)
    ep = torch.from_numpy(eps[lo:hi]).to(dev)
    width = sharding.max_shard(cells, world)
    padded = torch.zeros((width, cell.num_branches + 1, cell.num_embb), dtype=torch.int32,
                         device=dev)
    gathered = torch.empty((world * width,) + tuple(padded.shape[1:]), dtype=torch.int32,
                           device=dev)

    def step():
        if hi > lo:
            eng.run(al, ep)
            padded[: hi - lo].copy_(eng.codebooks[: hi - lo])
        if world > 1:
            dist.all_gather_into_tensor(gathered, padded)

    for _ in range(3):
        step()
    eng.check()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    return {"workload": "cfg4: one 256-cell batch (cfg2 geometry) split across ranks, codebooks "
                        "+ Mode-R trees, NCCL all-gather of the codebooks",
            "cells": cells, "cells_per_rank": hi - lo, "ranks": world, "ms_per_batch": ms,
            "codebooks_per_s": cells / (ms * 1e-3), "scaling": "strong",
            "timing": "CUDA events around back-to-back batches (no L2 flush), max over ranks"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    ap.add_argument("--no-tree", action="store_true")
    ap.add_argument("--latency-slots", type=int, default=10000)
    ap.add_argument("--no-mode-t", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
