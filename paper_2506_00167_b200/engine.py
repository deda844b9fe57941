"""The codebook hot path: drop-in ``build_codebook`` and the batched engine.

Drop-in surface (same names, argument meaning, layout and errors as
``punctsim/engine.py``):

* ``Streams`` / ``make_streams``  — engine.py:53-78 (one ``policy-branch``
  substream per codebook column j = 1..cap).
* ``Codebook``                    — engine.py:81-94 (``columns`` is a tuple of
  cap+1 tuples of Python ints, column j sums to j*L, column 0 is zeros;
  ``gen_ns`` is the host-observed build time; ``per_branch_us``).
* ``build_codebook(agent, schedule, streams, deterministic=False)`` —
  engine.py:97-116.  Branch noise is drawn on the host from
  ``streams.branch[j]`` exactly as sac.py:351-353 does (one E-draw per
  branch per call), then ONE synchronous C-ABI call runs the actor (K2) and
  the fused action->codebook kernel (K3) on the GPU.

Throughput surface (device tensors, asynchronous on the current stream):

* ``CodebookEngine`` — S slots per call (cfg3: 1024 slots; cfg4: a shard of
  cells), optional Mode-R arrival-tree node states (K1), host-buffer
  ``run_host`` variant with pinned H2D/D2H for end-to-end timing.
"""

from __future__ import annotations

import ctypes
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native
from . import device as _device
from .device import DevicePolicy, policy_for
from .seeding import substream

try:  # CPython fast path for the single-slot call (built with the library)
    from . import _fastpath
except ImportError:  # pragma: no cover - ctypes path below is equivalent
    _fastpath = None


@dataclass
class Streams:
    """Named random substreams; each consumer owns exactly one."""

    traffic: np.random.Generator
    channel: np.random.Generator
    scenario: np.random.Generator
    batch: np.random.Generator
    target_noise: np.random.Generator
    actor_noise: np.random.Generator
    agent_init: np.random.Generator
    branch: dict            # j -> generator, one per codebook column


def make_streams(master_seed: int, num_branches: int) -> Streams:
    return Streams(
        traffic=substream(master_seed, "traffic"),
        channel=substream(master_seed, "channel"),
        scenario=substream(master_seed, "scenario"),
        batch=substream(master_seed, "training-batch"),
        target_noise=substream(master_seed, "target-noise"),
        actor_noise=substream(master_seed, "actor-noise"),
        agent_init=substream(master_seed, "agent-init"),
        branch={j: substream(master_seed, "policy-branch", j)
                for j in range(1, num_branches + 1)},
    )


@dataclass
class Codebook:
    """Puncture vector per admissible packet count; column j sums to j*L."""

    columns: tuple
    gen_ns: int
    device_ns: int = 0      # CUDA-event time of the device section (extra)

    def column(self, j: int) -> tuple:
        return self.columns[j]

    @property
    def per_branch_us(self) -> float:
        return self.gen_ns / 1e3 / max(len(self.columns) - 1, 1)


def draw_branch_noise(streams, cap: int, num_users: int, slots: int = 1) -> np.ndarray:
    """(slots, cap, E) float64: what ``slots`` consecutive stochastic calls
    draw from the per-branch generators (sac.py:351-353).  Drawing (S, E) at
    once equals S sequential E-draws (PCG64 + ziggurat are stream-stable)."""
    eps = np.empty((slots, cap, num_users))
    for j in range(1, cap + 1):
        eps[:, j - 1, :] = streams.branch[j].standard_normal((slots, num_users))
    return eps


_BITGENS: dict = {}


def _bitgen_entry(streams, cap: int) -> tuple:
    """(branch dict, generators of j = 1..cap, their bitgen_t addresses),
    cached per Streams object (the entry goes when the Streams object
    does); the C fast path re-checks the generators' identity every call."""
    key = id(streams)
    entry = _BITGENS.get(key)
    branch = streams.branch
    if entry is not None and entry[0] is branch and len(entry[1]) == cap and all(
            branch.get(j) is g for j, g in enumerate(entry[1], start=1)):
        return entry
    gens = tuple(branch[j] for j in range(1, cap + 1))
    addrs = tuple(g.bit_generator.ctypes.bit_generator.value for g in gens)
    if key not in _BITGENS:
        weakref.finalize(streams, _BITGENS.pop, key, None)
    entry = _BITGENS[key] = (branch, gens, addrs)
    return entry


def branch_bitgens(streams, cap: int) -> tuple:
    """bitgen_t addresses of streams.branch[1..cap]."""
    return _bitgen_entry(streams, cap)[2]


_STALE_ARRAYS, _STALE_GENS = -100, -101


def build_codebook(agent, schedule, streams, deterministic: bool = False, *,
                   policy: DevicePolicy | None = None, precision: str | None = None) -> Codebook:
    """All branches of one slot on the GPU: actor, head, KL projection,
    Huntington-Hill — one coupled enforcement per slot (engine.py:97-116)."""
    cell = agent.cell
    if _fastpath is not None:
        # per-call bookkeeping in C: the registered weight arrays must still
        # be the actor's (identity), the branch generators the cached ones;
        # contents are compared by the library while the device computes
        actor = agent.actor
        branch = None if deterministic else streams.branch
        for _ in range(3):
            arrays = None
            if policy is not None:
                pol = policy
            else:
                entry = _device.fast_entry(actor, precision)
                if entry is None:
                    pol = policy_for(agent, precision, deferred=True)
                    entry = _device.fast_entry(actor, precision)
                else:
                    pol = entry.policy
                if entry is not None:
                    arrays = entry.arrays
            gens = addrs = None
            if branch is not None:
                _, gens, addrs = _bitgen_entry(streams, cell.num_branches)
            status, columns, gen_ns, dev_ns = _fastpath.codebook2(
                pol.handle.value, schedule.alloc, branch, gens, addrs, cell.total_scs,
                cell.urllc_sc_len, cell.num_embb, actor.weights, actor.biases, arrays)
            if status == _STALE_ARRAYS:
                policy_for(agent, precision, deferred=True)   # re-register (republishes)
                continue
            if status == _STALE_GENS:
                _BITGENS.pop(id(streams), None)
                continue
            if status:
                _native.check(status, "build_codebook")
            return Codebook(columns=columns, gen_ns=gen_ns, device_ns=dev_ns)
        raise RuntimeError("build_codebook: weight arrays or branch generators keep changing")
    cap = cell.num_branches
    users = cell.num_embb
    alloc = np.ascontiguousarray(schedule.alloc, dtype=np.int32)
    if alloc.shape != (users,):
        raise ValueError("input must be (input_dim, batch)")
    t0 = time.perf_counter_ns()
    pol = policy if policy is not None else policy_for(agent, precision, deferred=True)
    eps = None
    if not deterministic:
        eps = np.empty((cap, users))
        for j in range(1, cap + 1):
            eps[j - 1] = streams.branch[j].standard_normal(users)
    book = np.empty((cap + 1, users), dtype=np.int32)
    dev_ns = ctypes.c_int64(0)
    status = _native.lib().cyr_codebook_host(
        pol.handle, alloc.ctypes.data, None if eps is None else eps.ctypes.data, 1,
        cell.total_scs, cell.urllc_sc_len, book.ctypes.data, ctypes.byref(dev_ns))
    gen_ns = time.perf_counter_ns() - t0
    _native.check(status, "build_codebook")
    columns = tuple(tuple(row) for row in book.tolist())
    return Codebook(columns=columns, gen_ns=gen_ns, device_ns=dev_ns.value)


def build_codebooks_host(policy: DevicePolicy, cell, allocs, eps=None):
    """Synchronous batch of S independent slots from host arrays.

    allocs (S, E) ints; eps (S, cap, E) float64 or None (deterministic).
    Returns (codebooks (S, cap+1, E) int32, device_ns).
    """
    allocs = np.ascontiguousarray(allocs, dtype=np.int32)
    slots, users = allocs.shape
    cap = cell.num_branches
    if eps is not None:
        eps = np.ascontiguousarray(eps, dtype=np.float64)
        if eps.shape != (slots, cap, users):
            raise ValueError("eps must be (S, cap, E)")
    out = np.empty((slots, cap + 1, users), dtype=np.int32)
    dev_ns = ctypes.c_int64(0)
    _native.check(_native.lib().cyr_codebook_host(
        policy.handle, allocs.ctypes.data, None if eps is None else eps.ctypes.data, slots,
        cell.total_scs, cell.urllc_sc_len, out.ctypes.data, ctypes.byref(dev_ns)),
        "build_codebooks_host")
    return out, dev_ns.value


class CodebookEngine:
    """Device-resident batch engine: S slots per call, one stream.

    ``run(alloc, eps)`` takes CUDA tensors (alloc (S, E) int32, eps
    (S, cap, E) float64 or None) and enqueues K2 -> K3 (-> K1 when
    ``with_tree``) on the current torch stream without synchronising;
    results land in ``self.codebooks`` / ``self.node_state``.
    ``check()`` synchronises the stream of the last ``run`` (not the whole
    device) and raises the reference's exception for a failing slot.
    """

    def __init__(self, policy: DevicePolicy, cell, max_slots: int, with_tree: bool = False,
                 device=None):
        import torch
        from . import tree as _tree
        self.torch = torch
        self.policy = policy
        self.cell = cell
        self.max_slots = int(max_slots)
        self.cap = cell.num_branches
        self.users = cell.num_embb
        if self.users != policy.num_users:
            raise ValueError("policy and cell disagree on the number of eMBB users")
        dev = torch.device(device or "cuda")
        self.device = dev
        cap, e = self.cap, self.users
        raw_dtype = torch.float64 if policy.precision == "fp64" else torch.float32
        self.raw = torch.empty((self.max_slots * cap, 2 * e), dtype=raw_dtype, device=dev)
        self.codebooks = torch.empty((self.max_slots, cap + 1, e), dtype=torch.int32, device=dev)
        self.status = torch.zeros(4, dtype=torch.int32, device=dev)
        self.with_tree = with_tree
        self.node_state = None
        if with_tree:
            _tree.check_tree_geometry(cell)
            self.nodes = _tree.num_nodes(cap, cell.minislots)
            self.stride = _tree.state_stride(e)
            self.node_state = torch.empty((self.max_slots, self.nodes, self.stride),
                                          dtype=torch.int16, device=dev)

    def run(self, alloc, eps=None, slots: int | None = None, stream=None):
        lib = _native.lib()
        s = int(alloc.shape[0]) if slots is None else int(slots)
        if s > self.max_slots:
            raise ValueError("more slots than the engine was sized for")
        if eps is not None and tuple(eps.shape[1:]) != (self.cap, self.users):
            raise ValueError("eps must be (S, cap, E)")
        torch = self.torch
        self._stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        st = self._stream.cuda_stream
        cell = self.cell
        _native.check(lib.cyr_actor_forward_device(
            self.policy.handle, alloc.data_ptr(), s, cell.total_scs, self.cap,
            self.raw.data_ptr(), st), "actor")
        _native.check(lib.cyr_codebook_from_raw_device(
            self.policy.handle, self.raw.data_ptr(), alloc.data_ptr(),
            None if eps is None else eps.data_ptr(), s, cell.total_scs, cell.urllc_sc_len,
            self.codebooks.data_ptr(), None, None, None, None, self.status.data_ptr(), st),
            "codebook")
        if self.with_tree:
            _native.check(lib.cyr_tree_expand_device(
                self.codebooks.data_ptr(), s, self.users, self.cap, cell.minislots,
                self.node_state.data_ptr(), st), "tree")
        return self.codebooks[:s]

    def check(self, stream=None) -> None:
        """Synchronise ``stream`` (default: the stream of the last ``run``,
        else the device's current stream) and raise the reference's
        exception for a failing slot."""
        stream = stream or getattr(self, "_stream", None) or \
            self.torch.cuda.current_stream(self.device)
        stream.synchronize()
        code = int(self.status[0].item())
        if code:
            with self.torch.cuda.stream(stream):
                self.status.zero_()
            stream.synchronize()
            _native.check(code, "codebook batch")

    def run_host(self, alloc_pinned, eps_pinned=None, out_pinned=None, stream=None):
        """End-to-end batch: H2D of this step's inputs from pinned host memory,
        K2/K3(/K1), D2H of the codebooks; synchronous."""
        torch = self.torch
        s = int(alloc_pinned.shape[0])
        alloc_d = alloc_pinned.to(self.device, non_blocking=True)
        eps_d = None if eps_pinned is None else eps_pinned.to(self.device, non_blocking=True)
        self.run(alloc_d, eps_d, slots=s, stream=stream)
        if out_pinned is None:
            out_pinned = torch.empty((s, self.cap + 1, self.users), dtype=torch.int32,
                                     pin_memory=True)
        out_pinned.copy_(self.codebooks[:s], non_blocking=True)
        self.check()
        return out_pinned


@dataclass
class StreamBatch:
    """Handle of one ``CodebookStream.submit``."""

    ready: object          # event: codebooks are on the host
    tree_ready: object     # event: the batch's node states are in HBM (or None)
    engine: CodebookEngine
    out: object            # pinned host codebooks (S, cap+1, E)
    node_state: object     # device node states (S, nodes, Ep) of this batch, or None
    slots: int
    inputs: tuple          # device inputs, kept alive until their stream consumed them


class CodebookStream:
    """Slot-after-slot O-DU serving loop on one GPU (the batch API a
    scheduler calls every slot).

    ``submit(alloc_pinned, eps_pinned, out_pinned)`` enqueues one batch:
    H2D of its schedules and branch noise from pinned host memory, K2 -> K3
    (codebooks), the D2H of the codebooks into ``out_pinned``, and K1 (the
    arrival tree, left in HBM) when ``with_tree``.  Two batches are in
    flight: batch i+1's upload and actor/enforcement are issued while batch
    i's tree expansion and download run, on separate CUDA streams, with the
    device buffers — codebooks AND node states — double-buffered per batch.
    ``wait(handle)`` returns ``out_pinned`` once that batch's codebooks are
    on the host, raising the reference's exception for a failing slot.
    ``tree(handle)`` waits for that batch's K1 and returns its node states
    (valid until the second ``submit`` after it reuses the buffer set).
    Nothing is skipped: every batch does all of its H2D, kernels and D2H.
    """

    def __init__(self, policy: DevicePolicy, cell, max_slots: int, with_tree: bool = True,
                 device=None):
        import torch
        self.torch = torch
        self.engines = [CodebookEngine(policy, cell, max_slots, with_tree=False, device=device)
                        for _ in range(2)]
        eng = self.engines[0]
        self.cell, self.cap, self.users, self.device = cell, eng.cap, eng.users, eng.device
        self.with_tree = with_tree
        self.node_states = [None, None]
        if with_tree:
            from . import tree as _tree
            _tree.check_tree_geometry(cell)
            shape = (int(max_slots), _tree.num_nodes(self.cap, cell.minislots),
                     _tree.state_stride(self.users))
            self.node_states = [torch.empty(shape, dtype=torch.int16, device=eng.device)
                                for _ in range(2)]
        self.s_main = torch.cuda.Stream(device=eng.device)  # uploads, K2, K3, downloads
        self.s_tree = torch.cuda.Stream(device=eng.device)  # K1
        self.free = [torch.cuda.Event() for _ in range(2)]  # buffer set reusable
        self.count = 0
        self.waited = 0

    @property
    def node_state(self):
        """Node states of the most recent batch's buffer set (compatibility)."""
        return self.node_states[(self.count - 1) % 2] if self.count else self.node_states[0]

    def submit(self, alloc_pinned, eps_pinned=None, out_pinned=None) -> StreamBatch:
        torch = self.torch
        if self.count - self.waited >= 2:
            raise RuntimeError("at most two batches in flight: wait() for the oldest first")
        b = self.count % 2
        self.count += 1
        eng = self.engines[b]
        s = int(alloc_pinned.shape[0])
        if out_pinned is None:
            out_pinned = torch.empty((s, self.cap + 1, self.users), dtype=torch.int32,
                                     pin_memory=True)
        main = self.s_main
        main.wait_event(self.free[b])  # the tree of the batch that last used set b is done
        with torch.cuda.stream(main):
            alloc_d = alloc_pinned.to(eng.device, non_blocking=True)
            eps_d = None if eps_pinned is None else eps_pinned.to(eng.device, non_blocking=True)
            eng.run(alloc_d, eps_d, slots=s, stream=main)
            books = torch.cuda.Event()
            books.record(main)
            out_pinned.copy_(eng.codebooks[:s], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(main)
        tree_ready, states = None, None
        if self.with_tree:
            states = self.node_states[b]
            tree_stream = self.s_tree
            tree_stream.wait_event(books)
            _native.check(_native.lib().cyr_tree_expand_device(
                eng.codebooks.data_ptr(), s, self.users, self.cap, self.cell.minislots,
                states.data_ptr(), tree_stream.cuda_stream), "tree")
            tree_ready = torch.cuda.Event()
            tree_ready.record(tree_stream)
            self.free[b].record(tree_stream)
        else:
            self.free[b].record(main)
        return StreamBatch(ready, tree_ready, eng, out_pinned,
                           None if states is None else states[:s], s, (alloc_d, eps_d))

    def wait(self, handle: StreamBatch):
        handle.ready.synchronize()
        self.waited += 1
        eng = handle.engine
        code = int(eng.status[0].item())
        if code:
            with self.torch.cuda.stream(self.s_main):
                eng.status.zero_()
            _native.check(code, "codebook stream")
        return handle.out

    def tree(self, handle: StreamBatch):
        """Block until the batch's arrival tree is written; its node states
        (S, nodes, Ep) int16 on the device."""
        if handle.tree_ready is None:
            raise ValueError("this stream was built with_tree=False")
        handle.tree_ready.synchronize()
        return handle.node_state

    def drain(self):
        """Block until every submitted batch (trees included) has finished."""
        self.s_main.synchronize()
        self.s_tree.synchronize()
