"""Device-resident actor policy (the ``policy object`` of the drop-in API).

The reference evaluates ``agent.actor`` (an ``MlpParams`` of float64 numpy
arrays, sac.py:96-127) on every call and mutates it in place during training
(Adam, neural.py:122-141).  Here the actor lives on the GPU as a
``DevicePolicy`` (C handle ``cyr_policy``): weights transposed and cast once
at publish time, re-published with ``update()`` after a change.

``policy_for(agent)`` gives ``build_codebook`` the drop-in behaviour: one
device policy per actor object, and — in the default ``"check"`` sync mode —
an exact comparison of the host weights against the published snapshot on
every call, so an in-place Adam step is never served stale.  Callers that
publish explicitly (serving loops, the benchmark) switch to ``"manual"`` or
pass ``policy=`` and skip that host-side compare.
"""

from __future__ import annotations

import ctypes
import os
import weakref

import numpy as np

from . import _native
from .policy import flatten_actor, load_mlp

_DEFAULT_PRECISION = os.environ.get("CYRUS_PRECISION", "fp32")
_SYNC_MODE = "check"


def set_default_precision(precision: str) -> None:
    global _DEFAULT_PRECISION
    if precision not in _native.PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(_native.PRECISIONS)}")
    _DEFAULT_PRECISION = precision


def default_precision() -> str:
    return _DEFAULT_PRECISION


def set_weight_sync(mode: str) -> None:
    """"check": compare host weights with the published copy on every call;
    "manual": trust the published copy until ``DevicePolicy.update``."""
    global _SYNC_MODE
    if mode not in ("check", "manual"):
        raise ValueError("mode must be 'check' or 'manual'")
    _SYNC_MODE = mode


class DevicePolicy:
    """A published actor: ``sizes = [E+1, *hidden, 2E]`` on the current GPU."""

    def __init__(self, actor=None, precision: str | None = None, *, _handle=None):
        precision = precision or _DEFAULT_PRECISION
        if precision not in _native.PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(_native.PRECISIONS)}")
        self.precision = precision
        lib = _native.lib()
        if _handle is not None:
            self._h = _handle
        else:
            sizes, blob = flatten_actor(actor)
            h = ctypes.c_void_p()
            arr = np.asarray(sizes, dtype=np.int32)
            _native.check(lib.cyr_policy_create(ctypes.byref(h), arr.ctypes.data, len(sizes),
                                                blob.ctypes.data, _native.PRECISIONS[precision]),
                          "policy create")
            self._h = h
        n_users, n_sizes, prec = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _native.check(lib.cyr_policy_info(self._h, ctypes.byref(n_users), ctypes.byref(n_sizes),
                                          ctypes.byref(prec)))
        self.num_users = n_users.value
        self.depth = n_sizes.value - 1

    @classmethod
    def from_checkpoint(cls, path, precision: str | None = None) -> "DevicePolicy":
        """Publish a ``PSIMMLP1`` actor checkpoint (neural.py:186-225) directly."""
        precision = precision or _DEFAULT_PRECISION
        h = ctypes.c_void_p()
        _native.check(_native.lib().cyr_policy_load(ctypes.byref(h), os.fsencode(str(path)),
                                                    _native.PRECISIONS[precision]),
                      f"load {path}")
        return cls(precision=precision, _handle=h)

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("policy is closed")
        return self._h

    @property
    def elem_bytes(self) -> int:
        """Element size of the raw logits (bf16_tc writes fp32 logits)."""
        return 8 if self.precision == "fp64" else 4

    def update(self, actor) -> None:
        """Re-publish after an in-place actor change (same layer sizes)."""
        sizes, blob = flatten_actor(actor)
        if sizes[-1] != 2 * self.num_users or len(sizes) - 1 != self.depth:
            raise ValueError("actor shape differs from the published policy")
        _native.check(_native.lib().cyr_policy_update(self.handle, blob.ctypes.data), "update")

    def quiesce(self) -> None:
        """Stop the resident single-slot server kernel now (it also leaves by
        itself after 20 ms idle); the next drop-in call relaunches it."""
        _native.check(_native.lib().cyr_policy_quiesce(self.handle), "quiesce")

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            try:
                _native.lib().cyr_policy_destroy(self._h)
            finally:
                self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceMlp:
    """Any published ReLU MLP (``cyr_mlp_create``): the SAC critics and
    target critics (sac.py:114-127, sizes [2E+1, *hidden, 1]) for
    ``sac.critic_targets``; forward only (neural.py:66-84)."""

    def __init__(self, params, precision: str | None = None):
        precision = precision or _DEFAULT_PRECISION
        if precision == "bf16_tc":
            precision = "fp32"  # the critics run SIMT (not a codebook decision path)
        if precision not in ("fp32", "fp64"):
            raise ValueError("precision must be fp32 or fp64")
        self.precision = precision
        sizes, blob = flatten_actor(params)
        self.sizes = list(sizes)
        h = ctypes.c_void_p()
        arr = np.asarray(sizes, dtype=np.int32)
        _native.check(_native.lib().cyr_mlp_create(ctypes.byref(h), arr.ctypes.data, len(sizes),
                                                   blob.ctypes.data,
                                                   _native.PRECISIONS[precision]), "mlp create")
        self._h = h

    @classmethod
    def from_checkpoint(cls, path, precision: str | None = None) -> "DeviceMlp":
        """Publish a PSIMMLP1 network file (a critic / target critic of an
        agent directory, sac.py:374-393) through the C loader."""
        precision = precision or _DEFAULT_PRECISION
        if precision == "bf16_tc":
            precision = "fp32"
        h = ctypes.c_void_p()
        _native.check(_native.lib().cyr_mlp_load(ctypes.byref(h), os.fsencode(str(path)),
                                                 _native.PRECISIONS[precision]), f"load {path}")
        self = cls.__new__(cls)
        self.precision = precision
        self._h = h
        self.sizes = list(load_mlp(path).sizes)
        return self

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("mlp is closed")
        return self._h

    def update(self, params) -> None:
        sizes, blob = flatten_actor(params)
        if list(sizes) != self.sizes:
            raise ValueError("MLP shape differs from the published one")
        _native.check(_native.lib().cyr_policy_update(self.handle, blob.ctypes.data), "update")

    def forward(self, x, out=None, stream=None):
        """x: CUDA float64 (cols, in) -> (cols, out) CUDA tensor (fp32/fp64)."""
        import torch
        x = x.contiguous()
        if x.dtype != torch.float64 or x.dim() != 2 or x.shape[1] != self.sizes[0]:
            raise ValueError("input must be float64 (cols, input_dim)")
        dt = torch.float64 if self.precision == "fp64" else torch.float32
        if out is None:
            out = torch.empty((x.shape[0], self.sizes[-1]), dtype=dt, device=x.device)
        _native.check(_native.lib().cyr_mlp_forward_device(
            self.handle, x.data_ptr(), x.shape[0], out.data_ptr(),
            _native.stream_handle(stream)), "mlp forward")
        return out

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            try:
                _native.lib().cyr_policy_destroy(self._h)
            finally:
                self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Published:
    """A published actor (or MLP) and how its host weights are watched."""

    __slots__ = ("policy", "actor_ref", "arrays", "watched", "snapshot")

    def __init__(self, actor, policy):
        self.policy = policy
        self.actor_ref = weakref.ref(actor)
        self.arrays = None      # the registered host arrays (identity + keep-alive)
        self.watched = False    # registered with cyr_policy_watch (C-side compare)
        self.snapshot = None    # Python-side snapshot for arrays C cannot watch


def _arrays(actor) -> list:
    out = []
    for w, b in zip(actor.weights, actor.biases):
        out.append(w)
        out.append(b)
    return out


def _watchable(arrays) -> bool:
    return all(isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
               for a in arrays)


def _snapshot(arrays):
    return [a.copy() for a in arrays]


def _same(arrays, snap) -> bool:
    return len(arrays) == len(snap) and all(
        a.shape == s.shape and np.array_equal(a, s) for a, s in zip(arrays, snap))


def _watch(entry, arrays) -> None:
    """Register the host arrays with the C library (publishes them now);
    from then on every cyr_codebook_host call compares them with the
    published snapshot while the device computes (include/cyrus_b200.h)."""
    lib = _native.lib()
    if _watchable(arrays):
        n = len(arrays)
        ptrs = (ctypes.c_void_p * n)(*[a.ctypes.data for a in arrays])
        counts = np.asarray([a.size for a in arrays], dtype=np.int64)
        _native.check(lib.cyr_policy_watch(entry.policy.handle, ptrs, counts.ctypes.data, n),
                      "weight watch")
        entry.watched, entry.snapshot = True, None
    else:  # e.g. float32 or strided arrays: compare on the host instead
        if entry.watched:
            _native.check(lib.cyr_policy_watch(entry.policy.handle, None, None, 0))
        entry.policy.update(_Params(arrays))
        entry.watched, entry.snapshot = False, _snapshot(arrays)
    entry.arrays = tuple(arrays)


class _Params:
    def __init__(self, arrays):
        self.weights, self.biases = list(arrays[0::2]), list(arrays[1::2])


def _sync(entry, actor, deferred: bool) -> None:
    """"check" mode: the device copy follows in-place host updates.  Array
    identity is checked here (cheap); contents are compared in C — inside
    the codebook call itself when ``deferred`` (overlapped with the device
    work), else now (cyr_policy_sync)."""
    arrays = _arrays(actor)
    reg = entry.arrays
    if reg is None or len(reg) != len(arrays) or any(a is not b for a, b in zip(arrays, reg)):
        _watch(entry, arrays)
    elif entry.watched:
        if not deferred:
            _native.check(_native.lib().cyr_policy_sync(entry.policy.handle, None), "weight sync")
    elif not _same(arrays, entry.snapshot):
        entry.policy.update(_Params(arrays))
        entry.snapshot = _snapshot(arrays)


def _unwatch(entry) -> None:
    if entry.watched:
        _native.check(_native.lib().cyr_policy_watch(entry.policy.handle, None, None, 0))
    entry.watched, entry.arrays, entry.snapshot = False, None, None


_PUBLISHED: dict = {}


def _lookup(table, params, precision, make, deferred):
    key = (id(params), precision)
    entry = table.get(key)
    if entry is None or entry.actor_ref() is not params:
        entry = _Published(params, make(params, precision))
        table[key] = entry
        weakref.finalize(params, table.pop, key, None)
        if _SYNC_MODE == "check":
            _watch(entry, _arrays(params))
    elif _SYNC_MODE == "check":
        _sync(entry, params, deferred)
    elif entry.watched:
        _unwatch(entry)
    return entry.policy


def fast_entry(actor, precision: str | None = None):
    """The published entry of ``actor`` when the drop-in call can skip
    ``policy_for`` ("check" mode with the arrays registered in C): the C
    fast path then checks the arrays' identity itself.  None otherwise."""
    e = _PUBLISHED.get((id(actor), precision or _DEFAULT_PRECISION))
    if e is None or not e.watched or _SYNC_MODE != "check" or e.actor_ref() is not actor:
        return None
    return e


def policy_for(agent, precision: str | None = None, *, deferred: bool = False) -> DevicePolicy:
    """Device policy for ``agent.actor`` (published on first use).  In the
    default "check" mode the device copy follows in-place host updates
    (Adam, neural.py:122-141).  ``deferred``: the caller's next call is
    ``cyr_codebook_host``, which compares the weights itself while the
    device computes (build_codebook)."""
    return _lookup(_PUBLISHED, agent.actor, precision or _DEFAULT_PRECISION, DevicePolicy,
                   deferred)


_PUBLISHED_MLP: dict = {}


def mlp_for(params, precision: str | None = None) -> DeviceMlp:
    """Device copy of any MlpParams (e.g. ``agent.target1``), published on
    first use and kept in sync with in-place changes in "check" mode."""
    return _lookup(_PUBLISHED_MLP, params, precision or _DEFAULT_PRECISION, DeviceMlp, False)


def publish(agent, precision: str | None = None) -> DevicePolicy:
    """Force a re-publish of ``agent.actor`` (use after training steps in
    "manual" sync mode)."""
    policy = policy_for(agent, precision)
    policy.update(agent.actor)
    return policy


def quiesce_all() -> None:
    """Stop every resident slot server of the process (before a device-wide
    ``torch.cuda.synchronize()`` that should not wait for their idle exit)."""
    _native.check(_native.lib().cyr_quiesce_all(), "quiesce")
