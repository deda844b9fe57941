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
    __slots__ = ("policy", "snapshot", "actor_ref")

    def __init__(self, actor, policy):
        self.policy = policy
        self.actor_ref = weakref.ref(actor)
        self.snapshot = _snapshot(actor)


def _snapshot(actor):
    return [w.copy() for w in actor.weights] + [b.copy() for b in actor.biases]


def _same(actor, snap) -> bool:
    arrays = list(actor.weights) + list(actor.biases)
    if len(arrays) != len(snap):
        return False
    return all(a.shape == s.shape and np.array_equal(a, s) for a, s in zip(arrays, snap))


_PUBLISHED: dict = {}


def policy_for(agent, precision: str | None = None) -> DevicePolicy:
    """Device policy for ``agent.actor`` (published on first use)."""
    precision = precision or _DEFAULT_PRECISION
    actor = agent.actor
    key = (id(actor), precision)
    entry = _PUBLISHED.get(key)
    if entry is None or entry.actor_ref() is not actor:
        entry = _Published(actor, DevicePolicy(actor, precision))
        _PUBLISHED[key] = entry
        weakref.finalize(actor, _PUBLISHED.pop, key, None)
    elif _SYNC_MODE == "check" and not _same(actor, entry.snapshot):
        entry.policy.update(actor)
        entry.snapshot = _snapshot(actor)
    return entry.policy


_PUBLISHED_MLP: dict = {}


def mlp_for(params, precision: str | None = None) -> DeviceMlp:
    """Device copy of any MlpParams (e.g. ``agent.target1``), published on
    first use and re-published after an in-place change in "check" mode."""
    precision = precision or _DEFAULT_PRECISION
    key = (id(params), precision)
    entry = _PUBLISHED_MLP.get(key)
    if entry is None or entry.actor_ref() is not params:
        entry = _Published(params, DeviceMlp(params, precision))
        _PUBLISHED_MLP[key] = entry
        weakref.finalize(params, _PUBLISHED_MLP.pop, key, None)
    elif _SYNC_MODE == "check" and not _same(params, entry.snapshot):
        entry.policy.update(params)
        entry.snapshot = _snapshot(params)
    return entry.policy


def publish(agent, precision: str | None = None) -> DevicePolicy:
    """Force a re-publish of ``agent.actor`` (use after training steps in
    "manual" sync mode)."""
    policy = policy_for(agent, precision)
    key = (id(agent.actor), precision or _DEFAULT_PRECISION)
    policy.update(agent.actor)
    _PUBLISHED[key].snapshot = _snapshot(agent.actor)
    return policy
