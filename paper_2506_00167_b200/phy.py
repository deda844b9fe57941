"""Erasure-LDPC decodability on the GPU.

The reference's "erasure_ldpc" model (phy.py:83-213) treats a user's TTI
transport as a regular (dv, dc) LDPC codeword of n = M * n_e symbols
(symbol sc*M + tau), erases the punctured symbols (the first m_tau SCs of
mini-slot tau) and the channel-erased ones, and decodes by peeling.  Here:

* ``LdpcCode`` builds the same graph as phy.LdpcCode (configuration model
  seeded by SeedSequence([seed, n, dv, dc]), then parallel-edge repair by
  random socket swaps), with the same numpy random stream, so the edge lists
  are identical; it is published to the device once;
* ``DecodabilityModel.code_for`` pads and caches codes like phy.py:169-179;
* ``peel_decode_batch(code, erased)`` decodes B erasure patterns at once on
  the GPU (``cyr_ldpc_peel_device``, one CTA per pattern), equal to
  phy.peel_decode pattern by pattern;
* ``puncture_mask`` builds the punctured symbols of decode_user
  (phy.py:204-208).
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

from . import _native


def degree_pair(code_rate: float) -> tuple:
    """Smallest regular (dv, dc), dv >= 3, with 1 - dv/dc = rate (phy.py:146-151)."""
    frac = Fraction(1.0 - code_rate).limit_denominator(64)
    p, q = frac.numerator, frac.denominator
    k = max(1, math.ceil(3 / p))
    return p * k, q * k


class LdpcCode:
    """Regular (dv, dc) parity graph over n symbols (phy.py:83-120), plus its
    device copy (``edge_var`` / ``edge_check`` int32)."""

    def __init__(self, n: int, dv: int, dc: int, seed: int):
        if (n * dv) % dc != 0:
            raise ValueError("dv*n must be divisible by dc")
        self.n, self.dv, self.dc, self.seed = int(n), int(dv), int(dc), int(seed)
        self.n_checks = self.n * self.dv // self.dc
        rng = np.random.default_rng(np.random.SeedSequence([seed, n, dv, dc]))
        sockets = np.repeat(np.arange(self.n), self.dv)
        self.edge_var = sockets[rng.permutation(self.n * self.dv)]
        self.edge_check = np.repeat(np.arange(self.n_checks), self.dc)
        self._make_simple(rng)
        self._device = None

    def _make_simple(self, rng, max_rounds: int = 10_000):
        """Swap the variable socket of every repeated (check, variable) edge
        with a random edge until the graph is simple."""
        edges = self.edge_var.size
        for _ in range(max_rounds):
            key = self.edge_check.astype(np.int64) * self.n + self.edge_var
            order = np.argsort(key, kind="stable")
            repeated = order[np.flatnonzero(np.diff(key[order]) == 0) + 1]
            if repeated.size == 0:
                return
            for p in repeated:
                q = int(rng.integers(edges))
                self.edge_var[p], self.edge_var[q] = self.edge_var[q], self.edge_var[p]
        raise RuntimeError("parallel edge repair did not converge")

    @property
    def rate(self) -> float:
        return 1.0 - self.dv / self.dc

    def device(self):
        import torch
        if self._device is None:
            self._device = (torch.from_numpy(self.edge_var.astype(np.int32)).cuda(),
                            torch.from_numpy(self.edge_check.astype(np.int32)).cuda())
        return self._device


class DecodabilityModel:
    """The erasure_ldpc model's code cache (phy.py:153-179)."""

    def __init__(self, code_seed: int = 0):
        self.code_seed = int(code_seed)
        self._codes: dict = {}

    def code_for(self, n_symbols: int, code_rate: float) -> LdpcCode:
        dv, dc = degree_pair(code_rate)
        step = dc // math.gcd(dv, dc)
        n_padded = ((n_symbols + step - 1) // step) * step
        key = (n_padded, round(code_rate, 9))
        code = self._codes.get(key)
        if code is None:
            code = LdpcCode(n_padded, dv, dc, self.code_seed)
            self._codes[key] = code
        return code


def puncture_mask(code: LdpcCode, punctures, minislots: int) -> np.ndarray:
    """Erased symbols of decode_user (phy.py:204-208): symbol sc*M + tau for
    the first m_tau SCs of mini-slot tau; padding symbols are never erased."""
    erased = np.zeros(code.n, dtype=bool)
    for tau, m in enumerate(punctures):
        if m:
            erased[np.arange(int(m)) * minislots + tau] = True
    return erased


def peel_decode_batch(code: LdpcCode, erased, stream=None) -> np.ndarray:
    """phy.peel_decode for every row of ``erased`` (B, n) bool: True where
    peeling recovers every erasure.  One GPU launch for the batch."""
    import torch
    erased = np.ascontiguousarray(erased, dtype=np.uint8)
    if erased.ndim != 2 or erased.shape[1] != code.n:
        raise ValueError("erasure mask length mismatch")
    b = erased.shape[0]
    if b == 0:
        return np.zeros(0, dtype=bool)
    ev, ec = code.device()
    er = torch.from_numpy(erased).cuda()
    ok = torch.empty(b, dtype=torch.uint8, device="cuda")
    _native.check(_native.lib().cyr_ldpc_peel_device(
        ev.data_ptr(), ec.data_ptr(), code.n, code.n_checks, int(ev.numel()), er.data_ptr(), b,
        ok.data_ptr(), _native.stream_handle(stream)), "peel_decode_batch")
    return ok.cpu().numpy().astype(bool)


def peel_decode_counts(code: LdpcCode, counts, n_e: int, minislots: int, stream=None):
    """Peeling verdicts for B puncture patterns of one user given as
    per-mini-slot counts (B, M) (decode_user's layout, clean channel); the
    erasure masks are formed on the device.  Returns (B,) bool."""
    import torch
    counts = np.ascontiguousarray(counts, dtype=np.int32)
    if counts.ndim != 2 or counts.shape[1] != minislots:
        raise ValueError("counts must be (B, M)")
    if minislots * n_e > code.n:
        raise ValueError("codeword shorter than M * n_e")
    b = counts.shape[0]
    if b == 0:
        return np.zeros(0, dtype=bool)
    ev, ec = code.device()
    cd = torch.from_numpy(counts).cuda()
    ok = torch.empty(b, dtype=torch.uint8, device="cuda")
    _native.check(_native.lib().cyr_ldpc_peel_counts_device(
        ev.data_ptr(), ec.data_ptr(), code.n, code.n_checks, int(ev.numel()), cd.data_ptr(),
        minislots, minislots * n_e, b, ok.data_ptr(), _native.stream_handle(stream)),
        "peel_decode_counts")
    return ok.cpu().numpy().astype(bool)


def leaf_decode_ldpc(codebook, alloc, code_rates, minislots: int, model: DecodabilityModel):
    """Every leaf of one slot's arrival tree under the erasure_ldpc model with
    a clean channel: (leaves, E) bool, leaf q = the admitted counts of its
    base-(cap+1) digits (first mini-slot first), user e decoding its
    punctures codebook[k_tau][e] per mini-slot (decode_user,
    phy.py:188-213).  Each user's distinct patterns are decoded once, in one
    GPU batch."""
    book = np.asarray(codebook, dtype=np.int64)
    r, users = book.shape
    digits = np.stack(np.unravel_index(np.arange(r ** minislots), (r,) * minislots), axis=1)
    ok = np.ones((r ** minislots, users), dtype=bool)
    for e in range(users):
        n_e = int(alloc[e])
        if n_e <= 0:
            continue  # decode_user: no allocation decodes
        per_slot = book[digits, e]                           # (leaves, M)
        pats, inverse = np.unique(per_slot, axis=0, return_inverse=True)
        code = model.code_for(minislots * n_e, float(code_rates[e]))
        ok[:, e] = peel_decode_counts(code, pats, n_e, minislots)[inverse.ravel()]
    return ok
