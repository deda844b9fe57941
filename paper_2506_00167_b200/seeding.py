"""Named RNG substreams (contract of ``punctsim/seeding.py:19-27``).

A substream is ``default_rng(SeedSequence([seed, h(name), *idx]))`` where
``h`` is the little-endian integer of the first 8 bytes of SHA-256(name).
Branch noise for codebook column j comes from ``substream(seed,
"policy-branch", j)`` (``engine.py:76-77``); the hot path draws it on the
host before launch so the device never needs the generator state.
"""

from __future__ import annotations

import hashlib

import numpy as np

_U64 = (1 << 64) - 1


def name_hash(name: str) -> int:
    return int.from_bytes(hashlib.sha256(name.encode("utf-8")).digest()[:8], "little")


def substream(master_seed: int, name: str, *indices: int) -> np.random.Generator:
    words = [int(master_seed) & _U64, name_hash(name)]
    words += [int(i) & _U64 for i in indices]
    return np.random.default_rng(np.random.SeedSequence(words))
