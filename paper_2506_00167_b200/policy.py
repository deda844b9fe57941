"""Host-side policy objects: the actor the codebook path evaluates.

Mirrors the reference's policy surface so the drop-in call
``build_codebook(agent, schedule, streams, deterministic)`` accepts either a
``punctsim.sac.SacAgent`` or the ``SacAgent`` defined here:

* ``MlpParams`` / ``init_mlp``  — ``punctsim/neural.py:35-63`` (weights[l] is
  (out_l, in_l) float64, ReLU hidden layers, identity output; He-normal init
  N(0, 2/fan_in), last layer scaled by ``final_scale``, zero biases).
* ``AgentHyper`` / ``SacAgent`` / ``make_agent`` — ``punctsim/sac.py:83-127``
  (actor sizes ``[E+1, *actor_hidden, 2E]``; the actor is drawn FIRST from the
  ``agent-init`` stream, then the two critics, so weights are bit-identical to
  the reference for the same generator state).
* ``load_mlp`` — the ``PSIMMLP1`` checkpoint reader (``neural.py:186-225``),
  SURVEY §8(f) row f3: a pretrained actor can be published straight to the
  device policy.

Only the actor matters to the hot path.  Critics are created so that RNG
consumption and the object shape match the reference; nothing here trains.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

from .core import CellConfig

MLP_MAGIC = b"PSIMMLP1"
MLP_FORMAT_VERSION = 1


@dataclass
class MlpParams:
    """weights[l]: (out_l, in_l) float64; biases[l]: (out_l,)."""

    weights: list
    biases: list

    @property
    def sizes(self) -> list:
        return [self.weights[0].shape[1]] + [w.shape[0] for w in self.weights]

    def copy(self) -> "MlpParams":
        return MlpParams([w.copy() for w in self.weights], [b.copy() for b in self.biases])


def init_mlp(sizes, rng: np.random.Generator, final_scale: float = 1.0) -> MlpParams:
    sizes = [int(s) for s in sizes]
    if len(sizes) < 2:
        raise ValueError("need at least input and output sizes")
    weights, biases = [], []
    last = len(sizes) - 2
    for layer in range(len(sizes) - 1):
        fan_in, fan_out = sizes[layer], sizes[layer + 1]
        std = math.sqrt(2.0 / fan_in)
        if layer == last:
            std *= final_scale
        weights.append(rng.normal(0.0, std, size=(fan_out, fan_in)))
        biases.append(np.zeros(fan_out))
    return MlpParams(weights, biases)


@dataclass(frozen=True)
class AgentHyper:
    discount: float = 0.95
    zeta: float = 0.2
    batch: int = 256
    soft_rate: float = 0.005
    lr: float = 3e-4
    buffer_capacity: int = 20_000
    actor_hidden: tuple = (128,)
    critic_hidden: tuple = (256, 256)
    actor_final_scale: float = 0.01


@dataclass
class SacAgent:
    cell: CellConfig
    cfg: AgentHyper
    actor: MlpParams
    critic1: MlpParams = None
    critic2: MlpParams = None
    target1: MlpParams = None
    target2: MlpParams = None
    extras: dict = field(default_factory=dict)

    @property
    def act_dim(self) -> int:
        return self.cell.num_embb


def actor_sizes(cell, hidden) -> list:
    e = int(cell.num_embb)
    return [e + 1, *[int(h) for h in hidden], 2 * e]


def make_agent(cell, cfg: AgentHyper, rng: np.random.Generator) -> SacAgent:
    e = cell.num_embb
    actor = init_mlp(actor_sizes(cell, cfg.actor_hidden), rng,
                     final_scale=cfg.actor_final_scale)
    critic_sizes = [2 * e + 1, *cfg.critic_hidden, 1]
    c1 = init_mlp(critic_sizes, rng)
    c2 = init_mlp(critic_sizes, rng)
    return SacAgent(cell=cell, cfg=cfg, actor=actor, critic1=c1, critic2=c2,
                    target1=c1.copy(), target2=c2.copy())


def load_mlp(path) -> MlpParams:
    """Read a ``PSIMMLP1`` network (magic, u32 version, u32 n, n×u32 sizes,
    then per layer row-major LE float64 W then b)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:8] != MLP_MAGIC:
        raise ValueError(f"{path}: not a network checkpoint")
    version, n_sizes = struct.unpack_from("<II", blob, 8)
    if version != MLP_FORMAT_VERSION:
        raise ValueError(f"{path}: unsupported format version {version}")
    sizes = struct.unpack_from(f"<{n_sizes}I", blob, 16)
    off = 16 + 4 * n_sizes
    weights, biases = [], []
    for fan_in, fan_out in zip(sizes[:-1], sizes[1:]):
        for shape, dst in (((fan_out, fan_in), weights), ((fan_out,), biases)):
            count = int(np.prod(shape))
            if off + 8 * count > len(blob):
                raise ValueError(f"{path}: checkpoint truncated")
            dst.append(np.frombuffer(blob, "<f8", count, off).reshape(shape).copy())
            off += 8 * count
    if off != len(blob):
        raise ValueError(f"{path}: trailing bytes")
    return MlpParams(weights, biases)


def save_mlp(path, params: MlpParams) -> None:
    sizes = params.sizes
    with open(path, "wb") as fh:
        fh.write(MLP_MAGIC)
        fh.write(struct.pack("<II", MLP_FORMAT_VERSION, len(sizes)))
        fh.write(struct.pack(f"<{len(sizes)}I", *sizes))
        for w, b in zip(params.weights, params.biases):
            fh.write(np.ascontiguousarray(w, "<f8").tobytes())
            fh.write(np.ascontiguousarray(b, "<f8").tobytes())


def flatten_actor(actor) -> tuple[list, np.ndarray]:
    """(sizes, blob): the C-ABI weight layout — per layer W (out,in) row-major
    float64 followed by b (out,), i.e. exactly the PSIMMLP1 payload order."""
    parts = []
    for w, b in zip(actor.weights, actor.biases):
        parts.append(np.ascontiguousarray(w, dtype=np.float64).ravel())
        parts.append(np.ascontiguousarray(b, dtype=np.float64).ravel())
    sizes = [int(actor.weights[0].shape[1])] + [int(w.shape[0]) for w in actor.weights]
    return sizes, np.concatenate(parts)
