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
    adam_actor: "AdamState" = None     # optimiser states (sac.py:106-108; checkpoints only)
    adam_c1: "AdamState" = None
    adam_c2: "AdamState" = None
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
                    target1=c1.copy(), target2=c2.copy(), adam_actor=AdamState.zeros_like(actor),
                    adam_c1=AdamState.zeros_like(c1), adam_c2=AdamState.zeros_like(c2))


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


ADAM_MAGIC = b"PSIMADM1"


@dataclass
class AdamState:
    """Adam moments per parameter (neural.py:87-121); checkpointed, not used
    by the codebook path."""

    m_w: list
    v_w: list
    m_b: list
    v_b: list
    t: int = 0

    @classmethod
    def zeros_like(cls, params: MlpParams) -> "AdamState":
        return cls([np.zeros_like(w) for w in params.weights],
                   [np.zeros_like(w) for w in params.weights],
                   [np.zeros_like(b) for b in params.biases],
                   [np.zeros_like(b) for b in params.biases], 0)


def save_adam(path, state: AdamState, sizes) -> None:
    """``PSIMADM1``: magic, u32 version, u32 n, n×u32 sizes, u64 step, then
    m_w, v_w, m_b, v_b (row-major LE float64) — neural.py:228-236."""
    sizes = [int(x) for x in sizes]
    with open(path, "wb") as fh:
        fh.write(ADAM_MAGIC)
        fh.write(struct.pack("<II", MLP_FORMAT_VERSION, len(sizes)))
        fh.write(struct.pack(f"<{len(sizes)}I", *sizes))
        fh.write(struct.pack("<Q", int(state.t)))
        for group in (state.m_w, state.v_w, state.m_b, state.v_b):
            for arr in group:
                fh.write(np.ascontiguousarray(arr, "<f8").tobytes())


def load_adam(path, sizes) -> AdamState:
    """Read a ``PSIMADM1`` optimiser state (neural.py:239-259), with the
    reference's checks and messages."""
    sizes = [int(x) for x in sizes]
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:8] != ADAM_MAGIC:
        raise ValueError(f"{path}: not an optimiser checkpoint")
    version, n_sizes = struct.unpack_from("<II", blob, 8)
    if version != MLP_FORMAT_VERSION:
        raise ValueError(f"{path}: unsupported format version {version}")
    stored = list(struct.unpack_from(f"<{n_sizes}I", blob, 16))
    if stored != sizes:
        raise ValueError(f"{path}: layer sizes do not match network")
    off = 16 + 4 * n_sizes
    (t,) = struct.unpack_from("<Q", blob, off)
    off += 8
    w_shapes = [(o, i) for i, o in zip(sizes[:-1], sizes[1:])]
    b_shapes = [(o,) for o in sizes[1:]]
    groups = []
    for shapes in (w_shapes, w_shapes, b_shapes, b_shapes):
        arrs = []
        for shape in shapes:
            count = int(np.prod(shape))
            if off + 8 * count > len(blob):
                raise ValueError("checkpoint truncated")
            arrs.append(np.frombuffer(blob, "<f8", count, off).reshape(shape).copy())
            off += 8 * count
        groups.append(arrs)
    if off != len(blob):
        raise ValueError(f"{path}: trailing bytes")
    return AdamState(*groups, t=int(t))


NET_FILES = ("actor", "critic1", "critic2", "target1", "target2")


def save_agent(directory, agent) -> None:
    """One PSIMMLP1 file per network plus three PSIMADM1 optimiser states
    (sac.py:361-371)."""
    from pathlib import Path
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    nets = (agent.actor, agent.critic1, agent.critic2, agent.target1, agent.target2)
    for name, net in zip(NET_FILES, nets):
        save_mlp(directory / f"{name}.net", net)
    for name, attr, net in (("actor", "adam_actor", agent.actor),
                            ("critic1", "adam_c1", agent.critic1),
                            ("critic2", "adam_c2", agent.critic2)):
        state = getattr(agent, attr, None) or AdamState.zeros_like(net)
        save_adam(directory / f"{name}.adam", state, net.sizes)


def load_agent_host(directory, cell, cfg: AgentHyper) -> SacAgent:
    """sac.load_agent (sac.py:374-393) on the host: the five networks with
    the reference's presence and shape checks, and the optimiser states."""
    from pathlib import Path
    directory = Path(directory)
    nets = {}
    for name in NET_FILES:
        path = directory / f"{name}.net"
        if not path.exists():
            raise FileNotFoundError(f"checkpoint file missing: {path}")
        nets[name] = load_mlp(path)
    e = cell.num_embb
    if nets["actor"].sizes[0] != e + 1 or nets["actor"].sizes[-1] != 2 * e:
        raise ValueError("actor checkpoint does not match cell dimensions")
    if nets["critic1"].sizes[0] != 2 * e + 1:
        raise ValueError("critic checkpoint does not match cell dimensions")
    agent = SacAgent(cell=cell, cfg=cfg, actor=nets["actor"], critic1=nets["critic1"],
                     critic2=nets["critic2"], target1=nets["target1"], target2=nets["target2"])
    agent.adam_actor = load_adam(directory / "actor.adam", nets["actor"].sizes)
    agent.adam_c1 = load_adam(directory / "critic1.adam", nets["critic1"].sizes)
    agent.adam_c2 = load_adam(directory / "critic2.adam", nets["critic2"].sizes)
    return agent


def flatten_actor(actor) -> tuple[list, np.ndarray]:
    """(sizes, blob): the C-ABI weight layout — per layer W (out,in) row-major
    float64 followed by b (out,), i.e. exactly the PSIMMLP1 payload order."""
    parts = []
    for w, b in zip(actor.weights, actor.biases):
        parts.append(np.ascontiguousarray(w, dtype=np.float64).ravel())
        parts.append(np.ascontiguousarray(b, dtype=np.float64).ravel())
    sizes = [int(actor.weights[0].shape[1])] + [int(w.shape[0]) for w in actor.weights]
    return sizes, np.concatenate(parts)
