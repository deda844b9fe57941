"""Access to tests/golden/reference_golden.npz (made by make_golden.py from
the unmodified reference) plus regeneration of the reference's actors."""

from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass

import numpy as np

from paper_2506_00167_b200.core import CellConfig
from paper_2506_00167_b200.policy import AgentHyper, make_agent
from paper_2506_00167_b200.seeding import substream

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")


def weights_digest(actor) -> str:
    h = hashlib.sha256()
    for w, b in zip(actor.weights, actor.biases):
        h.update(np.ascontiguousarray(w, "<f8").tobytes())
        h.update(np.ascontiguousarray(b, "<f8").tobytes())
    return h.hexdigest()


@dataclass
class Config:
    name: str
    meta: dict
    data: dict

    @property
    def cell(self):
        m = self.meta
        return CellConfig(total_scs=m["total_scs"], num_embb=m["num_embb"],
                          urllc_sc_len=m["urllc_sc_len"], minislots=m["minislots"], rb_size=12)

    def agent(self):
        m = self.meta
        hyper = AgentHyper(actor_hidden=tuple(m["actor_hidden"]),
                           actor_final_scale=m["final_scale"])
        agent = make_agent(self.cell, hyper, substream(m["seed"], "agent-init"))
        assert weights_digest(agent.actor) == m["weights_sha256"], "actor differs from reference"
        return agent

    def __getitem__(self, key):
        return self.data[f"{self.name}/{key}"]


class Golden:
    def __init__(self, npz):
        self.npz = npz
        self.meta = json.loads(str(npz["meta_json"]))
        self._cache = {}

    @classmethod
    def load(cls):
        return cls(dict(np.load(PATH)))

    def config(self, name) -> Config:
        return Config(name, self.meta[name], self.npz)

    @property
    def names(self):
        return sorted(self.meta)

    def enforcer_groups(self):
        """Yield (b, caps, demand, m_hat, nu, degenerate, grants) per group."""
        z = self.npz
        r0 = 0
        for rows, width in zip(z["enf/rows"], z["enf/width"]):
            sl = slice(r0, r0 + int(rows))
            r0 += int(rows)
            yield (z["enf/b"][sl, :width], z["enf/caps"][sl, :width], z["enf/demand"][sl],
                   z["enf/m_hat"][sl, :width], z["enf/nu"][sl], z["enf/degenerate"][sl],
                   z["enf/grants"][sl, :width])


CRITIC_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                           "critic_golden.npz")


@dataclass
class CriticCase:
    """One sac.critic_targets fixture (make_critic_golden.py)."""
    name: str
    meta: dict
    data: dict

    @property
    def cell(self):
        m = self.meta
        return CellConfig(total_scs=m["total_scs"], num_embb=m["num_embb"],
                          urllc_sc_len=m["urllc_sc_len"], minislots=m["minislots"], rb_size=12)

    def agent(self):
        m = self.meta
        hyper = AgentHyper(actor_hidden=tuple(m["actor_hidden"]),
                           actor_final_scale=m["final_scale"])
        agent = make_agent(self.cell, hyper, substream(m["seed"], "agent-init"))
        assert weights_digest(agent.actor) == m["actor_sha256"]
        assert weights_digest(agent.target1) == m["target1_sha256"]
        assert weights_digest(agent.target2) == m["target2_sha256"]
        return agent

    def arrays(self):
        e = self.meta["num_embb"]
        k = self["k"]
        return (self["alloc"], k, np.zeros(k.shape + (e,)), self["reward"])

    def rng(self):
        return np.random.default_rng(self.meta["rng_seed"])

    def __getitem__(self, key):
        return self.data[f"{self.name}/{key}"]


def critic_cases():
    z = dict(np.load(CRITIC_PATH))
    meta = json.loads(str(z["meta_json"]))
    return [CriticCase(n, meta[n], z) for n in sorted(meta)]
