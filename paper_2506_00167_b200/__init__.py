"""B200-native RT O-DU puncturing-codebook path (Cyrus+, arXiv 2506.00167).

Drop-in for ``punctsim.engine.build_codebook`` and its callees; see
DESIGN.md.  The CUDA library (``libcyrus_b200.so``) is loaded on first use;
there is no CPU fallback.
"""

from .core import CellConfig, PuncturingVector, ScheduleVector
from .device import DevicePolicy, policy_for, publish, set_default_precision, set_weight_sync
from .engine import (
    Codebook,
    CodebookEngine,
    CodebookStream,
    Streams,
    build_codebook,
    build_codebooks_host,
    draw_branch_noise,
    make_streams,
)
from ._native import InfeasibleDemandError, NativeLibraryError
from .policy import AgentHyper, MlpParams, SacAgent, init_mlp, load_mlp, make_agent, save_mlp
from .seeding import substream

__all__ = [
    "AgentHyper", "CellConfig", "Codebook", "CodebookEngine", "CodebookStream", "DevicePolicy",
    "InfeasibleDemandError", "MlpParams", "NativeLibraryError", "PuncturingVector",
    "SacAgent", "ScheduleVector", "Streams", "build_codebook", "build_codebooks_host",
    "draw_branch_noise", "init_mlp", "load_mlp", "make_agent", "make_streams", "policy_for",
    "publish", "save_mlp", "set_default_precision", "set_weight_sync", "substream",
]
