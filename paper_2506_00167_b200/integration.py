"""Patching the reference package onto the B200 path.

``patch_punctsim(punctsim)`` applies the maintainer patch of INTEGRATION.md
to an imported, unmodified ``punctsim``:

* ``punctsim.engine.build_codebook`` (engine.py:97-116) -> this package's
  ``build_codebook`` (actor + projection on the GPU), returning the
  reference's own ``punctsim.engine.Codebook`` so every caller — ``run_tti``
  (engine.py:227-230), ``acl_pretrain`` (engine.py:344-345), the CLI — is
  untouched;
* optionally ``punctsim.sac.critic_targets`` (sac.py:167-214) -> the GPU
  ``sac.critic_targets`` (``critic_targets=True``).

The reference's objects (``SacAgent``, ``ScheduleVector``, ``Streams``) are
passed through as they are; branch noise is drawn from the reference's own
generators, so seeded runs stay byte-identical.  Returns a callable that
restores the original functions.
"""

from __future__ import annotations

from . import engine as _engine
from . import sac as _sac


def patch_punctsim(punctsim, precision: str | None = None, critic_targets: bool = False):
    eng = punctsim.engine
    ref_codebook = eng.Codebook
    original_build = eng.build_codebook

    def build_codebook(agent, schedule, streams, deterministic=False):
        cb = _engine.build_codebook(agent, schedule, streams, deterministic,
                                    precision=precision)
        return ref_codebook(columns=cb.columns, gen_ns=cb.gen_ns)

    build_codebook.__doc__ = original_build.__doc__
    eng.build_codebook = build_codebook
    restore = [(eng, "build_codebook", original_build)]
    if critic_targets:
        sac = punctsim.sac
        original_targets = sac.critic_targets

        def targets(agent, arrays, rng):
            return _sac.critic_targets(agent, arrays, rng, precision=precision)

        targets.__doc__ = original_targets.__doc__
        sac.critic_targets = targets
        restore.append((sac, "critic_targets", original_targets))

    def undo():
        for mod, name, fn in restore:
            setattr(mod, name, fn)

    return undo
