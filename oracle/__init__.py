"""TEST INFRASTRUCTURE — CPU oracle for the codebook hot path.

This package restates, in float64 numpy, the reference algorithm of the RT
O-DU codebook path (``punctsim.engine.build_codebook`` and its callees,
``/root/reference/pkg/src/punctsim/{engine,sac,neural,enforcer}.py``).  It is
the CHECKER, never the product:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the shipped package ``paper_2506_00167_b200`` never imports it and fails
  loudly when its CUDA library is missing.

Parity pinning: ``tests/golden/make_golden.py`` runs the unmodified reference
(importable in the build container) and freezes its outputs; the
``-m "not gpu"`` suite checks this oracle against those fixtures bit for bit
(codebooks, grants, m_hat, nu) and against the reference's own known-answer
tests (``pkg/tests/test_enforcer.py``).

Modules:
  projection   — KL water-filling + Huntington-Hill (enforcer.py:49-165, 201-207)
  mlp          — actor forward + tanh-Gaussian head (neural.py:25-84, 144-183;
                 sac.py:334-355)
  slot         — one slot's codebook (engine.py:97-116), batched over slots
  pf           — proportional-fair scheduler (scheduler.py:79-106; §8(f) f4)
  leaf_score   — threshold decode + reward at every tree leaf (§8(f) f2)
  critic       — SAC critic targets (sac.py:167-214)
  arrival_tree — Mode-R arrival tree node states (no
                 reference counterpart: composition of engine.py:230 lookups)
"""
