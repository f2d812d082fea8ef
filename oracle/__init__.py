"""CPU oracle for the PI²-RH control step — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference ``pimpc`` algorithm for the
hot path named by BASELINE.json's north star: noise addressing
(``rng.py``), the frozen float32 LWPR fast path (``lwpr.py:329-407``), the
chunked rollout engine (``controller.py:142-322``), the cost plugin
(``simworld.py:133-198``) and the path-integral update / optimisation
loop (``controller.py:356-413``).  Every function cites the reference
file:line it follows (paths relative to the reference ``pkg/src/pimpc``).

Who may use it: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs — as the
checker or the timed CPU baseline, never as the product.  The product
package ``paper_1503_00330_b200`` never imports it and has no CPU fallback.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(importable in the build container only) on seeded inputs and commits the
outputs as ``tests/golden/*.npz``; ``tests/test_oracle.py`` checks this
restatement against them (bitwise on the generating machine's numpy build).

Deliberate deviation from the reference: cost-plugin scratch buffers are
per call, not shared per shape (``simworld.py:149-155`` hands the same
buffers to every worker thread, a data race when workers > 1 — SURVEY.md
§0.3).  With one worker the two are bitwise identical.
"""
