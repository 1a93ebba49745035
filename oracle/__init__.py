"""CPU oracle for the DASO hot path (arXiv 2104.05588) — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct numpy fp64 implementation of what the GPU path
computes, written from /root/reference/PAPER.md (cited as ``P:<line>``) and
the readings listed in DESIGN.md §3 (R1..R21).  It simulates every one of the
W = P*G ranks of a virtual cluster explicitly in one process.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2104_05588_b200``) never imports it and shares no code with it; the
only shared module is ``synthetic`` (seeded random inputs, no method arithmetic).

Modules
  topology  — rank map, node groups, global groups, rotation
  numerics  — average, Eq. (1) weighted stale average, bf16 RNE
  sgd       — momentum-SGD local optimizer step
  schedule  — warm-up / cycling / cool-down, B/S halving and reset
  daso_sim  — the per-batch DASO step over all ranks
  toy       — linear-regression model used by the toy config
  bench     — times the oracle as-is for bench.py's cpu_baseline

Pins: every function here is checked by ``tests/test_oracle_*.py`` against
values / identities fixed by the paper or by mathematics (see the test module
docstrings and DESIGN.md §4).  Nothing here is "parity unpinned" except where a
docstring says so explicitly.
"""
