"""ORACLE -- TEST INFRASTRUCTURE ONLY (plain, slow, fp64).

A direct CPU implementation of what the hot path computes, written from the
paper (PAPER.md, arXiv 2402.15322).  It shares no code with the CUDA path in
paper_2402_15322_b200/ and neither imports the other.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it.  Inputs come from se2_synth (no method arithmetic there).

Citations: P:n = /root/reference/PAPER.md line n (+ the equation label).
Readings of silent/garbled passages are DESIGN.md "Readings" R1..R12.

Parity pins: every function below is pinned in tests/test_oracle_pins.py
against closed forms, worked values, brute force or invariants; see DESIGN.md
"Oracle pins".  Whole runs at full config scale are "parity unpinned" beyond
those pins (the paper prints no worked numbers for them).
"""
from .se2_oracle import *  # noqa: F401,F403
from . import se2_lift  # noqa: F401  (lifting / projection)
