"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct fp64 CPU implementation (numpy / scipy) of the
hot path of arXiv 2508.13386's multilevel timestep solver, written from
PAPER.md and the readings of SURVEY.md §8(c) / DESIGN.md.  Every function cites
the passage it follows.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything under `oracle/`.  The product path
(`paper_2508_13386_b200`) never imports it and shares no code with it; both
receive the same inputs from `precompute/` (mesh + basis), which holds none of
the hot path's arithmetic.

Parity pins (tests/test_oracle_*.py) tie every function to the paper or the
mathematics: closed forms, finite differences, invariants, brute force on tiny
inputs and textbook special cases.  Functions without such a pin say
"parity unpinned" in their docstring (also listed in DESIGN.md).
"""
