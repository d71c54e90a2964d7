"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of what Orion's expansion
decode step computes, written from the paper
(§3.3, Alg. 1, Eqs. (1)-(3)) and its reading in
DESIGN.md §"Readings".  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import this package.
The product path (`paper_2510_24390_b200`) never imports it, and it never
imports the product path: they share no code, headers or tables.  The only
common module is `workloads/` (seeded input generators, no method arithmetic).

Parity status (DESIGN.md §"Oracle pins"):
  dag.levels / dag.waves / dag.segment_lists : pinned (paper/SPEC goldens, brute force, invariants)
  bind.bind_segments                          : pinned (masked-pool second oracle, closed forms)
  attention.expand_attn                       : pinned (closed forms, fp64 SDPA equivalences, O3')
  append.kv_append                            : pinned (contiguous-view re-derivation, whole-cache diff)
"""
