"""Poseidon hot-path ORACLE — plain, slow, obviously-correct CPU implementation (fp64 / exact ints).

*** TEST INFRASTRUCTURE ONLY. ***
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` leg / `--impl reference`
arm may import, call or execute anything under `oracle/`. The product path
(`paper_1706_03292_b200`, `include/`, `csrc/`) never imports it and shares no code with it;
both sides only share the seeded generators in `synth_inputs/` (which hold none of the
method's arithmetic).

Every function cites the PAPER.md passage (`PAPER:<line> §<section>`, /root/reference/PAPER.md)
it restates. Readings of silent/ambiguous points follow SURVEY.md §8(c) S1..S19 and are listed in
DESIGN.md §"Readings".

Modules:
  cost    Table 1 cost formulas (exact Fractions) and Algorithm 1 BestScheme.
  shard   contiguous equal PS shard table (reading S9).
  sync    the updated-weight definitions: SFB (Eq. 2 with per-sample outer products),
          PS (three PS steps through the shard table), WFBP (order independence).
  netsim  message-passing simulator of the PS / SFB / ring exchanges that COUNTS elements
          per node — an independent pin of Table 1 (not a retyping of it).

Parity pins: see tests/test_oracle_*.py. No function here is "parity unpinned".
"""
