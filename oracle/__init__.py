"""CPU oracle for Crossover-SGD's segment-wise gossip round (arXiv 2012.15198).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import or execute
anything under `oracle/`.  The product path (the C-ABI library under
`paper_2012_15198_b200/`) never imports it and shares no code with it.

Plain, slow, obviously-correct NumPy/pure-Python restatements of the paper:

  philox.py     Philox4x32-10 counter-based RNG (Salmon et al., SC'11) — the
                draw primitive of the topology reading C-4.
  topology.py   PAPER.md:165-191 (§3.2, Alg. 2) load-balanced random topology,
                with readings C-1, C-4..C-7; segment plan (C-2).
  gossip.py     PAPER.md:120-155 (§3.1, Alg. 1) segment-wise exchange + merge
                l.17, preceded by the local momentum-SGD update (PAPER.md:122,
                reading C-8/C-9); push-sum weights (reading C-11).
  hierarchical.py  PAPER.md:193-203 (§3.3) three-step hierarchical variant (C-12, C-13).
  diagnostics.py   consensus distance / mean checksum, fp64.
  interval.py      communication-interval accumulator (Table 1).
  lars.py          LARS per-layer rates + layer-aligned segment plan (Table 1; §8(f) #2).
  sgp.py           SGP directed exponential graph, the comparison baseline (§8(f) #3).
  wire.py          bf16 wire format for received segments (§8(f) #4; reading C-20).

Every function is pinned by `-m "not gpu"` tests against values fixed by the
paper or mathematics (tests/test_oracle_*.py).  Parity unpinned:
the *specific* permutation drawn for a given seed (any derangement is a valid
topology, reading C-16) — only its law (exact, brute-forced) is pinned.
"""
