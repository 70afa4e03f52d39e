"""CPU oracle for the Skrull (arXiv 2505.19609) DACP varlen-attention hot path.

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything here.
The product path (`paper_2505_19609_b200/`) never imports, links or executes
this package, and this package never imports the product: the two share no
code, headers, tables or constants. Inputs come from `synth/` (random draws
only).

Every function cites the PAPER.md passage it follows (`P:n` = line n of
/root/reference/PAPER.md; `S:n` = line n of SPEC.md; `R#` = a reading in
DESIGN.md's ambiguity ledger). Plain and slow on purpose:
  * cost_model  -- Eq. 12-15, Memory(S) -> C      (exact integers / floats)
  * schedule    -- Alg. 1 + Alg. 3 (DACP), Alg. 2 (GDS), LPT binpack, Eq. 1-7
                   evaluator, exhaustive optimum     (exact Fractions)
  * pack        -- per-CP-rank packed layout (R20-R23)
  * attention   -- fp64 naive masked causal attention fwd + analytic bwd
  * metrics     -- useful-FLOP accounting (R32) and the plan floor

Pins: tests/test_oracle_*.py (marked `not gpu`) pin each function to values
the paper prints, closed forms, invariants, brute force and finite differences.
Parity status per function is listed in DESIGN.md ("Oracle pins").
"""
