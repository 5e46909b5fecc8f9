"""CPU ORACLE -- test infrastructure only, never the product path.

Restatements of the reference `reslice` algorithms on this hot path, used by
tests/, __graft_entry__.smoke() and bench.py's `cpu_baseline` / `--impl
reference` legs as the CHECKER (and as the reference's CPU path when timed).
Nothing in paper_2307_08771_b200/ imports this package.

  apply_plan_ref  numpy restatement of apply_plan's weight math
                  (planner.py:648-796, input mode), applied plan by plan exactly
                  like pipeline.py:140-142 -- deliberately NOT the composed
                  single-pass scheme the GPU export uses.
  interp_ref      numpy restatement of interp.run / check_equivalence
                  (interp.py:36-121) on the channel-collapsed IR.
  spatial_ref     CPU (torch fp32/fp64) executor of the same op semantics with
                  the real spatial ops substituted (conv, BN, pools): the
                  logits oracle for the GPU engine and the timed CPU baseline.

Pinning: tests/golden/ holds fixtures generated from
the reference itself by tools/make_golden.py and tools/make_assets.py (exported
graphs, per-layer sha256 of exported weights, interpreter outputs, plans).
"""
