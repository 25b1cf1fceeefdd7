"""TEST INFRASTRUCTURE ONLY.

`oracle/` is the CPU checker for the B200 hot path: a numpy restatement of
the reference `randcp` algorithms (leverage-score samplers, sampled-nonzero
gather, downsampled MTTKRP, accumulator-stationary solve, ALS round loop).
It is pinned against golden vectors produced by the reference itself
(`tests/golden/make_golden.py`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (the `cpu_baseline`
leg and `--impl reference`) may import it, and only as the checker or the
timed CPU baseline.  The product package `paper_2210_05105_b200` never
imports anything from here.
"""
