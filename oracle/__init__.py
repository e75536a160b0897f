"""CPU oracle for the NeuS2 training hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference `hashsdf` package (arXiv 2212.05231 CPU
restatement, `/root/reference/pkg/src/hashsdf`) for the static training step:
hash encoding, bias-free ReLU MLPs with the Theorem-1 backward, the neural field,
occupancy marching / NeuS compositing and its backward, losses, progressive level
masking and Adam.  Every function cites the reference file:line it follows.

Parity status: PINNED.  `tests/golden/make_golden.py` imports the reference itself
(in the build container) and writes golden vectors to `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this oracle against them (integers bit-exact,
floats to 1e-6 relative or bit-exact where the arithmetic order is the same).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg /
`--impl reference` arm may import this package — as the checker or the timed CPU
baseline, never as part of the product path (`paper_2212_05231_b200`), which has no
CPU fallback.
"""
