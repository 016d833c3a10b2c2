"""CPU oracle for the Pipe-SGD communication hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the algorithm of the reference package
`gradpipe` (Python + numpy, /root/reference/pkg/src/gradpipe) for every
function on the hot path: the gradient codecs, the ring schedule and its
fold order, the SGD consumer, and the engine's width-K trajectory.

Who may import it: `tests/`, `__graft_entry__.smoke()` (as the checker) and
`bench.py`'s `cpu_baseline` / `--impl reference` legs. The product package
`paper_1811_03619_b200` never imports, calls or links anything in here, and
it raises loudly when its CUDA library is missing instead of falling back.

Parity pinning: every function here is checked against golden vectors that
`tests/golden/make_golden.py` produced by running the real reference
(`tests/test_oracle_golden.py`), and — when /root/reference is mounted —
against the live reference on fresh random inputs (`tests/test_oracle_live.py`).
"""
