"""CPU oracle for the semi-naive fixpoint path — TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product: only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import it. The engine in `paper_2604_20073_b200`
has no CPU fallback and never imports this package.

Contents
--------
storage.py   numpy restatement of the reference's flat sorted-column storage
             operations (reference: pkg/src/flatlog/rowops.py:1-143,
             pkg/src/flatlog/storage.py:28-418): sort_dedup, set difference,
             head/body merge with the flush threshold, incremental histograms.
gj.py        vectorised generic join (attribute-at-a-time over sorted
             relations, reference: pkg/src/flatlog/executor.py:342-431 and
             pkg/src/flatlog/storage.py:156-216) and the stratified semi-naive
             fixpoint loop (reference: pkg/src/flatlog/runtime.py:259-315),
             with its own rule grouping (Kosaraju) and its own variable order,
             sharing only the parsed AST with the engine.
gj_native.cpp + native.py
             the same generic join and semi-naive loop (same rule grouping,
             variable orders and column orders, encoded by native.py from
             gj's own functions) in C++ on all host cores (OpenMP): the
             checker at BASELINE sizes (tests/golden/make_baseline_digests.py)
             and the CPU baseline / reference arm of bench.py.
digest.py    order-checked streaming digests of sorted relations (n, sha256
             of the columns, order-independent 64-bit fold) for full-size
             parity without committing gigabytes of tuples.

Pinning
-------
gj.py, storage.py and the C++ restatement are all checked against golden
fixtures produced by running the reference package itself in the build
container
(tests/golden/make_golden.py -> tests/golden/*.json*), see
tests/test_oracle_golden.py. Parity status: pinned.
"""
