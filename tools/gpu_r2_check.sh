#!/bin/bash
# round-2 check: full -m gpu suite (incl. the BASELINE-size digest parity),
# smoke, default bench (DOOP) and the TC/SG/triangle benches
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for w in ${BENCHES:-doop}; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > $O/bench_$w.json 2> $O/bench_$w.err
done
exit 0
