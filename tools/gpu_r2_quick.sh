#!/bin/bash
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-storage or engine}" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for w in ${KERNS:-doop tc}; do
  timeout 600 python tools/phase_report.py --workload $w --kernels > $O/kern_$w.log 2>&1
done
for w in ${BENCHES:-doop tc triangle}; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
exit 0
