#!/bin/bash
# full GPU suite + host profile + kernel breakdowns + benches
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python tools/host_profile.py --workload doop > $O/host_doop.txt 2>&1
for w in ${KERNS:-tc doop}; do
  timeout 600 python tools/phase_report.py --workload $w --kernels > $O/kern_$w.log 2>&1
done
for w in ${BENCHES:-doop triangle sg tc andersen}; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > $O/bench_$w.json 2> $O/bench_$w.err
done
exit 0
