#!/bin/bash
# One GPU session: build check, gpu tests, smoke, benches, launch list, ncu capture.
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for w in ${WORKLOADS:-triangle tc sg andersen}; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; echo "rc=$?" >> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
if [ -n "$NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_triangle.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:wcoj -c 2 -o $O/prof_wcoj python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
fi
exit 0
