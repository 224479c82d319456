#!/bin/bash
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "storage or engine or (baseline and (tc or doop or andersen))" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/host_profile.py --workload doop > $O/host_doop.txt 2>&1
timeout 600 python tools/phase_report.py --workload doop --kernels > $O/kern_doop.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep_pass --launch-skip 20 -c 1 \
  -o /tmp/prof_sort python tools/phase_report.py --workload tc > $O/ncu_sort.log 2>&1
python tools/ncu_summary.py /tmp/prof_sort.ncu-rep > $O/ncu_sort_summary.txt 2>&1
python tools/ncu_lines.py /tmp/prof_sort.ncu-rep > $O/ncu_sort_lines.txt 2>&1
for w in doop tc sg triangle andersen; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err
done
exit 0
