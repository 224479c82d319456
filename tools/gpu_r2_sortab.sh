#!/bin/bash
# onesweep items-per-thread A/B (8 vs 16), storage tests under 8, ncu of an
# 8-item pass, multi-rank exchange volumes, DOOP host profile
O=gpurun_out
E=$O/sab
mkdir -p $E
SRDL_SORT_ITEMS=8 timeout 900 python -m pytest tests/test_gpu_storage.py -m gpu -q -x --timeout 600 > $E/pytest_storage8.log 2>&1; echo "rc=$?" >> $E/pytest_storage8.log
for it in 8 16; do
  for w in tc sg doop; do
    SRDL_SORT_ITEMS=$it timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-parity > $E/bench_${w}_$it.json 2> $E/bench_${w}_$it.err
  done
done
for it in 8 16; do
  SRDL_SORT_ITEMS=$it timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep_pass --launch-skip 16 -c 1 -o /tmp/sab_sort$it \
    python tools/phase_report.py --workload tc > $E/ncu_sort$it.log 2>&1
  python tools/ncu_summary.py /tmp/sab_sort$it.ncu-rep > $E/ncu_sort${it}_kernel.txt 2>&1
  python tools/ncu_lines.py /tmp/sab_sort$it.ncu-rep > $E/ncu_sort${it}_lines.txt 2>&1
done
timeout 1500 python -m pytest tests/test_dist.py -m gpu -k "doop_200k" -s -q > $E/dist_doop200k.log 2>&1
timeout 600 python tools/host_profile.py --workload doop --top 40 > $E/host_doop.txt 2>&1
exit 0
