#!/bin/bash
# A/B of Compute Delta through the hash set vs sort + anti-join, per workload;
# CUPTI kernel totals; host profile of DOOP
O=gpurun_out
mkdir -p $O/ab
for w in tc sg andersen doop; do
  timeout 600 python tools/phase_report.py --workload $w --kernels > $O/ab/kern_${w}_hash.log 2>&1
  SRDL_HASH_MIN_FULL=1000000000000 timeout 600 python tools/phase_report.py --workload $w --kernels > $O/ab/kern_${w}_nohash.log 2>&1
done
for w in tc sg; do
  SRDL_HASH_MIN_FULL=1000000000000 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-parity > $O/ab/bench_${w}_nohash.json 2>&1
done
timeout 600 python tools/host_profile.py --workload doop --top 60 > $O/ab/host_doop.txt 2>&1
exit 0
