#!/bin/bash
# hash-set policy check + allocator behaviour of the DOOP fixpoint
O=gpurun_out
mkdir -p $O/pol
for w in andersen tc; do
  SRDL_DEBUG_DELTA=1 timeout 600 python tools/phase_report.py --workload $w --kernels > $O/pol/dbg_$w.log 2>&1
done
for w in tc sg andersen doop; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/pol/bench_$w.json 2> $O/pol/bench_$w.err
done
timeout 600 python tools/host_profile.py --workload doop --top 30 > $O/pol/host_doop_exp.txt 2>&1
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:False timeout 600 python tools/host_profile.py --workload doop --top 30 > $O/pol/host_doop_noexp.txt 2>&1
exit 0
