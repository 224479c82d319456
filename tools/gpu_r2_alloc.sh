#!/bin/bash
O=gpurun_out
mkdir -p $O/al
timeout 600 python tools/alloc_trace.py --workload doop --steps 5 > $O/al/alloc_doop_exp.log 2>&1
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:False timeout 600 python tools/alloc_trace.py --workload doop --steps 5 > $O/al/alloc_doop_noexp.log 2>&1
SRDL_DEBUG_DELTA=1 timeout 600 python tools/phase_report.py --workload andersen --kernels > $O/al/dbg_andersen.log 2>&1
for w in andersen tc; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/al/bench_$w.json 2> $O/al/bench_$w.err
done
exit 0
