#!/bin/bash
# round-2 probe: where each workload's fixpoint time goes (CUPTI kernel
# totals + per-phase device times), the new bench on TC, and an ncu --set
# full summary of the delta-maintenance kernels on TC (report deleted
# after summarising: gpurun_out must stay under 64 MiB)
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
timeout 300 python -m pytest tests/test_gpu_baseline_parity.py -k rmat -q -x > $O/pytest_rmat.log 2>&1
timeout 600 python bench.py --workload tc --steps 3 --warmup 3 > $O/bench_tc.json 2> $O/bench_tc.err
for w in tc sg andersen doop triangle; do
  timeout 600 python tools/phase_report.py --workload $w --kernels > $O/kern_$w.log 2>&1
  timeout 600 python tools/phase_report.py --workload $w --rules 12 > $O/phase_$w.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"radix_scatter|radix_hist|mp_diff|mp_merge|rank_merge|scatter_unpack|pack_keys|check_sorted|gather_kernel|tile_scan|flag_keys|bs_diff" \
  --launch-skip 150 -c 40 -o /tmp/prof_delta_tc python tools/phase_report.py --workload tc > $O/ncu_delta.log 2>&1
python tools/ncu_summary.py /tmp/prof_delta_tc.ncu-rep > $O/ncu_delta_summary.txt 2>&1
exit 0
