#!/bin/bash
# round-2 evidence, final build: bench lines of every config (parity, cpu
# baseline), reference arms, ncu --set full of the dominant kernels (with the
# issue-rate figures), DRAM traffic per family, launch lists, multi-rank
# exchange volumes, DOOP per-rule device times. Small files only.
O=gpurun_out
E=$O/ev3
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $E/gpu.txt 2>&1; nproc >> $E/gpu.txt
for w in ${BENCHES:-doop triangle tc sg andersen}; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 > $E/bench_$w.json 2> $E/bench_$w.err
done
if [ -z "$SKIP_REF" ]; then
timeout 900 python bench.py --impl reference --workload doop --steps 3 --warmup 3 > $E/ref_doop.json 2> $E/ref_doop.err
timeout 900 python bench.py --impl reference --workload tc --steps 3 --warmup 3 > $E/ref_tc.json 2> $E/ref_tc.err
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srdl_jit_wcoj -c 1 -o /tmp/ev_tri \
  python tools/phase_report.py --workload triangle > $E/ncu_tri.log 2>&1
python tools/ncu_summary.py /tmp/ev_tri.ncu-rep --json $E/issue_triangle.json > $E/ncu_triangle_kernel.txt 2>&1
python tools/ncu_lines.py /tmp/ev_tri.ncu-rep > $E/ncu_triangle_kernel_lines.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:srdl_jit_wcoj --launch-skip 600 -c 3 -o /tmp/ev_doop \
  python tools/phase_report.py --workload doop > $E/ncu_doop.log 2>&1
python tools/ncu_summary.py /tmp/ev_doop.ncu-rep --json $E/issue_doop.json > $E/ncu_doop_kernels.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:onesweep_pass --launch-skip 16 -c 2 -o /tmp/ev_sort \
  python tools/phase_report.py --workload tc > $E/ncu_sort.log 2>&1
python tools/ncu_summary.py /tmp/ev_sort.ncu-rep > $E/ncu_sort_kernel.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"mp_merge_rows|hset_filter_rows" --launch-skip 40 -c 2 -o /tmp/ev_merge \
  python tools/phase_report.py --workload sg > $E/ncu_merge.log 2>&1
python tools/ncu_summary.py /tmp/ev_merge.ncu-rep > $E/ncu_merge_hash_kernels.txt 2>&1
for w in triangle doop tc sg; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $E/launches_${w}_bench.log 2>&1
  python tools/launch_summary.py $E/launches_$w.csv 30 > $E/launches_$w.txt 2>&1; rm -f $E/launches_$w.csv
done
for w in doop sg tc triangle andersen; do
  K=""
  case $w in doop|andersen|triangle) K="-k regex:srdl_jit_wcoj|wcoj_kernel|gather_kernel";; esac
  timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none $K --csv \
    --log-file $E/traffic_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --profile-steps 1 --no-parity --no-cpu-baseline \
    > $E/traffic_bench_$w.json 2>$E/traffic_$w.err
  python tools/traffic_summary.py $E/traffic_$w.csv $w $E/traffic_bench_$w.json > $E/traffic_$w.txt 2>&1
  rm -f $E/traffic_$w.csv
done
timeout 900 python tools/phase_report.py --workload doop --rules 25 > $E/rules_doop.log 2>&1
timeout 600 python tools/host_profile.py --workload doop --top 40 > $E/host_doop.txt 2>&1
timeout 1500 python -m pytest tests/test_dist.py -m gpu -k "doop_200k" -s -q > $E/dist_doop200k.log 2>&1
exit 0
