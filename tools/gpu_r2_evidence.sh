#!/bin/bash
# round-2 evidence: bench lines of every config, the reference arm, ncu launch
# lists, DRAM traffic per family (profiles/traffic.json), ncu --set full of
# the dominant kernels, multi-rank exchange volumes. Outputs small files only.
O=gpurun_out
mkdir -p $O/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/ev/gpu.txt 2>&1
nproc >> $O/ev/gpu.txt
for w in doop triangle tc sg andersen; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 > $O/ev/bench_$w.json 2> $O/ev/bench_$w.err
done
timeout 900 python bench.py --impl reference --workload doop --steps 5 --warmup 3 > $O/ev/ref_doop.json 2> $O/ev/ref_doop.err
timeout 900 python bench.py --impl reference --workload tc --steps 5 --warmup 3 > $O/ev/ref_tc.json 2> $O/ev/ref_tc.err
for w in triangle tc sg andersen doop; do
  K=""
  case $w in doop|andersen|triangle) K="-k regex:srdl_jit_wcoj|wcoj_kernel|gather_kernel";; esac
  timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none $K --csv \
     --log-file $O/ev/traffic_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-parity --no-cpu-baseline \
     > $O/ev/traffic_bench_$w.json 2>$O/ev/traffic_$w.err
  python tools/traffic_summary.py $O/ev/traffic_$w.csv $w $O/ev/traffic_bench_$w.json > $O/ev/traffic_$w.txt 2>&1
  rm -f $O/ev/traffic_$w.csv
done
cp profiles/traffic.json $O/ev/traffic.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ev/launches_doop.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > $O/ev/launches_doop_bench.log 2>&1
python tools/launch_summary.py $O/ev/launches_doop.csv 40 > $O/ev/launches_doop.txt 2>&1; rm -f $O/ev/launches_doop.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ev/launches_triangle.csv \
  python bench.py --workload triangle --steps 1 --warmup 3 --no-cpu-baseline --no-parity > $O/ev/launches_triangle_bench.log 2>&1
python tools/launch_summary.py $O/ev/launches_triangle.csv 40 > $O/ev/launches_triangle.txt 2>&1; rm -f $O/ev/launches_triangle.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srdl_jit_wcoj -c 1 -o /tmp/ev_tri \
  python tools/phase_report.py --workload triangle > $O/ev/ncu_tri.log 2>&1
python tools/ncu_summary.py /tmp/ev_tri.ncu-rep > $O/ev/ncu_triangle_kernel.txt 2>&1
python tools/ncu_lines.py /tmp/ev_tri.ncu-rep > $O/ev/ncu_triangle_kernel_lines.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:srdl_jit_wcoj --launch-skip 400 -c 3 -o /tmp/ev_doop \
  python tools/phase_report.py --workload doop > $O/ev/ncu_doop.log 2>&1
python tools/ncu_summary.py /tmp/ev_doop.ncu-rep > $O/ev/ncu_doop_kernels.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:onesweep_pass --launch-skip 20 -c 1 -o /tmp/ev_sort \
  python tools/phase_report.py --workload tc > $O/ev/ncu_sort.log 2>&1
python tools/ncu_summary.py /tmp/ev_sort.ncu-rep > $O/ev/ncu_sort_kernel.txt 2>&1
timeout 1200 python -m pytest tests/test_dist.py -m gpu -k doop_200k -s -q > $O/ev/dist_doop200k.log 2>&1
exit 0
