#!/bin/bash
# round-2 evidence, part 2: launch lists, ncu --set full of the dominant
# kernels, multi-rank exchange volumes, DOOP/SG traffic (bounded)
O=gpurun_out
mkdir -p $O/ev
timeout 1200 python -m pytest tests/test_dist.py -m gpu -k "doop_200k or bench_two" -s -q > $O/ev/dist_doop200k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srdl_jit_wcoj -c 1 -o /tmp/ev_tri \
  python tools/phase_report.py --workload triangle > $O/ev/ncu_tri.log 2>&1
python tools/ncu_summary.py /tmp/ev_tri.ncu-rep > $O/ev/ncu_triangle_kernel.txt 2>&1
python tools/ncu_lines.py /tmp/ev_tri.ncu-rep > $O/ev/ncu_triangle_kernel_lines.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:srdl_jit_wcoj --launch-skip 600 -c 3 -o /tmp/ev_doop \
  python tools/phase_report.py --workload doop > $O/ev/ncu_doop.log 2>&1
python tools/ncu_summary.py /tmp/ev_doop.ncu-rep > $O/ev/ncu_doop_kernels.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:onesweep_pass --launch-skip 10 -c 1 -o /tmp/ev_sort \
  python tools/phase_report.py --workload tc > $O/ev/ncu_sort.log 2>&1
python tools/ncu_summary.py /tmp/ev_sort.ncu-rep > $O/ev/ncu_sort_kernel.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:hset_filter_rows --launch-skip 4 -c 1 -o /tmp/ev_hash \
  python tools/phase_report.py --workload tc > $O/ev/ncu_hash.log 2>&1
python tools/ncu_summary.py /tmp/ev_hash.ncu-rep > $O/ev/ncu_hash_kernel.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ev/launches_triangle.csv \
  python bench.py --workload triangle --steps 1 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $O/ev/launches_triangle_bench.log 2>&1
python tools/launch_summary.py $O/ev/launches_triangle.csv 30 > $O/ev/launches_triangle.txt 2>&1; rm -f $O/ev/launches_triangle.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ev/launches_tc.csv \
  python bench.py --workload tc --steps 1 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $O/ev/launches_tc_bench.log 2>&1
python tools/launch_summary.py $O/ev/launches_tc.csv 30 > $O/ev/launches_tc.txt 2>&1; rm -f $O/ev/launches_tc.csv
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"srdl_jit_wcoj|wcoj_kernel|gather_kernel" --csv \
  --log-file $O/ev/traffic_doop.csv python bench.py --workload doop --steps 1 --warmup 3 --profile-steps 1 --no-parity --no-cpu-baseline \
  > $O/ev/traffic_bench_doop.json 2>$O/ev/traffic_doop.err
python tools/traffic_summary.py $O/ev/traffic_doop.csv doop $O/ev/traffic_bench_doop.json > $O/ev/traffic_doop.txt 2>&1
rm -f $O/ev/traffic_doop.csv
exit 0
