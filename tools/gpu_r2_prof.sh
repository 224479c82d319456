#!/bin/bash
# profile the per-rule kernels: DOOP / triangle timelines and ncu of the
# triangle's per-rule count kernel and DOOP's heaviest ones (summaries only)
O=gpurun_out
for w in doop triangle sg tc; do
  timeout 600 python tools/phase_report.py --workload $w --kernels > $O/kern_$w.log 2>&1
done
timeout 600 python tools/phase_report.py --workload doop --rules 20 > $O/phase_doop.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srdl_jit_wcoj -c 1 \
  -o /tmp/prof_tri python tools/phase_report.py --workload triangle > $O/ncu_tri.log 2>&1
python tools/ncu_summary.py /tmp/prof_tri.ncu-rep > $O/ncu_tri_summary.txt 2>&1
python tools/ncu_lines.py /tmp/prof_tri.ncu-rep > $O/ncu_tri_lines.txt 2>&1
cp /tmp/prof_tri.ncu-rep $O/ 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_doop.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > $O/ncu_doop_bench.log 2>&1
python tools/launch_summary.py $O/launches_doop.csv 40 > $O/launches_doop_summary.txt 2>&1
rm -f $O/launches_doop.csv
exit 0
