#!/bin/bash
# final bench lines of every config (parity, cpu baseline, issue roofline),
# reference arms, launch lists of the default config
O=gpurun_out
E=$O/fev
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $E/gpu.txt 2>&1; nproc >> $E/gpu.txt
for w in doop triangle tc sg andersen; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > $E/bench_$w.json 2> $E/bench_$w.err
done
timeout 900 python bench.py --impl reference --workload doop --steps 3 --warmup 3 > $E/ref_doop.json 2> $E/ref_doop.err
timeout 900 python bench.py --impl reference --workload tc --steps 3 --warmup 3 > $E/ref_tc.json 2> $E/ref_tc.err
for w in doop triangle; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $E/launches_${w}_bench.log 2>&1
  python tools/launch_summary.py $E/launches_$w.csv 30 > $E/launches_$w.txt 2>&1; rm -f $E/launches_$w.csv
done
exit 0
