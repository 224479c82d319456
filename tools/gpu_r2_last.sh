#!/bin/bash
# last round-2 run on the final build: full -m gpu suite, smoke, final bench
# lines of every config, slice-size points beyond the default (triangle)
O=gpurun_out
E=$O/last
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $E/gpu.txt 2>&1; nproc >> $E/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --durations 10 > $E/pytest_gpu.log 2>&1; echo "rc=$?" >> $E/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo "rc=$?" >> $E/smoke.log
for w in doop triangle tc sg andersen; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > $E/bench_$w.json 2> $E/bench_$w.err
done
for u in 32768 65536; do
  SRDL_MIN_SLICE_UNITS=$u timeout 600 python bench.py --workload triangle --steps 3 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $E/triangle_slice$u.json 2> $E/triangle_slice$u.err
done
exit 0
