#!/bin/bash
# storage/engine correctness of the onesweep sort, host profile of DOOP,
# merge-path threshold sweep on the triangle (per-rule kernels), benches
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_storage.py tests/test_gpu_engine.py -q -x > $O/pytest_sort.log 2>&1; echo "rc=$?" >> $O/pytest_sort.log
timeout 600 python tools/host_profile.py --workload doop > $O/host_doop.txt 2>&1
for d in "" "-DSRDL_MERGE_RATIO=4" "-DSRDL_MERGE_RATIO=2" "-DSRDL_MERGE_MIN=128" "-DSRDL_MERGE_MIN=256 -DSRDL_MERGE_RATIO=4" "-DSRDL_MERGE_MIN=1000000000"; do
  tag=$(echo "x$d" | tr -c 'a-zA-Z0-9\n' '_')
  SRDL_JIT_DEFINES="$d" timeout 600 python bench.py --workload triangle --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/sweep_$tag.json 2>&1
done
for w in tc sg doop; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
exit 0
