#!/bin/bash
O=gpurun_out
E=$O/bo
mkdir -p $E
SRDL_SORT_BACKOFF=128 timeout 900 python -m pytest tests/test_gpu_storage.py -m gpu -q -x --timeout 600 > $E/pytest_storage.log 2>&1; echo "rc=$?" >> $E/pytest_storage.log
for b in 0 64 256 1000; do
  for w in tc sg doop; do
    SRDL_SORT_BACKOFF=$b timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-parity > $E/bench_${w}_$b.json 2> $E/bench_${w}_$b.err
  done
done
exit 0
