#!/bin/bash
O=gpurun_out
E=$O/ms
mkdir -p $E
export SRDL_JIT_DEFINES="-DSRDL_MERGE_SKIP=1"
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_baseline_parity.py -m gpu -q -x --timeout 600 -k "matches_generic or triangle" > $E/pytest.log 2>&1; echo "rc=$?" >> $E/pytest.log
for w in triangle doop andersen; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $E/${w}_skip.json 2> $E/${w}_skip.err
done
unset SRDL_JIT_DEFINES
for w in triangle doop andersen; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $E/${w}_base.json 2> $E/${w}_base.err
done
exit 0
