#!/bin/bash
O=gpurun_out
E=$O/fu
mkdir -p $E
timeout 2000 python -m pytest tests/test_gpu_engine.py tests/test_gpu_baseline_parity.py tests/test_dist.py tests/test_gpu_jit.py -m gpu -q -x --timeout 600 > $E/pytest.log 2>&1; echo "rc=$?" >> $E/pytest.log
for w in ${BENCHES:-doop sg andersen tc triangle}; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $E/bench_$w.json 2> $E/bench_$w.err
done
timeout 600 python tools/phase_report.py --workload doop --kernels > $E/kern_doop.log 2>&1
exit 0
