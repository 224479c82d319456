#!/bin/bash
O=gpurun_out
mkdir -p $O/st
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_jit.py -q -x > $O/st/pytest.log 2>&1; echo "rc=$?" >> $O/st/pytest.log
for w in doop sg andersen; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/st/bench_$w.json 2> $O/st/bench_$w.err
done
timeout 600 python tools/host_profile.py --workload doop --top 40 > $O/st/host_doop.txt 2>&1
timeout 600 python tools/phase_report.py --workload doop --kernels > $O/st/kern_doop.log 2>&1
exit 0
