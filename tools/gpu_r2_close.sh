#!/bin/bash
# closing run: correctness of the final slice default (engine, JIT vs
# generic, full-size parity) and the final bench lines of every config
O=gpurun_out
E=$O/close
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $E/gpu.txt 2>&1; nproc >> $E/gpu.txt
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_baseline_parity.py tests/test_gpu_jit.py -m gpu -q -x --timeout 600 -k "not golden_joins" > $E/pytest.log 2>&1; echo "rc=$?" >> $E/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo "rc=$?" >> $E/smoke.log
for w in doop triangle tc sg andersen; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > $E/bench_$w.json 2> $E/bench_$w.err
done
exit 0
