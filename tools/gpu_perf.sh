#!/bin/bash
# tests + benches (+ optional ncu) on one GPU box; outputs under gpurun_out/
O=gpurun_out
export PYTHONFAULTHANDLER=1
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
fi
for spec in ${BENCHES:-triangle}; do
  w=${spec%%:*}; env=${spec#*:}; [ "$env" = "$spec" ] && env=""
  tag=$(echo "$spec" | tr ':=' '__')
  timeout 900 env $env python bench.py --workload $w --steps 3 --warmup 3 ${BENCH_ARGS} > $O/bench_$tag.json 2> $O/bench_$tag.err
done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wcoj -c 1 -o $O/prof_$NCU python bench.py --workload $NCU --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
fi
exit 0
