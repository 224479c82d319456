O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for v in default prev; do
  lib=""; [ $v != default ] && lib="SRDL_LIBRARY=$PWD/paper_2604_20073_b200/libsrdl_$v.so"
  for w in triangle sg doop andersen tc; do timeout 600 env $lib python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/lc_${v}_$w.json 2>$O/lc_${v}_$w.err; done
done
exit 0
