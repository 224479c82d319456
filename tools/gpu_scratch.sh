O=gpurun_out
for v in default ihist nispec; do
  lib=""; [ $v != default ] && lib="SRDL_LIBRARY=$PWD/paper_2604_20073_b200/libsrdl_$v.so"
  for w in triangle sg doop andersen; do timeout 600 env $lib python bench.py --workload $w --steps 6 --warmup 3 --no-cpu-baseline > $O/v2_${v}_$w.json 2>$O/v2_${v}_$w.err; done
done
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -x > $O/pytest_engine.log 2>&1; echo rc=$? >> $O/pytest_engine.log
exit 0
