O=gpurun_out
export PYTHONFAULTHANDLER=1
for v in default unroll noinl; do
  lib=""; [ $v != default ] && lib="SRDL_LIBRARY=$PWD/paper_2604_20073_b200/libsrdl_$v.so"
  for w in triangle sg andersen doop; do timeout 600 env $lib python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $O/v_${v}_$w.json 2>$O/v_${v}_$w.err; done
done
exit 0
