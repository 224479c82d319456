O=gpurun_out
for v in default jw8 jw2; do
  lib=""; [ $v != default ] && lib="SRDL_LIBRARY=$PWD/paper_2604_20073_b200/libsrdl_$v.so"
  for w in triangle sg doop andersen; do timeout 600 env $lib python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/jw_${v}_$w.json 2>$O/jw_${v}_$w.err; done
done
exit 0
