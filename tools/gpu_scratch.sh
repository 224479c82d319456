O=gpurun_out
export PYTHONFAULTHANDLER=1
for v in default mb6 mb5; do
  lib=""; [ $v != default ] && lib="SRDL_LIBRARY=$PWD/paper_2604_20073_b200/libsrdl_$v.so"
  for w in triangle sg andersen doop; do timeout 600 env $lib python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $O/m_${v}_$w.json 2>$O/m_${v}_$w.err; done
done
timeout 600 python tools/phase_report.py --workload sg --kernels > $O/busy2_sg.txt 2>&1
exit 0
