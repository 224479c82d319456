O=gpurun_out
for spec in "SRDL_MERGE_RATIO=4" "SRDL_MERGE_RATIO=8" "SRDL_MERGE_RATIO=32" "SRDL_MERGE_MIN=32" "SRDL_MERGE_MIN=128" "SRDL_MERGE_MIN=1000000000" "SRDL_MIN_SLICE_UNITS=1024" "SRDL_MIN_SLICE_UNITS=16384" "X=default"; do
  tag=$(echo "$spec" | tr '=' '_')
  timeout 600 env $spec python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/w_$tag.json 2>$O/w_$tag.err
done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --replay-mode application -k regex:wcoj_kernel -c 2 --csv --log-file $O/traffic_triangle.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_traffic_tri.log 2>&1
for w in tc sg andersen doop; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:wcoj_kernel -c 400 --csv --log-file $O/traffic_$w.csv python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_traffic_$w.log 2>&1
done
exit 0
