O=gpurun_out
timeout 600 python bench.py > $O/default_bench.json 2> $O/default_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_triangle_v6.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:"wcoj_kernel|gather_kernel" -c 2 -o $O/prof_tri_v6 python bench.py --scale 19 --edges 8000000 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tri_v6.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --replay-mode application -k regex:"wcoj_kernel|gather_kernel" -c 2 --csv --log-file $O/traffic_triangle.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_traffic_tri.log 2>&1
for w in tc sg andersen doop; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"wcoj_kernel|gather_kernel" -c 400 --csv --log-file $O/traffic_$w.csv python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_traffic_$w.log 2>&1
done
exit 0
