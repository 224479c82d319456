O=gpurun_out
timeout 900 python tools/phase_report.py --workload doop --schedule seq --rules 25 > $O/rules_doop.txt 2>&1
timeout 600 python tools/phase_report.py --workload sg --schedule seq --rules 12 > $O/rules_sg.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:wcoj_kernel -c 2 -o $O/prof_tri_v5 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tri.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:wcoj_kernel -s 1 -c 1 -o $O/prof_tri_mat_s18 python bench.py --scale 18 --edges 4000000 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tri_mat.log 2>&1
exit 0
