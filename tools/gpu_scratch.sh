O=gpurun_out
for w in tc sg andersen; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $O/u_$w.json 2>$O/u_$w.err; done
timeout 300 python -m pytest tests/test_gpu_storage.py -m gpu -q -x -k "sort or delta or merge" > $O/pytest_sort.log 2>&1; echo rc=$? >> $O/pytest_sort.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"wcoj_kernel<.*0.*2>" -s 60 -c 2 -o $O/prof_doop_gen python tools/phase_report.py --workload doop --kernels > $O/ncu_doopg.log 2>&1
exit 0
