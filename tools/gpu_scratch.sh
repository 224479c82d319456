O=gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for w in triangle sg andersen doop tc; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $O/s_$w.json 2>$O/s_$w.err; done
for w in sg doop; do timeout 600 python tools/phase_report.py --workload $w --kernels > $O/busy3_$w.txt 2>&1; done
timeout 600 env SRDL_LIBRARY=$PWD/paper_2604_20073_b200/libsrdl_mb5.so python bench.py --workload sg --steps 3 --warmup 3 --no-cpu-baseline > $O/s_mb5_sg.json 2>$O/s_mb5_sg.err
exit 0
