O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_storage.py -m gpu -q -x > $O/pytest_storage.log 2>&1; echo "rc=$?" >> $O/pytest_storage.log
for w in tc sg andersen triangle doop; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $O/r_$w.json 2>$O/r_$w.err; done
timeout 600 python tools/phase_report.py --workload tc --kernels > $O/busy5_tc.txt 2>&1
exit 0
