O=gpurun_out
export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests -m gpu -q --deselect "tests/test_dist.py" > $O/pytest_gpu_rest.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_rest.log
timeout 300 python -m pytest tests/test_dist.py -m gpu -q -s -k "tc" > $O/pytest_dist_tc.log 2>&1; echo "rc=$?" >> $O/pytest_dist_tc.log
timeout 600 python -m pytest tests/test_dist.py -m gpu -q > $O/pytest_dist_all.log 2>&1; echo "rc=$?" >> $O/pytest_dist_all.log
exit 0
