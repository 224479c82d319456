O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -k "speculative or golden_fixpoints" > $O/pytest_spec.log 2>&1; echo rc=$? >> $O/pytest_spec.log
for c in 128 256 512; do for w in triangle sg doop andersen; do SRDL_SPEC_CHUNK=$c timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $O/c${c}_$w.json 2>$O/c${c}_$w.err; done; done
exit 0
