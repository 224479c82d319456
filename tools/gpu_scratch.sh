O=gpurun_out
export PYTHONFAULTHANDLER=1
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python bench.py --workload andersen --small --steps 1 --warmup 3 --no-cpu-baseline > $O/sanit_andersen.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --workload andersen --steps 1 --warmup 3 --no-cpu-baseline > $O/andersen_blocking.log 2>&1
for spec in "SRDL_HASH_SLOTS=1024 SRDL_HASH_RATIO=1" "SRDL_HASH_SLOTS=1024 SRDL_HASH_RATIO=2" "SRDL_HASH_SLOTS=1024 SRDL_HASH_RATIO=4" "SRDL_HASH_SLOTS=2048 SRDL_HASH_RATIO=1" "SRDL_HASH_SLOTS=0"; do
  tag=$(echo "$spec" | tr ' =' '__')
  timeout 600 env $spec python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/tri_$tag.json 2>$O/tri_$tag.err
done
exit 0
