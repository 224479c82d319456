O=gpurun_out
timeout 600 python bench.py > $O/final_default.json 2> $O/final_default.err
for w in tc sg andersen doop; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/final_$w.json 2> $O/final_$w.err; done
timeout 600 python bench.py --impl reference --steps 1 > $O/final_ref.json 2> $O/final_ref.err
exit 0
