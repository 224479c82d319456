#!/bin/bash
O=gpurun_out
E=$O/sl
mkdir -p $E
run() { tag=$1; w=$2; shift 2; env "$@" timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $E/${w}_$tag.json 2> $E/${w}_$tag.err; }
for u in 16384 65536 131072 262144 524288; do run s$u triangle SRDL_MIN_SLICE_UNITS=$u; done
for w in doop andersen sg tc; do
  for u in 16384 131072; do run s$u $w SRDL_MIN_SLICE_UNITS=$u; done
done
exit 0
