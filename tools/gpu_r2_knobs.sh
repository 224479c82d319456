#!/bin/bash
# launch-geometry knob sweep on the final build (triangle, DOOP)
O=gpurun_out
E=$O/kn
mkdir -p $E
run() { tag=$1; w=$2; shift 2; env "$@" timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --profile-steps 1 --no-cpu-baseline --no-parity > $E/${w}_$tag.json 2> $E/${w}_$tag.err; }
run base triangle
run slice1k triangle SRDL_MIN_SLICE_UNITS=1024
run slice16k triangle SRDL_MIN_SLICE_UNITS=16384
run chunk64 triangle SRDL_SPEC_CHUNK=64
run chunk256 triangle SRDL_SPEC_CHUNK=256
run base doop
run slice1k doop SRDL_MIN_SLICE_UNITS=1024
run slice16k doop SRDL_MIN_SLICE_UNITS=16384
run chunk256 doop SRDL_SPEC_CHUNK=256
run chunk64 doop SRDL_SPEC_CHUNK=64
exit 0
