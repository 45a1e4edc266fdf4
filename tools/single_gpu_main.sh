#!/bin/bash
# Main single-GPU bench lines (each config at its threshold and at h = 1.01) -> gpurun_out/$1/
set -u
O=gpurun_out/${1:-r02_main}; mkdir -p $O
run() { out=$1; shift; timeout 900 python bench.py "$@" > $O/$out 2>> $O/err.log; echo "$out rc=$?"; }
run C2.json --config C2 --steps 20 --warmup 5
run C2_plain.json --config C2 --h 1.01 --steps 20 --warmup 5 --no-cpu-baseline
run C3.json --config C3 --steps 20 --warmup 5 --no-cpu-baseline
run C3_plain.json --config C3 --h 1.01 --steps 20 --warmup 5 --no-cpu-baseline
run C4.json --config C4 --steps 10 --warmup 3 --no-cpu-baseline
run C4_plain.json --config C4 --h 1.01 --steps 10 --warmup 3 --no-cpu-baseline
run C5.json --config C5 --steps 5 --warmup 3 --no-cpu-baseline
run C5_plain.json --config C5 --h 1.01 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
tail -3 $O/err.log
