#!/bin/bash
# Single-GPU bench lines: every config at its threshold and at h = 1.01 (plain top-k MoE, the Vanilla
# comparison), the C3 threshold sweep 0.80-0.99, the C4 12-block stack with / without history shortcuts,
# the oracle reference arm.  -> gpurun_out/$TAG/*.json
set -u
TAG=${1:-r02_single}
O=gpurun_out/$TAG; mkdir -p $O
run() { out=$1; shift; timeout 900 python bench.py "$@" > $O/$out 2>> $O/err.log; echo "$out rc=$?"; }
run C2.json --config C2 --steps 20 --warmup 5
run C2_plain.json --config C2 --h 1.01 --steps 20 --warmup 5 --no-cpu-baseline
run C3.json --config C3 --steps 20 --warmup 5
run C3_plain.json --config C3 --h 1.01 --steps 20 --warmup 5 --no-cpu-baseline
for h in 0.80 0.85 0.90 0.95 0.99; do run C3_h$h.json --config C3 --h $h --steps 20 --warmup 5 --no-cpu-baseline --no-e2e; done
run C4.json --config C4 --steps 10 --warmup 3
run C4_plain.json --config C4 --h 1.01 --steps 10 --warmup 3 --no-cpu-baseline
run C5.json --config C5 --steps 5 --warmup 3
run C5_plain.json --config C5 --h 1.01 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
run C4stack.json --config C4 --stack 12 --steps 5 --warmup 3
run C4stack_hist.json --config C4 --stack 12 --steps 5 --warmup 3 --history 0.8,0.2
run ref_C2.json --impl reference --config C2 --steps 3 --warmup 3
tail -3 $O/err.log
