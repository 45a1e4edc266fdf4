#!/bin/bash
# Extra multi-GPU lines (C3 N=2/4, C4 N=2, C5 N=2) on a 4-GPU box -> gpurun_out/$1/
set -u
O=gpurun_out/${1:-r02_extra}; mkdir -p $O
runN() { n=$1; out=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
  --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n "$@" > $O/$out 2>> $O/err.log; echo "$out rc=$?"; }
runN 2 C3_n2.json --config C3 --steps 20 --warmup 5 --no-cpu-baseline
runN 4 C3_n4.json --config C3 --steps 20 --warmup 5 --no-cpu-baseline
runN 2 C4_n2.json --config C4 --steps 10 --warmup 3 --no-cpu-baseline
runN 2 C5_n2.json --config C5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline
tail -3 $O/err.log
