#!/bin/bash
# Multi-GPU bench lines on one box (run under `gpurun --gpus 4`): C2 at N=2/4 (+ migration), C5 at N=4,
# and the C4 12-block stack with sequence migration off / on at N=2 and N=4.  -> gpurun_out/$TAG/*.json
set -u
TAG=${1:-r02_multi}
O=gpurun_out/$TAG; mkdir -p $O
runN() { n=$1; out=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
  --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n "$@" > $O/$out 2>> $O/err.log; \
  echo "$out rc=$?"; }
runN 2 C2_n2.json --config C2 --steps 20 --warmup 5
runN 4 C2_n4.json --config C2 --steps 20 --warmup 5
runN 2 C2_n2_q2.json --config C2 --steps 20 --warmup 5 --migrate 2
runN 4 C5_n4.json --config C5 --steps 10 --warmup 3 --no-e2e
runN 2 C4stack_n2_off.json --config C4 --stack 12 --steps 5 --warmup 3
runN 2 C4stack_n2_q2.json --config C4 --stack 12 --steps 5 --warmup 3 --migrate 2
runN 4 C4stack_n4_off.json --config C4 --stack 12 --steps 5 --warmup 3
runN 4 C4stack_n4_q2.json --config C4 --stack 12 --steps 5 --warmup 3 --migrate 2
tail -5 $O/err.log
