#!/bin/bash
# Round-end multi-GPU set on a 4-GPU box: multi-rank parity (N=2, 4) at HEAD, then the N=2/4 bench lines.
set -u
TAG=${1:-r02_endB}
O=gpurun_out/$TAG; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/multirank_parity.log 2>&1; echo "pytest rc=$?" >> $O/multirank_parity.log
runN() { n=$1; out=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
  --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n "$@" > $O/$out 2>> $O/err.log; echo "$out rc=$?"; }
runN 2 C2_n2.json --config C2 --steps 20 --warmup 5 --no-cpu-baseline
runN 4 C2_n4.json --config C2 --steps 20 --warmup 5 --no-cpu-baseline
runN 2 C2_n2_q2.json --config C2 --steps 20 --warmup 5 --migrate 2 --no-cpu-baseline
runN 4 C5_n4.json --config C5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline
runN 4 C4_n4.json --config C4 --steps 10 --warmup 3 --no-cpu-baseline
runN 2 C4stack_n2_off.json --config C4 --stack 12 --steps 5 --warmup 3
runN 2 C4stack_n2_q2.json --config C4 --stack 12 --steps 5 --warmup 3 --migrate 2
runN 4 C4stack_n4_off.json --config C4 --stack 12 --steps 5 --warmup 3
runN 4 C4stack_n4_q2.json --config C4 --stack 12 --steps 5 --warmup 3 --migrate 2
tail -3 $O/err.log
