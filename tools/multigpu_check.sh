#!/bin/bash
# 4-GPU check: multi-rank parity (N=2,4) and C2 bench A/B of the dispatch push (TMA bulk vs warp stores)
set -u
O=gpurun_out/${1:-r02_mg}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs 2>&1 | tail -5 > $O/parity.log
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
  for v in 1 0; do
    LUFFY_PUSH_TMA=$v timeout 400 $P --nproc-per-node $n --master-port $((29800 + n * 10 + v)) bench.py --gpus $n --config C2 \
      --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/C2_n${n}_tma$v.json 2>> $O/err.log
  done
done
cat $O/parity.log
for f in $O/C2_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); nv=d['nvlink']['per_rank'][0]
print('$f', d['ms_per_step'], (nv.get('dispatch_push') or {}).get('GBps'), (nv.get('dispatch_push') or {}).get('us'), nv.get('nvml_counters_rank'))" 2>/dev/null || echo "$f bad"; done
