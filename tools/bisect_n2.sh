# A/B of several builds at N=2 (C2), each with its own bench.py: tools/bisect_n2.sh dir1 dir2 ...
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
A="--gpus 2 --config C2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
i=0
for d in "$@"; do
  i=$((i+1))
  (cd $d && timeout 300 $P --master-port $((29600 + i)) bench.py $A > /root/repo/gpurun_out/bis_$i.json 2>/dev/null)
  python -c "
import json; d=json.loads(open('gpurun_out/bis_$i.json').read().strip().splitlines()[-1]); print('$d', d['ms_per_step'], sum(d['breakdown_ms'].values()))" 2>/dev/null || echo "$d failed"
done
