P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
A="--gpus 2 --config C2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-ktab"
run() { tag=$1; shift; env "$@" timeout 300 $P --master-port $((29700 + RANDOM % 100)) bench.py $A > gpurun_out/abe_$tag.json 2>/dev/null;
  python -c "
import json; d=json.loads(open('gpurun_out/abe_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['ms_per_step'], sum(d['breakdown_ms'].values()))" 2>/dev/null || echo "$tag failed"; }
run head X=1
run nonvml LUFFY_NO_NVML=1
run oldlayout LUFFY_LAYOUT_SMEM=0
run both LUFFY_NO_NVML=1 LUFFY_LAYOUT_SMEM=0
