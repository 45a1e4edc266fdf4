P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556"
A="--gpus 2 --config C2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
(cd _r1wt && timeout 300 $P bench.py $A > ../gpurun_out/ab_r1.json 2>/dev/null)
timeout 300 $P bench.py $A --no-ktab > gpurun_out/ab_head.json 2>/dev/null
LUFFY_PDL=0 timeout 300 $P bench.py $A --no-ktab > gpurun_out/ab_head_nopdl.json 2>/dev/null
(cd _r1wt && timeout 300 $P bench.py $A > ../gpurun_out/ab_r1b.json 2>/dev/null)
export CUDA_VISIBLE_DEVICES=0
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_gate" 2>&1 | grep -E "Error|error|status" | head -5 > gpurun_out/ab_fp32.log
for f in ab_r1 ab_head ab_head_nopdl ab_r1b; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d.get('host_enqueue_ms_per_step'), sum(d['breakdown_ms'].values()))"; done
cat gpurun_out/ab_fp32.log
