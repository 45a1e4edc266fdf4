# Round-end bench lines (run on a 4-GPU box): python bench.py per config / world size -> gpurun_out/v6_*.json
set -u
O=gpurun_out/bench_v6; mkdir -p $O
run1() { python bench.py "$@" 2>$O/err.log | tail -1; }
runN() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $n "$@" 2>>$O/err.log | tail -1; }
run1 --config C2 > $O/v6_b1_C2.json
runN 2 --config C2 > $O/v6_b2_C2.json
runN 4 --config C2 > $O/v6_b4_C2.json
runN 2 --config C2 --migrate 2 > $O/v6_b2_C2_q2.json
run1 --config C3 > $O/v6_b1_C3.json
run1 --config C4 --steps 60 > $O/v6_b1_C4.json
runN 2 --config C4 --steps 60 > $O/v6_b2_C4.json
runN 4 --config C4 --steps 60 > $O/v6_b4_C4.json
run1 --config C5 --steps 20 > $O/v6_b1_C5.json
python bench.py --impl reference --steps 3 --warmup 3 > $O/v6_ref_C2.json 2>>$O/err.log
for f in $O/v6_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1], d.get('n_gpus'), round(d['value']/1e6,3), 'M', round(d.get('ms_per_step',0),4), 'e2e', round((d.get('e2e') or {}).get('value',0)/1e6,3), 'frac', round((d.get('roofline') or {}).get('frac',0),3), (d.get('clocks') or {}).get('sm_mhz'))
" 2>/dev/null || echo "$f bad"; done
# warm per-kernel table and the ncu launch list of the default (C2, N=1) command
LUFFY_PDL=0 CUDA_VISIBLE_DEVICES=0 python bench.py --steps 100 --warmup 5 --kprof 100 --kprof-dir $O --no-cpu-baseline --no-e2e > $O/kprof_bench.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_v6.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
