#!/bin/bash
# Per-config ncu --set full capture of one bench step (GPU box, one GPU): the stats pass and the first
# warm-up step of `bench.py --config C` (~30 launches), summarised to profiles/<tag>_ncu_full_<C>_n1.json,
# which bench.py reads for the roofline's `traffic` (DRAM read+write of the 6 GEMMs and of the Gram).
#   tools/ncu_capture.sh C2 r02 [extra bench args]
set -u
C=$1; TAG=$2; shift 2
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'gemm_tc|gram_tc|route|gather_norm|group_build|greedy|layout|pack_rows|uncondense|unpack|wg_' \
  -c 32 -f -o gpurun_out/${TAG}_ncu_full_${C} \
  python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ktab "$@" > gpurun_out/${TAG}_ncu_full_${C}.log 2>&1
python profiles/ncu_summary.py gpurun_out/${TAG}_ncu_full_${C}.ncu-rep --json profiles/${TAG}_ncu_full_${C}_n1.json \
  > profiles/${TAG}_ncu_full_${C}_n1.txt
cp profiles/${TAG}_ncu_full_${C}_n1.* gpurun_out/
# the full report stays on the box unless KEEP_REP=1 (gpurun brings back at most 64 MiB)
[ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/${TAG}_ncu_full_${C}.ncu-rep
