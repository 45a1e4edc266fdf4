#!/bin/bash
# Memory-side kernel change check on one GPU: single-GPU parity tests, C2/C3/C4 bench lines with the
# per-kernel table.  -> gpurun_out/$1/
set -u
O=gpurun_out/${1:-mab}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_gemm.py -x -q > $O/pytest.log 2>&1; echo pytest rc=$?
for c in C2 C3 C4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/$c.json 2>$O/$c.err; done
