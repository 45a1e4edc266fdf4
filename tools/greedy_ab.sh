#!/bin/bash
# Greedy change check on one GPU: greedy/layout parity tests, C2/C3/C4 bench lines with the per-kernel
# table, then the fine phase timeline (diagnostic build).  -> gpurun_out/$1/
set -u
O=gpurun_out/${1:-gab}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $O/pytest.log 2>&1; echo pytest rc=$?
for c in C2 C3 C4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/$c.json 2>$O/$c.err; done
LUFFY_NVCC_DEFS=-DLUFFY_GREEDY_FINE python -m paper_2411_15419_b200.build > /dev/null 2>&1
for c in C2 C4; do timeout 300 python tools/greedy_timeline.py $c; done > $O/fine.txt 2>&1
