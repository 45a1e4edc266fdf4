#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of one fwd+bwd at the C1 (fp32) and C2S (bf16) shapes.
set -u
mkdir -p gpurun_out
for C in C1 C2S; do
  for T in memcheck synccheck racecheck; do
    echo "== $T $C"
    timeout 900 compute-sanitizer --tool $T --kernel-name kns=5luffy \
      --print-limit 20 python tools/sanitize_step.py $C 2>&1 | tail -15
  done
done
