set -u
mkdir -p gpurun_out/probe
for p in 0 37 18; do
  for r in 2304 4736; do
    echo "== pairs=$p rpe=$r"; LUFFY_GEMM_PAIRS=$p timeout 300 python tools/gemm_probe.py $r
  done
done > gpurun_out/probe/pairs.txt 2>&1
