#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list and a full capture of the top kernel.
# Usage (from this container):  gpurun --timeout 1500 -- 'bash tools/gpu_round.sh TAG [KERNEL_REGEX] [PARENTS] [SKIP]'
# SKIP=1 skips pytest/smoke (bench + profiles only).
set -u
TAG=${1:-r01}
KRE=${2:-k_hash_keys}
PARENTS=${3:-4096}
SKIP=${4:-0}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt" 2>&1
if [ "$SKIP" = "0" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.log"
fi
timeout 600 python bench.py --parents "$PARENTS" > "$OUT/bench.json" 2> "$OUT/bench.err"
# launch list of the timed steps only (bench calls cudaProfilerStart/Stop around them when EF_NCU=1)
EF_NCU=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --parents "$PARENTS" --steps 2 --warmup 1 --no-cpu \
    > "$OUT/launches.log" 2>&1
EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:$KRE" -c 6 -o "$OUT/prof" python bench.py --parents "$PARENTS" --steps 1 --warmup 1 --no-cpu \
    > "$OUT/prof.log" 2>&1
echo done
