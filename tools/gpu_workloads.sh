#!/bin/bash
# Every BASELINE config as a bench workload (one JSON line each) -> gpurun_out/$1/
OUT=gpurun_out/${1:-workloads}
mkdir -p "$OUT"
for w in ${WORKLOADS:-squeezenet resnet50 inception_v3 nasnet_a dag:1000 dag:5000 dag:20000}; do
  f=$(echo "$w" | tr ':' '_')
  timeout 900 python bench.py --workload "$w" --steps 5 --warmup 3 --cpu-budget 10 --no-extras > "$OUT/$f.json" 2> "$OUT/$f.err"
  echo "$w exit $?" >> "$OUT/status.txt"
done
