set -u
OUT=gpurun_out/r02ag; mkdir -p $OUT
EF_LIB=$PWD/exp/libef200_mb8.so timeout 600 python bench.py --workload dag:20000 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d20_mb8.json 2> $OUT/d20_mb8.err
EF_LIB=$PWD/exp/libef200_mb8.so timeout 600 python bench.py --workload dag:5000 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d5_mb8.json 2> $OUT/d5_mb8.err
bash tools/gpu_workloads.sh r02ag/workloads
echo done
