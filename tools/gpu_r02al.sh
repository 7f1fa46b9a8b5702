set -u
OUT=gpurun_out/r02al; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_large.py -q > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
timeout 600 python bench.py --sharded --workload dag:20000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/d20_sharded.json 2> $OUT/d20_sharded.err
timeout 600 python bench.py --sharded --workload dag:5000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/d5_sharded.json 2> $OUT/d5_sharded.err
echo done
