set -u
OUT=gpurun_out/r02m; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_shard.py -q -x > $OUT/pytest_shard.log 2>&1; echo "exit $?" >> $OUT/pytest_shard.log
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
echo done
