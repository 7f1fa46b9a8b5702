set -u
OUT=gpurun_out/r02o; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_commit.py -q > $OUT/pytest_shard.log 2>&1; echo "exit $?" >> $OUT/pytest_shard.log
echo done
