set -u
OUT=gpurun_out/r02n; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_commit.py -q -x > $OUT/pytest_commit.log 2>&1; echo "exit $?" >> $OUT/pytest_commit.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest "tests/test_gpu_shard.py::test_sharded_search_equals_single" -q -x -k squeezenet > $OUT/sanitizer.log 2>&1; echo "exit $?" >> $OUT/sanitizer.log
echo done
