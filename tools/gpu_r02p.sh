set -u
OUT=gpurun_out/r02p; mkdir -p $OUT
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest "tests/test_gpu_shard.py::test_sharded_search_equals_single" -q -x -k resnet50 > $OUT/sanitizer.log 2>&1; echo "exit $?" >> $OUT/sanitizer.log
echo done
