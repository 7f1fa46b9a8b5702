set -u
OUT=gpurun_out/r02ae; mkdir -p $OUT
( time timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err ) 2> $OUT/bench.time
timeout 900 python -m pytest tests/test_gpu_searches.py tests/test_gpu_models.py -q > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
echo done
