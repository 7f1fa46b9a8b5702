set -u
OUT=gpurun_out/r02v; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_division.py -q > $OUT/pytest_div.log 2>&1; echo "exit $?" >> $OUT/pytest_div.log
timeout 1200 python -m pytest tests/test_gpu_models.py tests/test_gpu_searches.py tests/test_gpu_parity.py -q > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for m in 0 1 2; do
  EF_SPEC_PRICE=$m timeout 600 python bench.py --workload dag:20000 --parents 9 --steps 4 --warmup 3 --no-cpu --no-extras > $OUT/d20_s$m.json 2> $OUT/d20_s$m.err
  EF_SPEC_PRICE=$m timeout 600 python bench.py --workload inception_v3 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/inc_s$m.json 2> $OUT/inc_s$m.err
done
echo done
