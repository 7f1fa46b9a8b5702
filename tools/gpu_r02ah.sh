set -u
OUT=gpurun_out/r02ah; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_gpu_models.py tests/test_gpu_searches.py -q -x > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for l in 8 4 16; do
  EF_WIDE_LPC=$l timeout 600 python bench.py --workload dag:20000 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d20_l$l.json 2> $OUT/d20_l$l.err
done
for w in dag:5000 nasnet_a dag:1000; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/w_${w/:/_}.json 2> $OUT/w_${w/:/_}.err
done
echo done
