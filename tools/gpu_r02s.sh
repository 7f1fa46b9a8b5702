set -u
OUT=gpurun_out/r02s; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_models.py tests/test_gpu_searches.py -q -x > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for p in 7 9; do
  timeout 600 python bench.py --workload dag:20000 --parents $p --steps 3 --warmup 3 --no-cpu --no-extras > $OUT/dag20k_p$p.json 2> $OUT/dag20k_p$p.err
done
for w in dag:5000 nasnet_a inception_v3; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/w_${w/:/_}.json 2> $OUT/w_${w/:/_}.err
done
echo done
