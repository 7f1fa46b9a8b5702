set -u
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_models.py -q -x > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for m in 0 1; do
for w in dag:20000 dag:5000 nasnet_a inception_v3 dag:1000; do
  EF_SPEC_PRICE=$m timeout 600 python bench.py --workload $w --steps 4 --warmup 3 --no-cpu --no-extras > $OUT/w_${w/:/_}_s$m.json 2> $OUT/w_${w/:/_}_s$m.err
done
done
EF_SPEC_PRICE=1 timeout 600 python bench.py --workload dag:20000 --parents 7 --steps 4 --warmup 3 --no-cpu --no-extras > $OUT/w_dag_20000_p7_s1.json 2> $OUT/w_dag_20000_p7_s1.err
echo done
