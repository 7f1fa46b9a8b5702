set -u
OUT=gpurun_out/r02bc; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_models.py tests/test_gpu_searches.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
EF_PRICE_LANES=0 timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_searches.py -q -x -p no:cacheprovider > $OUT/pytest_l0.log 2>&1; echo "exit $?" >> $OUT/pytest_l0.log
for w in resnet50 inception_v3 nasnet_a dag:1000; do
  f=$(echo $w | tr ':' '_')
  timeout 600 python bench.py --workload $w --no-cpu --no-extras --steps 5 > $OUT/${f}_l2.json 2>/dev/null
  EF_PRICE_LANES=0 timeout 600 python bench.py --workload $w --no-cpu --no-extras --steps 5 > $OUT/${f}_l0.json 2>/dev/null
  EF_PRICE_LANES=0 EF_SPARSE_SWEEP=0 timeout 600 python bench.py --workload $w --no-cpu --no-extras --steps 5 > $OUT/${f}_l0d.json 2>/dev/null
done
echo done
