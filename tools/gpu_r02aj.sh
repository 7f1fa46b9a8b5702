set -u
OUT=gpurun_out/r02aj; mkdir -p $OUT
for l in 4 2 8; do
EF_PRICE_LANES=$l timeout 1200 python -m pytest tests/test_gpu_models.py tests/test_gpu_searches.py tests/test_gpu_parity.py -q -x > $OUT/pytest_l$l.log 2>&1; echo "exit $?" >> $OUT/pytest_l$l.log
done
for l in 0 2 4 8; do
  for w in resnet50 inception_v3 nasnet_a; do
    EF_PRICE_LANES=$l timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-extras > $OUT/${w}_l$l.json 2> $OUT/${w}_l$l.err
  done
  EF_PRICE_LANES=$l EF_SPEC_PRICE=0 timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/d20s0_l$l.json 2> $OUT/d20s0_l$l.err
done
echo done
