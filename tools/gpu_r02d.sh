set -u
OUT=gpurun_out/r02d; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py -x -q > $OUT/pytest_large.log 2>&1; echo "exit $?" >> $OUT/pytest_large.log
for cfg in "default" "EF_DIRTY_BIG=0" "EF_WIDE_LPC=32" "EF_WIDE_LPC=16" "EF_WIDE_LPC=4" "EF_WIDE_MIN=128" "EF_WIDE_MIN=2048"; do
  env EF_X=1 $cfg timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 2 --no-cpu > $OUT/dag20k_$cfg.json 2> $OUT/dag20k_$cfg.err
done
timeout 600 python bench.py --workload nasnet_a --steps 3 --warmup 2 --no-cpu > $OUT/nasnet.json 2> $OUT/nasnet.err
timeout 600 python bench.py --workload dag:1000 --steps 3 --warmup 2 --no-cpu > $OUT/dag1k.json 2> $OUT/dag1k.err
timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
echo done
