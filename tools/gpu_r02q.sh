set -u
OUT=gpurun_out/r02q; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_commit.py tests/test_gpu_large.py -q > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for p in 5 6 7 8 9 10 11; do
  timeout 600 python bench.py --workload dag:20000 --parents $p --steps 3 --warmup 3 --no-cpu --no-extras > $OUT/dag20k_p$p.json 2> $OUT/dag20k_p$p.err
done
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
echo done
