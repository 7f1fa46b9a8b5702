set -u
OUT=gpurun_out/r02l; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_large.py -q -x > $OUT/pytest_shard_large.log 2>&1; echo "exit $?" >> $OUT/pytest_shard_large.log
timeout 900 python tools/make_frontier_fixture.py dag:20000 64 > $OUT/fixture.log 2>&1
cp bench_frontiers/dag_20000_64.json $OUT/ 2>/dev/null
for p in 4 8 12; do
  timeout 600 python bench.py --workload dag:20000 --parents $p --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/dag20k_p$p.json 2> $OUT/dag20k_p$p.err
done
timeout 1500 python -m pytest tests -q -x -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
echo done
