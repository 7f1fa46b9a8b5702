set -u
OUT=gpurun_out/r02bd; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for w in inception_v3 nasnet_a dag:1000 dag:5000; do
  f=$(echo $w | tr ':' '_')
  timeout 600 python bench.py --workload $w --no-cpu --no-extras --steps 5 > $OUT/${f}.json 2>/dev/null
  EF_MS_MIN_ROWS=0 timeout 600 python bench.py --workload $w --no-cpu --no-extras --steps 5 > $OUT/${f}_ms0.json 2>/dev/null
done
timeout 600 python bench.py --no-cpu --no-extras --steps 5 > $OUT/dag_20000.json 2>/dev/null
echo done
