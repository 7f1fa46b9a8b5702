set -u
OUT=gpurun_out/r02be; mkdir -p $OUT
EF_MS_MIN_ROWS=0 EF_MS_SORT_MIN=0 timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_large.py -q -x -p no:cacheprovider > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
for w in inception_v3 nasnet_a dag:1000 resnet50; do
  f=$(echo $w | tr ':' '_')
  timeout 600 python bench.py --workload $w --no-cpu --no-extras --steps 5 > $OUT/${f}.json 2>/dev/null
  EF_MS_MIN_ROWS=0 EF_MS_SORT_MIN=0 timeout 600 python bench.py --workload $w --no-cpu --no-extras --steps 5 > $OUT/${f}_all.json 2>/dev/null
  EF_MS_MIN_ROWS=0 EF_MS_SORT_MIN=512 timeout 600 python bench.py --workload $w --no-cpu --no-extras --steps 5 > $OUT/${f}_s512.json 2>/dev/null
done
echo done
