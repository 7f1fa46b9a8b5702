set -u
OUT=gpurun_out/r02r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_models.py -q -x > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for m in 0 1 2; do
  EF_SPEC_PRICE=$m timeout 600 python bench.py --workload dag:20000 --parents 9 --steps 3 --warmup 3 --no-cpu --no-extras > $OUT/dag20k_s$m.json 2> $OUT/dag20k_s$m.err
  EF_SPEC_PRICE=$m timeout 600 python bench.py --workload resnet50 --steps 10 --warmup 3 --no-cpu --no-extras > $OUT/r50_s$m.json 2> $OUT/r50_s$m.err
done
EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_sortbig|k_merge_big" -c 2 -o $OUT/prof_sort python bench.py --parents 8 --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
echo done
