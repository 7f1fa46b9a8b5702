set -u
OUT=gpurun_out/r02x; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_gpu_models.py tests/test_gpu_searches.py tests/test_gpu_shard.py -q -x > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for w in dag:20000 dag:5000 dag:1000 nasnet_a inception_v3 resnet50; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/w_${w/:/_}.json 2> $OUT/w_${w/:/_}.err
done
EF_NCU=1 timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_dirty_big|k_merge_big|k_digest_pm|k_prefix|k_keys_wide" -c 5 -o /tmp/prof \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
ncu -i /tmp/prof.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source cuda,sass > $OUT/prof_source.csv 2>/dev/null
gzip -f $OUT/prof_source.csv
echo done
