set -u
OUT=gpurun_out/r02aa; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py -q -x > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
timeout 600 python bench.py --workload dag:20000 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d20.json 2> $OUT/d20.err
timeout 600 python bench.py --workload dag:5000 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d5.json 2> $OUT/d5.err
# launch lists (timed steps only) of both bench lines
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-extras > $OUT/launch.log 2>&1
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r50.csv \
    python bench.py --workload resnet50 --steps 2 --warmup 1 --no-cpu --no-extras > $OUT/launch_r50.log 2>&1
# full captures: the DAG-20k step's kernels, then ResNet-50's
EF_NCU=1 timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_keys_wide|k_digest_pm|k_dirty_big|k_sortbig|k_merge_big|k_prefix|k_price_v|k_keys<" -c 8 -o /tmp/prof \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
ncu -i /tmp/prof.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_keys|k_digest_pm|k_dirty_warp|k_merge|k_price_v|k_match|k_plan|k_reach" -c 12 -o /tmp/prof_r50 \
    python bench.py --workload resnet50 --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof_r50.log 2>&1
ncu -i /tmp/prof_r50.ncu-rep --page raw --csv > $OUT/prof_r50_raw.csv 2>/dev/null
ncu -i /tmp/prof_r50.ncu-rep --page source --csv --print-source cuda,sass > $OUT/prof_r50_source.csv 2>/dev/null
gzip -f $OUT/prof_r50_source.csv
ls -la $OUT
echo done
