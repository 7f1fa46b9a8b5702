set -u
OUT=gpurun_out/r02an; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_models.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_m1.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/launch_m1.log 2>&1
EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_merge_scatter" -c 1 -o /tmp/prof_ms \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
ncu -i /tmp/prof_ms.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
ncu -i /tmp/prof_ms.ncu-rep --page source --csv --print-source cuda,sass > $OUT/prof_source.csv 2>/dev/null
gzip -f $OUT/prof_source.csv
echo done
