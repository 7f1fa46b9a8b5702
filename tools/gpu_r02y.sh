set -u
OUT=gpurun_out/r02y; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py -q > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for w in dag:20000 dag:5000 dag:1000; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/w_${w/:/_}.json 2> $OUT/w_${w/:/_}.err
done
EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_prefix|k_merge_big|k_sortbig" -c 3 -o /tmp/prof \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
ncu -i /tmp/prof.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source cuda,sass > $OUT/prof_source.csv 2>/dev/null
gzip -f $OUT/prof_source.csv
echo done
