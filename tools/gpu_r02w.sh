set -u
OUT=gpurun_out/r02w; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_shard.py -q -x > $OUT/pytest_a.log 2>&1; echo "exit $?" >> $OUT/pytest_a.log
for p in 9 10 11; do
  timeout 600 python bench.py --workload dag:20000 --parents $p --steps 4 --warmup 3 --no-cpu --no-extras > $OUT/d20_p$p.json 2> $OUT/d20_p$p.err
done
for w in dag:1000 dag:5000 nasnet_a; do
  for cfg in "0 2" "0 1" "2048 2"; do set -- $cfg
    EF_SPEC_MIN_ROWS=$1 EF_SPEC_PRICE=$2 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/w_${w/:/_}_r$1_m$2.json 2> $OUT/w_${w/:/_}_r$1_m$2.err
  done
done
for l in 4 8; do
  EF_WIDE_LPC=$l timeout 600 python bench.py --workload dag:20000 --parents 9 --steps 4 --warmup 3 --no-cpu --no-extras > $OUT/d20_lpc$l.json 2> $OUT/d20_lpc$l.err
done
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --parents 9 --steps 2 --warmup 1 --no-cpu --no-extras > $OUT/launch.log 2>&1
EF_NCU=1 timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_keys_wide|k_digest_pm|k_dirty_big|k_sortbig|k_merge_big|k_price_v|k_keys<" -c 7 -o /tmp/prof \
    python bench.py --parents 9 --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
ncu -i /tmp/prof.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source cuda,sass > $OUT/prof_source.csv 2>/dev/null
gzip -f $OUT/prof_source.csv
ls -la $OUT
echo done
