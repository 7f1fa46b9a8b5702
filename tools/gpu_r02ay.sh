set -u
OUT=gpurun_out/r02ay; mkdir -p $OUT
EF_SPEC_PRICE=0 EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_price_v" -c 1 -o /tmp/prof_pr \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
ncu -i /tmp/prof_pr.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
ncu -i /tmp/prof_pr.ncu-rep --page source --csv --print-source cuda,sass > $OUT/prof_source.csv 2>/dev/null
gzip -f $OUT/prof_source.csv
echo done
