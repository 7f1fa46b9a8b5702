set -u
OUT=gpurun_out/r02k; mkdir -p $OUT
EF_NCU=1 timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_digest_pm|k_keys_wide|k_price_v|k_sortbig|k_dirty_big|k_merge_big" -c 6 -o $OUT/prof_dag20k \
    python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/prof.log 2>&1
echo done
