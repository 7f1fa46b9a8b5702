set -u
OUT=gpurun_out/r02as; mkdir -p $OUT
EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_merge_scatter" -c 1 -o /tmp/prof_ms \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
ncu -i /tmp/prof_ms.ncu-rep --page raw --csv > $OUT/prof_raw.csv 2>/dev/null
ncu -i /tmp/prof_ms.ncu-rep --page source --csv --print-source cuda,sass > $OUT/prof_source.csv 2>/dev/null
gzip -f $OUT/prof_source.csv
python - <<'PY' > $OUT/dhist.txt 2>&1
import sys; sys.path.insert(0,'.')
PY
echo done
