set -u
# end-of-round evidence at HEAD: default bench line, launch lists and full captures of the
# DAG-20k and ResNet-50 steps, every BASELINE config as a workload line
OUT=gpurun_out/r02c; mkdir -p $OUT/d20 $OUT/r50
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/d20/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-extras > $OUT/d20/launch.log 2>&1
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r50/launches.csv \
    python bench.py --workload resnet50 --steps 2 --warmup 1 --no-cpu --no-extras > $OUT/r50/launch.log 2>&1
EF_NCU=1 timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_keys_wide|k_digest_pm|k_dirty_big|k_merge_scatter|k_merge_dir|k_prefix|k_pfx_chain|k_price_v|k_price_nsk|k_keys<" -c 10 -o /tmp/prof_d20 \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/d20/prof.log 2>&1
ncu -i /tmp/prof_d20.ncu-rep --page raw --csv > $OUT/d20/prof_raw.csv 2>/dev/null
EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_keys|k_digest_pm|k_dirty_warp|k_merge|k_price_v|k_match|k_plan|k_reach" -c 12 -o /tmp/prof_r50 \
    python bench.py --workload resnet50 --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/r50/prof.log 2>&1
ncu -i /tmp/prof_r50.ncu-rep --page raw --csv > $OUT/r50/prof_raw.csv 2>/dev/null
bash tools/gpu_workloads.sh r02c/workloads
echo done
