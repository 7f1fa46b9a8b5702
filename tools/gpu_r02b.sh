set -u
OUT=gpurun_out/r02b; mkdir -p $OUT
timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 3 --no-cpu > $OUT/dag20k.json 2> $OUT/dag20k.err
EF_NCU=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_dag20k.csv python bench.py --workload dag:20000 --steps 1 --warmup 1 --no-cpu > $OUT/launches.log 2>&1
timeout 600 python tools/gpu_prof_search_cfg.py inception_v3 linear0.5 1.05 1000 64 > $OUT/prof_inc.txt 2>&1
timeout 600 python tools/gpu_prof_search_cfg.py nasnet_a energy 1.05 1000 64 > $OUT/prof_nas.txt 2>&1
echo done
