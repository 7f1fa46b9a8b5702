set -u
OUT=gpurun_out/r02aw; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_shard.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/launch.log 2>&1
timeout 600 python bench.py --no-cpu --no-extras > $OUT/bench.json 2> $OUT/bench.err
echo done
