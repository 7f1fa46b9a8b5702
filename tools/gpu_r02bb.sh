set -u
OUT=gpurun_out/r02bb; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/launch.log 2>&1
timeout 600 python bench.py --no-cpu --no-extras > $OUT/bench.json 2> $OUT/bench.err
EF_SPEC_PRICE=0 timeout 600 python bench.py --no-cpu --no-extras --steps 5 > $OUT/bench_s0.json 2> $OUT/bench_s0.err
echo done
