set -u
OUT=gpurun_out/r02e; mkdir -p $OUT
timeout 600 python tools/make_frontier_fixture.py dag:20000 32 > $OUT/fixture.log 2>&1
cp bench_frontiers/*.json $OUT/ 2>/dev/null
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err
EF_NCU=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_dag20k.csv python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/launches.log 2>&1
echo done
