set -u
OUT=gpurun_out/r02ac; mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "exit $?" >> $OUT/smoke.log
( time timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err ) 2> $OUT/bench.time
( time timeout 1200 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err ) 2> $OUT/bench_ref.time
echo done
