set -u
OUT=gpurun_out/r02i; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py -q > $OUT/pytest_large.log 2>&1; echo "exit $?" >> $OUT/pytest_large.log
timeout 600 python tools/gpu_search_seq.py 1000 > $OUT/seq.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/dag20k.json 2> $OUT/dag20k.err
EF_DIGEST_PF=0 timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/dag20k_pf0.json 2> $OUT/dag20k_pf0.err
echo done
