set -u
OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 600 python tools/gpu_search_seq.py 1000 skip > $OUT/seq.txt 2>&1
EF_DIRTY_BIG=0 timeout 600 python tools/gpu_search_seq.py 1000 skip > $OUT/seq_dirty0.txt 2>&1
EF_WIDE_LPC=32 timeout 600 python tools/gpu_search_seq.py 1000 skip > $OUT/seq_lpc32.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_acceptance.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/dag20k.json 2> $OUT/dag20k.err
echo done
