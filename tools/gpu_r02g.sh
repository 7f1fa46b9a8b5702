set -u
OUT=gpurun_out/r02g; mkdir -p $OUT
CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/gpu_search_seq.py 1000 > $OUT/seq_blocking.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck --show-backtrace no --print-limit 5 python tools/gpu_search_seq.py 40 > $OUT/seq_memcheck.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
echo done
