set -u
OUT=gpurun_out/r02f; mkdir -p $OUT
CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/gpu_prof_search_cfg.py nasnet_a energy 1.05 300 64 > $OUT/nas_search.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --show-backtrace no --print-limit 5 python tools/gpu_prof_search_cfg.py nasnet_a energy 1.05 60 64 > $OUT/nas_memcheck.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
echo done
