set -u
OUT=gpurun_out/r02ad; mkdir -p $OUT
timeout 600 python tools/gpu_search_regress.py alone > $OUT/alone.log 2>&1
timeout 600 python tools/gpu_search_regress.py big > $OUT/big.log 2>&1
EF_SPEC_PRICE=0 timeout 600 python tools/gpu_search_regress.py alone > $OUT/alone_s0.log 2>&1
echo done
