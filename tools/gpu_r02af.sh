set -u
OUT=gpurun_out/r02af; mkdir -p $OUT
PROF=1 timeout 600 python tools/gpu_search_regress.py alone inception_v3:1.05:1000 > $OUT/inc_alone.log 2>&1
timeout 600 python tools/gpu_search_regress.py big inception_v3:1.05:1000 > $OUT/inc_big.log 2>&1
EF_SPEC_PRICE=0 timeout 600 python tools/gpu_search_regress.py alone inception_v3:1.05:1000 > $OUT/inc_alone_s0.log 2>&1
echo done
