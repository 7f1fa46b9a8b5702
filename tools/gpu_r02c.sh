set -u
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_models.py tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for cfg in "default::" "quadall:EF_QUAD_MAX=100000000:EF_WIDE_MIN=0" "quad_wide2k:EF_QUAD_MAX=100000000:EF_WIDE_MIN=2048" ; do
  name=${cfg%%:*}; rest=${cfg#*:}; e1=${rest%%:*}; e2=${rest#*:}
  env ${e1:+$e1} ${e2:+$e2} timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 2 --no-cpu > $OUT/dag20k_$name.json 2> $OUT/dag20k_$name.err
done
timeout 600 python bench.py --workload nasnet_a --steps 3 --warmup 2 --no-cpu > $OUT/nasnet.json 2> $OUT/nasnet.err
EF_QUAD_MAX=100000000 EF_WIDE_MIN=0 timeout 600 python bench.py --workload nasnet_a --steps 3 --warmup 2 --no-cpu > $OUT/nasnet_quad.json 2> $OUT/nasnet_quad.err
timeout 600 python tools/gpu_prof_search_cfg.py inception_v3 linear0.5 1.05 1000 64 > $OUT/prof_inc.txt 2>&1
echo done
