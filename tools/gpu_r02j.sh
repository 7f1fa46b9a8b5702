set -u
OUT=gpurun_out/r02j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_large.py -q -x > $OUT/pytest_large.log 2>&1; echo "exit $?" >> $OUT/pytest_large.log
timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/dag20k.json 2> $OUT/dag20k.err
EF_FUSE_MERGE=0 timeout 600 python bench.py --workload dag:20000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/dag20k_fuse0.json 2> $OUT/dag20k_fuse0.err
timeout 600 python bench.py --workload resnet50 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/resnet.json 2> $OUT/resnet.err
timeout 600 python bench.py --workload nasnet_a --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/nasnet.json 2> $OUT/nasnet.err
timeout 1200 python -m pytest tests -q -x -m gpu > $OUT/pytest_all.log 2>&1; echo "exit $?" >> $OUT/pytest_all.log
echo done
