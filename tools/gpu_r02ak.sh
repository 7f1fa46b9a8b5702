set -u
OUT=gpurun_out/r02ak; mkdir -p $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --sharded --workload resnet50 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/r50_sharded.json 2> $OUT/r50_sharded.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --sharded --workload dag:20000 --steps 3 --warmup 2 --no-cpu --no-extras > $OUT/d20_sharded.json 2> $OUT/d20_sharded.err
NCCL_DEBUG=INFO timeout 600 python bench.py --gpus 1 --sharded --workload squeezenet --steps 3 --warmup 3 --no-cpu --no-extras > $OUT/sq_sharded.json 2> $OUT/sq_sharded.err
echo done
