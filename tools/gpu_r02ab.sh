set -u
OUT=gpurun_out/r02ab; mkdir -p $OUT
for v in main reg; do
  if [ $v = reg ]; then L="EF_LIB=$PWD/exp/libef200_reg.so"; else L=""; fi
  env $L timeout 600 python bench.py --workload resnet50 --steps 10 --warmup 3 --no-cpu --no-extras > $OUT/r50_$v.json 2> $OUT/r50_$v.err
  env $L timeout 600 python bench.py --workload dag:20000 --steps 4 --warmup 3 --no-cpu --no-extras > $OUT/d20_$v.json 2> $OUT/d20_$v.err
  env $L timeout 600 python bench.py --workload inception_v3 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/inc_$v.json 2> $OUT/inc_$v.err
done
echo done
