set -u
OUT=gpurun_out/r02h; mkdir -p $OUT
for L in default exp/libef_w5.so exp/libef_w6.so; do
  T=$(basename $L .so)
  if [ $L = default ]; then unset EF_LIB; else export EF_LIB=$PWD/$L; fi
  timeout 600 python bench.py --no-cpu --no-extras --steps 5 > $OUT/bench_$T.json 2>/dev/null
  timeout 600 python bench.py --workload dag:5000 --no-cpu --no-extras --steps 5 > $OUT/d5_$T.json 2>/dev/null
done
echo done
