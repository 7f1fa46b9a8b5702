set -u
OUT=gpurun_out/r02z; mkdir -p $OUT
for m in 3 1 2 0; do
  EF_SPEC_PRICE=$m timeout 600 python bench.py --workload dag:20000 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d20_m$m.json 2> $OUT/d20_m$m.err
done
for m in 3 2; do
  EF_SPEC_PRICE=$m timeout 600 python bench.py --workload dag:5000 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d5_m$m.json 2> $OUT/d5_m$m.err
done
EF_SPEC_PRICE=3 timeout 600 python bench.py --workload dag:20000 --parents 10 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d20_m3_p10.json 2> $OUT/d20_m3_p10.err
echo done
