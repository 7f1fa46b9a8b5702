set -u
OUT=gpurun_out/r02ai; mkdir -p $OUT
for cfg in "4 9" "3 9" "1 9" "3 10" "3 8"; do set -- $cfg
  EF_SPEC_PRICE=$1 timeout 600 python bench.py --workload dag:20000 --parents $2 --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/d20_m$1_p$2.json 2> $OUT/d20_m$1_p$2.err
done
echo done
