set -u
OUT=gpurun_out/r02u; mkdir -p $OUT
for v in 2 3 4; do for m in 0 1; do
  EF_LIB=$PWD/exp/libef200_pf$v.so EF_SPEC_PRICE=$m timeout 600 python bench.py --workload dag:20000 --parents 9 --steps 4 --warmup 3 --no-cpu --no-extras > $OUT/d20_pf${v}_s$m.json 2> $OUT/d20_pf${v}_s$m.err
done; done
EF_SPEC_PRICE=0 EF_NCU=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_price_v" -c 1 -o $OUT/prof_price_inc python bench.py --workload inception_v3 --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
echo done
