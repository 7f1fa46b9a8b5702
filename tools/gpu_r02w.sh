set -u
OUT=gpurun_out/r02w; mkdir -p $OUT
for w in dag:1000 dag:5000 nasnet_a; do
  for cfg in "0 2" "0 1" "2048 2"; do set -- $cfg
    EF_SPEC_MIN_ROWS=$1 EF_SPEC_PRICE=$2 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-extras > $OUT/w_${w/:/_}_r$1_m$2.json 2> $OUT/w_${w/:/_}_r$1_m$2.err
  done
done
EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --parents 9 --steps 2 --warmup 1 --no-cpu --no-extras > $OUT/launch.log 2>&1
EF_NCU=1 timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -c 40 -o $OUT/prof \
    python bench.py --parents 9 --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/prof.log 2>&1
echo done
