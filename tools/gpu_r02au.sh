set -u
OUT=gpurun_out/r02au; mkdir -p $OUT
for L in default exp/libef_d8192.so exp/libef_d16384.so; do
  T=$(basename $L .so)
  if [ $L = default ]; then unset EF_LIB; else export EF_LIB=$PWD/$L; fi
  EF_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file $OUT/launches_$T.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > $OUT/launch_$T.log 2>&1
done
echo done
