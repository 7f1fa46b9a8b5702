set -u
OUT=gpurun_out/r02ax; mkdir -p $OUT
for M in -1 0 1 2 3 4; do
  EF_SPEC_PRICE=$M timeout 600 python bench.py --no-cpu --no-extras --steps 5 > $OUT/bench_s$M.json 2> $OUT/bench_s$M.err
done
echo done
