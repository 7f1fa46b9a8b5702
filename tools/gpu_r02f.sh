set -u
OUT=gpurun_out/r02f; mkdir -p $OUT
for i in 1 2; do
python exp/search_ab.py > $OUT/def_$i.json 2>&1
EF_PRICE_LANES=2 python exp/search_ab.py > $OUT/l2_$i.json 2>&1
EF_PRICE_LANES=0 python exp/search_ab.py > $OUT/l0_$i.json 2>&1
done
echo done
