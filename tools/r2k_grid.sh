set -u
OUT=gpurun_out
mkdir -p $OUT
for part in c0 c1 c3 c2 c4; do
  rm -f $OUT/r2k_grid_$part.jsonl
  timeout 1500 python tools/grid.py $part --out $OUT/r2k_grid_$part.jsonl > $OUT/r2k_grid_$part.log 2>&1
  echo grid_$part=$?
done
wc -l $OUT/r2k_grid_*.jsonl
