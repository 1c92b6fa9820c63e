#!/bin/bash
# Bench line + ncu launch list + one full ncu capture of the dominant kernel.
# Usage (on the GPU box): bash tools/profile_bench.sh TAG [extra bench args]
set -u
TAG=$1; shift
OUT=gpurun_out
python bench.py "$@" > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err || { tail -20 $OUT/bench_$TAG.err; exit 1; }
DOM=$(python -c "import json;print(json.load(open('$OUT/bench_$TAG.json'))['roofline']['kernel'])")
echo "dominant kernel: $DOM"
export BENCH_ALLOW_SHORT=1
python bench.py "$@" --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > $OUT/plain_launches.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py "$@" --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > $OUT/ncu_launches_$TAG.log 2>&1
python bench.py "$@" --only "$DOM" --steps 1 --warmup 1 --no-cpu-baseline > $OUT/plain_dom.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:_decode_kernel -s 1 -c 1 \
    -o $OUT/prof_dom_$TAG python bench.py "$@" --only "$DOM" --steps 1 --warmup 1 --no-cpu-baseline \
    > $OUT/ncu_dom_$TAG.log 2>&1
tail -2 $OUT/ncu_dom_$TAG.log
