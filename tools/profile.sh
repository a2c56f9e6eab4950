#!/bin/bash
# Profiling recipe (run under gpurun on ONE GPU): launch list + ncu --set full
# captures of the hot kernels of one bench step. Outputs in gpurun_out/.
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
# 1. every launch with its device time (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_launches_bench.log 2>&1
# 2. full captures of the top kernels (after warm-up launches)
for K in k1_trace k4_route k3_eval; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
      -o $OUT/${TAG}_$K -f $BENCH > $OUT/${TAG}_${K}_bench.log 2>&1
  ncu -i $OUT/${TAG}_$K.ncu-rep --page raw --csv > $OUT/${TAG}_${K}_raw.csv 2>/dev/null
  ncu -i $OUT/${TAG}_$K.ncu-rep --page details --csv > $OUT/${TAG}_${K}_details.csv 2>/dev/null
  ncu -i $OUT/${TAG}_$K.ncu-rep --page source --csv > $OUT/${TAG}_${K}_source.csv 2>/dev/null
done
ls -la $OUT
