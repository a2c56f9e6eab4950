#!/bin/bash
# Profiling recipe (run under gpurun on ONE GPU): the launch list of the bench
# command, then ncu --set full captures of each hot kernel, then a markdown
# summary. Outputs in gpurun_out/ (copy what is judged into profiles/).
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
# 1. every launch of the bench command with its device time (cold-cache, serialised: compare shares)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_launches_bench.log 2>&1
# 2. full captures: name, kernel regex, launches to skip, command
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s "$3" -c 1 \
      -o $OUT/${TAG}_$1 -f $4 > $OUT/${TAG}_$1.log 2>&1
  ncu -i $OUT/${TAG}_$1.ncu-rep --page raw --csv > $OUT/${TAG}_$1_raw.csv 2>/dev/null
  ncu -i $OUT/${TAG}_$1.ncu-rep --page details --csv > $OUT/${TAG}_$1_details.csv 2>/dev/null
}
MAIN="$BENCH --no-next1 --no-next2 --no-next4 --no-k3-grid"
cap trace k1_trace 3 "$MAIN"
cap route k4_route_packed 3 "$MAIN"
cap eval k3_eval 3 "$MAIN"
RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=29561 cap pick_nccl k_pick_route 3 "$MAIN --collectives"
cap k1_raw k1_trace 2 "python tools/raw_only.py 1000000000"
cap k4_raw k4_route_raw 2 "python tools/raw_only.py 1000000000"
cap c1_maps c1_maps 1 "python tools/calib_only.py --reps 1"
cap c3_replay c3_replay 1 "python tools/calib_only.py --reps 1"
cap k1w_hist k1w_hist 1 "$BENCH --no-next1 --no-next2 --no-k3-grid"
cap k2w_peaks k2w_peaks 1 "$BENCH --no-next1 --no-next2 --no-k3-grid"
cap k3_large k3_eval 1 "python tools/k3_only.py"
ls -la $OUT
