#!/bin/bash
# Round-2 profiling recipe (ONE GPU, under gpurun): launch lists of the bench's
# main step (speculative, the default, and --no-speculate), ncu --set full
# (+source) captures of every hot kernel, summaries and profiles/ncu_traffic.json.
set -u
TAG=${1:-r02a}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
MAIN="$BENCH --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-variants"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv $MAIN > $OUT/${TAG}_launches_bench.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches_nospec.csv $MAIN --no-speculate > $OUT/${TAG}_launches_nospec.log 2>&1
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s "$3" -c 1 \
      -o $OUT/${TAG}_$1 -f $4 > $OUT/${TAG}_$1.log 2>&1
  ncu -i $OUT/${TAG}_$1.ncu-rep --page raw --csv > $OUT/${TAG}_$1_raw.csv 2>/dev/null
  ncu -i $OUT/${TAG}_$1.ncu-rep --page details --csv > $OUT/${TAG}_$1_details.csv 2>/dev/null
  ncu -i $OUT/${TAG}_$1.ncu-rep --page source --csv > $OUT/${TAG}_$1_source.csv 2>/dev/null
}
# gpurun copies back at most 64 MiB of gpurun_out/: the reports are summarised
# below and then removed (the raw/details/source CSV exports stay)
# per step with speculation: K1 sample, K3 sample, K1 full, K3 full, K4v
cap sample k1_trace 2 "$MAIN"
cap trace k1_trace 3 "$MAIN"
cap sample_eval k3_cluster 2 "$MAIN"
cap eval k3_cluster 3 "$MAIN"
cap verify k4_route_verify 1 "$MAIN"
cap trace_ns k1_trace 3 "$MAIN --no-speculate"
cap route_ns k4_route_packed 3 "$MAIN --no-speculate"
cap k3_large "k3_(factored|grid|cluster)" 1 "python tools/k3_only.py"
cap c1_maps c1_maps 1 "python tools/calib_only.py --reps 1"
cap c3_replay c3_replay 1 "python tools/calib_only.py --reps 1"
cap k1w_hist k1w_hist 1 "$BENCH --no-next1 --no-next2 --no-k3-grid --no-configs --no-variants"
cp profiles/ncu_traffic.json $OUT/${TAG}_ncu_traffic.json
python tools/ncu_summary.py $OUT/${TAG}_summary.md \
  --traffic "$OUT/${TAG}_ncu_traffic.json@C5-spec=trace:trace,route:verify,eval:eval,sample:sample,sample_eval:sample_eval" \
  --traffic "$OUT/${TAG}_ncu_traffic.json@C5=trace:trace_ns,route:route_ns,eval:eval" \
  sample=$OUT/${TAG}_sample.ncu-rep trace=$OUT/${TAG}_trace.ncu-rep:1000000000 \
  sample_eval=$OUT/${TAG}_sample_eval.ncu-rep:4096 eval=$OUT/${TAG}_eval.ncu-rep:4096 \
  verify=$OUT/${TAG}_verify.ncu-rep trace_ns=$OUT/${TAG}_trace_ns.ncu-rep:1000000000 \
  route_ns=$OUT/${TAG}_route_ns.ncu-rep:1000000000 k3_large=$OUT/${TAG}_k3_large.ncu-rep:16777216 \
  c1_maps=$OUT/${TAG}_c1_maps.ncu-rep:1000000000 c3_replay=$OUT/${TAG}_c3_replay.ncu-rep:1000000000 \
  k1w_hist=$OUT/${TAG}_k1w_hist.ncu-rep:1000000000 > $OUT/${TAG}_summary.log 2>&1
rm -f $OUT/${TAG}_*.ncu-rep $OUT/${TAG}_*_source.csv
ls -la $OUT | grep $TAG
