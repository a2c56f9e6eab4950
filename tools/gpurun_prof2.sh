OUT=gpurun_out
T=r02c
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s "$3" -c 1 -o $OUT/${T}_$1 -f $4 > $OUT/${T}_$1.log 2>&1
  ncu -i $OUT/${T}_$1.ncu-rep --page raw --csv > $OUT/${T}_$1_raw.csv 2>/dev/null
  ncu -i $OUT/${T}_$1.ncu-rep --page details --csv > $OUT/${T}_$1_details.csv 2>/dev/null
}
cap c3_k1 k1_trace 2 "python tools/k3_c5_only.py C3 100000000"
cap c3_k4b k4_route_bins 2 "python tools/k3_c5_only.py C3 100000000"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${T}_launch_peak.csv python tools/peak_only.py --window-s 60 1 --reps 1 > $OUT/${T}_peak.log 2>&1
