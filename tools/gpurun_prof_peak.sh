OUT=gpurun_out
T=r02d
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s "$3" -c 1 -o $OUT/${T}_$1 -f $4 > $OUT/${T}_$1.log 2>&1
  ncu -i $OUT/${T}_$1.ncu-rep --page raw --csv > $OUT/${T}_$1_raw.csv 2>/dev/null
  ncu -i $OUT/${T}_$1.ncu-rep --page details --csv > $OUT/${T}_$1_details.csv 2>/dev/null
  ncu -i $OUT/${T}_$1.ncu-rep --page source --csv > $OUT/${T}_$1_source.csv 2>/dev/null
}
cap k0w "k0w_bounds" 1 "python tools/peak_only.py --window-s 1 --reps 1"
cap k2w "k2w_peaks" 1 "python tools/peak_only.py --window-s 1 --reps 1"
cap k1w "k1w_hist" 1 "python tools/peak_only.py --window-s 1 --reps 1"
