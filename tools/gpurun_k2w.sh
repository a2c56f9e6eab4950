OUT=gpurun_out
T=${1:-r02e}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2w_peaks -s 1 -c 1 -o $OUT/${T}_k2w -f python tools/peak_only.py --window-s 1 --reps 1 > $OUT/${T}_k2w.log 2>&1
ncu -i $OUT/${T}_k2w.ncu-rep --page raw --csv > $OUT/${T}_k2w_raw.csv 2>/dev/null
ncu -i $OUT/${T}_k2w.ncu-rep --page source --csv > $OUT/${T}_k2w_source.csv 2>/dev/null
