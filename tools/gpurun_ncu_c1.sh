OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:c1_maps -s 1 -c 1 -o $OUT/r2e_c1 -f python tools/calib_only.py --reps 1 > $OUT/r2e_c1.log 2>&1
ncu -i $OUT/r2e_c1.ncu-rep --page raw --csv > $OUT/r2e_c1_raw.csv
ncu -i $OUT/r2e_c1.ncu-rep --page details --csv > $OUT/r2e_c1_details.csv
ncu -i $OUT/r2e_c1.ncu-rep --page source --csv > $OUT/r2e_c1_source.csv
