set -u
OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k3_factored -s 2 -c 1 -o $OUT/r2b_k3f -f python tools/k3_only.py > $OUT/r2b_k3f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_cluster -s 2 -c 1 -o $OUT/r2b_k3c -f python tools/k3_c5_only.py C5 > $OUT/r2b_k3c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2b_launch_c5.csv python tools/k3_c5_only.py C5 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2b_launch_c2.csv python tools/k3_c5_only.py C2 10300000 > /dev/null 2>&1
for r in r2b_k3f r2b_k3c; do ncu -i $OUT/$r.ncu-rep --page raw --csv > $OUT/${r}_raw.csv 2>/dev/null; ncu -i $OUT/$r.ncu-rep --page source --csv > $OUT/${r}_src.csv 2>/dev/null; ncu -i $OUT/$r.ncu-rep --page details --csv > $OUT/${r}_details.csv 2>/dev/null; done
ls -la $OUT | grep r2b
