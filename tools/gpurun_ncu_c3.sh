OUT=gpurun_out
TAG=${1:-c3k1}
B="python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_trace -s 3 -c 1 -o $OUT/${TAG}_k1 -f $B > $OUT/${TAG}_k1.log 2>&1
ncu -i $OUT/${TAG}_k1.ncu-rep --page raw --csv > $OUT/${TAG}_k1_raw.csv 2>/dev/null
ncu -i $OUT/${TAG}_k1.ncu-rep --page source --csv > $OUT/${TAG}_k1_source.csv 2>/dev/null
ncu -i $OUT/${TAG}_k1.ncu-rep --page details --csv > $OUT/${TAG}_k1_details.csv 2>/dev/null
rm -f $OUT/${TAG}_k1.ncu-rep
