OUT=gpurun_out
python tools/k3_phases.py > $OUT/sm_phases.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/sm_launch_c2.csv python tools/k3_c5_only.py C2 10300000 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/sm_launch_c3.csv python tools/k3_c5_only.py C3 100000000 > /dev/null 2>&1
python bench.py --config C2 --steps 200 --warmup 10 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/sm_bench_c2.json 2> $OUT/sm_bench_c2.err
