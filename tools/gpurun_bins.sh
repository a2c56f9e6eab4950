OUT=gpurun_out
TAG=${1:-bins}
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "bin_pass or clamped or full_size or route" > $OUT/${TAG}_pytest.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest.log
for c in C3 C2 C4; do
python bench.py --config $c --steps 50 --warmup 5 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/${TAG}_bench_$c.json 2> $OUT/${TAG}_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launch_c3.csv python tools/k3_c5_only.py C3 100000000 > /dev/null 2>&1
