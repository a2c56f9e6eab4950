OUT=gpurun_out
TAG=${1:-sp}
timeout 1200 python -m pytest tests/test_gpu_speculate.py -x -q -m gpu > $OUT/${TAG}_pytest.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest.log
B="python bench.py --steps 50 --warmup 5 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0"
$B > $OUT/${TAG}_bench_spec.json 2> $OUT/${TAG}_bench_spec.err
$B --no-speculate > $OUT/${TAG}_bench_nospec.json 2> $OUT/${TAG}_bench_nospec.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 --no-variants > /dev/null 2>&1
