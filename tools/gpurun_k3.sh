OUT=gpurun_out
TAG=${1:-k3}
timeout 1200 python -m pytest tests -x -q -m gpu -k "factored or forced_k3 or k3" > $OUT/${TAG}_pytest.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest.log
python bench.py --steps 20 --warmup 5 --no-next1 --no-next2 --no-next4 --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launch_k3l.csv python tools/k3_only.py > /dev/null 2>&1
