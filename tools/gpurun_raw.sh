OUT=gpurun_out
TAG=${1:-raw}
timeout 1200 python -m pytest tests/test_gpu_speculate.py tests/test_gpu_estimate.py -x -q -m gpu > $OUT/${TAG}_pytest.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest.log
python bench.py --steps 10 --warmup 3 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
