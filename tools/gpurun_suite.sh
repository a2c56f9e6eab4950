# full GPU suite + bench configs (TAG)
OUT=gpurun_out
TAG=${1:-suite}
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/${TAG}_pytest.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest.log
python bench.py --config C3 --steps 50 --warmup 5 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/${TAG}_bench_c3.json 2> $OUT/${TAG}_bench_c3.err
