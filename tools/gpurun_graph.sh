OUT=gpurun_out
TAG=${1:-gr1}
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
timeout 600 python tools/graph_bench.py > $OUT/${TAG}_bench.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 0 --no-next1 --no-next2 --no-next4 --no-k3-grid > $OUT/${TAG}_mainbench.json 2> $OUT/${TAG}_mainbench.err
