OUT=gpurun_out
TAG=${1:-sp4}
timeout 900 python -m pytest tests/test_gpu_speculate.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size_configs and C3" > $OUT/${TAG}_full_c3.log 2>&1; echo rc=$? >> $OUT/${TAG}_full_c3.log
timeout 600 python bench.py --config C3 --no-cpu-baseline --e2e-steps 0 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs > $OUT/${TAG}_bench_c3.json 2> $OUT/${TAG}_bench_c3.err
timeout 600 python bench.py --config C3 --no-speculate --no-cpu-baseline --e2e-steps 0 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs > $OUT/${TAG}_bench_c3_nospec.json 2> $OUT/${TAG}_bench_c3_nospec.err
