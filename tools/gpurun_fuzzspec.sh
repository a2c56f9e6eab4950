OUT=gpurun_out
TAG=${1:-fz1}
timeout 1500 python -m pytest tests/test_gpu_fuzz.py -x -q -k speculative -rs > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
