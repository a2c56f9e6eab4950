OUT=gpurun_out
TAG=${1:-sp5}
timeout 900 python -m pytest tests/test_gpu_speculate.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
B="python bench.py --config C3 --no-cpu-baseline --e2e-steps 0 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs"
for n in 100000000 300000000 1000000000; do
  FP_SPEC_MIN_WIDE_LOG2=26 timeout 600 $B --n $n > $OUT/${TAG}_c3_spec_$n.json 2> $OUT/${TAG}_c3_spec_$n.err
  timeout 600 $B --n $n --no-speculate > $OUT/${TAG}_c3_nospec_$n.json 2> $OUT/${TAG}_c3_nospec_$n.err
done
