OUT=gpurun_out
TAG=${1:-k3lc}
for lc in 16 32 64 8; do
  FP_K3_LC=$lc python bench.py --steps 3 --warmup 3 --no-next1 --no-next2 --no-next4 --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/${TAG}_$lc.json 2> $OUT/${TAG}_$lc.err
done
FP_K3_LC=64 timeout 600 python -m pytest tests -x -q -m gpu -k "factored" > $OUT/${TAG}_pytest64.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest64.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "bin_pass or clamped or C3 or C2" > $OUT/${TAG}_pytest_bins.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest_bins.log
for c in C3 C2; do
python bench.py --config $c --steps 50 --warmup 5 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/${TAG}_bench_$c.json 2> $OUT/${TAG}_bench_$c.err
done
