# compute-sanitizer over the round-2 kernels (memcheck: per-tensor allocations so OOB is visible)
OUT=gpurun_out/san
mkdir -p $OUT
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 $CS --tool memcheck python tools/memcheck_canary.py > $OUT/canary.log 2>&1
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_calibrate.py -x -q -m gpu -k "not full_size" > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 1200 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "clamped or factored or bin_pass_misaligned" > $OUT/racecheck_parity.log 2>&1; echo "rc=$?" >> $OUT/racecheck_parity.log
timeout 1200 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_calibrate.py -x -q -m gpu > $OUT/racecheck_calib.log 2>&1; echo "rc=$?" >> $OUT/racecheck_calib.log
timeout 1200 $CS --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_calibrate.py -x -q -m gpu -k "clamped or factored or bin_pass_misaligned or calib" > $OUT/synccheck.log 2>&1; echo "rc=$?" >> $OUT/synccheck.log
unset PYTORCH_NO_CUDA_MEMORY_CACHING
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "random_prices or fallbacks" > $OUT/random_k3.log 2>&1; echo "rc=$?" >> $OUT/random_k3.log
