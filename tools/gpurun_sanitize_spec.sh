OUT=gpurun_out/san2
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1800 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_speculate.py -x -q -m gpu > $OUT/memcheck_spec.log 2>&1; echo "rc=$?" >> $OUT/memcheck_spec.log
timeout 1800 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_speculate.py -x -q -m gpu -k "hit" > $OUT/racecheck_spec.log 2>&1; echo "rc=$?" >> $OUT/racecheck_spec.log
timeout 1800 $CS --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_speculate.py -x -q -m gpu > $OUT/synccheck_spec.log 2>&1; echo "rc=$?" >> $OUT/synccheck_spec.log
timeout 1200 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "clamped or bin_pass_misaligned or factored" > $OUT/memcheck_parity.log 2>&1; echo "rc=$?" >> $OUT/memcheck_parity.log
