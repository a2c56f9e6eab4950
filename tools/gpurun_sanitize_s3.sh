# session-3 code under compute-sanitizer: u16-LUT speculation, the captured step graph,
# the streaming calibration kernel (opt-in), K0w interpolation; plus the fixed graph test
OUT=gpurun_out/san3
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q > $OUT/pytest_graph.log 2>&1; echo "rc=$?" >> $OUT/pytest_graph.log
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1800 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_speculate.py -x -q -m gpu -k wide > $OUT/memcheck_spec_wide.log 2>&1; echo "rc=$?" >> $OUT/memcheck_spec_wide.log
timeout 1800 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_speculate.py -x -q -m gpu -k wide > $OUT/racecheck_spec_wide.log 2>&1; echo "rc=$?" >> $OUT/racecheck_spec_wide.log
timeout 1800 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_graph.py -x -q -m gpu -k "C1 or C2 or refuses" > $OUT/memcheck_graph.log 2>&1; echo "rc=$?" >> $OUT/memcheck_graph.log
timeout 1800 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_calibrate.py -x -q -m gpu -k "True and (37 or 100003 or skew or one_sided)" > $OUT/memcheck_calib_stream.log 2>&1; echo "rc=$?" >> $OUT/memcheck_calib_stream.log
timeout 1800 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_calibrate.py -x -q -m gpu -k "True and (37 or 100003)" > $OUT/racecheck_calib_stream.log 2>&1; echo "rc=$?" >> $OUT/racecheck_calib_stream.log
timeout 1800 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_peak.py -x -q -m gpu > $OUT/memcheck_peak.log 2>&1; echo "rc=$?" >> $OUT/memcheck_peak.log
