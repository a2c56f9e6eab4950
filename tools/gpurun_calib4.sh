OUT=gpurun_out
TAG=${1:-cs4}
FP_CALIB_STREAM=1 FP_CALIB_VERBOSE=1 FP_CALIB_PROFILE=1 timeout 120 python tools/calib_only.py --reps 3 > $OUT/${TAG}_prof.log 2>&1
timeout 300 python -m pytest tests/test_gpu_calibrate.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
FP_CALIB_STREAM=1 timeout 120 python tools/calib_only.py --reps 10 > $OUT/${TAG}_time_stream.log 2>&1
timeout 120 python tools/calib_only.py --reps 10 > $OUT/${TAG}_time_twopass.log 2>&1
