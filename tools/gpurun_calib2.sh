# NEXT-3 streaming replay: parity, timing (stream vs two-pass), launch list
OUT=gpurun_out
TAG=${1:-cs1}
timeout 600 python -m pytest tests/test_gpu_calibrate.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
FP_CALIB_VERBOSE=1 timeout 120 python tools/calib_only.py --reps 10 > $OUT/${TAG}_time_stream.log 2>&1
FP_CALIB_TWOPASS=1 timeout 120 python tools/calib_only.py --reps 10 > $OUT/${TAG}_time_twopass.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python tools/calib_only.py --reps 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_full_size_next.py -x -q -k next3 > $OUT/${TAG}_full.log 2>&1; echo rc=$? >> $OUT/${TAG}_full.log
