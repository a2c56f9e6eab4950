OUT=gpurun_out
TAG=${1:-ch1}
timeout 900 python -m pytest tests/test_gpu_calibrate.py -x -q -k chunked > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
for c in 4 8 16; do FP_CALIB_CHUNKS=$c timeout 300 python tools/calib_only.py --reps 10 > $OUT/${TAG}_time_c$c.log 2>&1; done
FP_CALIB_SERIAL=1 timeout 300 python tools/calib_only.py --reps 10 > $OUT/${TAG}_time_serial.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python tools/calib_only.py --reps 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_full_size_next.py -x -q -k next3 > $OUT/${TAG}_full.log 2>&1; echo rc=$? >> $OUT/${TAG}_full.log
