OUT=gpurun_out
TAG=${1:-pk1}
timeout 900 python -m pytest tests/test_gpu_peak.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_pytest.log
timeout 300 python tools/peak_only.py --reps 10 > $OUT/${TAG}_time.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python tools/peak_only.py --reps 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_full_size_next.py -x -q -k next4 > $OUT/${TAG}_full.log 2>&1; echo rc=$? >> $OUT/${TAG}_full.log
