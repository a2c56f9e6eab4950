OUT=gpurun_out
TAG=${1:-pk}
timeout 1200 python -m pytest tests -x -q -m gpu -k "peak" > $OUT/${TAG}_pytest.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest.log
python tools/peak_only.py --window-s 60 1 0.1 --reps 5 > $OUT/${TAG}_peak.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launch_peak.csv python tools/peak_only.py --window-s 60 1 --reps 1 > /dev/null 2>&1
