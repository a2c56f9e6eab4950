OUT=gpurun_out
TAG=${1:-c1p}
for rep in 1 2; do
for v in c1base c1pair; do
  FLEETPLAN_LIB=tools/libvariants/$v.so timeout 300 python tools/calib_only.py --reps 10 > $OUT/${TAG}_${v}_$rep.log 2>&1
done
done
FLEETPLAN_LIB=tools/libvariants/c1pair.so timeout 600 python -m pytest tests/test_gpu_calibrate.py -x -q > $OUT/${TAG}_c1pair_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_c1pair_pytest.log
for v in c1base c1pair; do
  FLEETPLAN_LIB=tools/libvariants/$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_${v}_launches.csv python tools/calib_only.py --reps 1 > /dev/null 2>&1
done
