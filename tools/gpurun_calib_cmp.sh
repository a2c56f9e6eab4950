# NEXT-3 A/B: the in-tree library ("new") vs variants under tools/libvariants/ (same script)
OUT=gpurun_out
TAG=${1:-cmp}; shift
for v in "$@"; do
  if [ $v = new ]; then unset FLEETPLAN_LIB; else export FLEETPLAN_LIB=tools/libvariants/$v.so; fi
  python tools/calib_only.py --reps 10 > $OUT/${TAG}_$v.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_${v}_launches.csv python tools/calib_only.py --reps 1 > /dev/null 2>&1
  timeout 600 python -m pytest tests -x -q -m gpu -k "calib" > $OUT/${TAG}_${v}_pytest.log 2>&1; echo rc=$? >> $OUT/${TAG}_${v}_pytest.log
done
unset FLEETPLAN_LIB
