OUT=gpurun_out
TAG=${1:-pkd}
for rep in 1 2; do
for v in pk_cur pk_noflush pk_onepass; do
  FLEETPLAN_LIB=tools/libvariants/$v.so timeout 300 python tools/peak_only.py --reps 20 > $OUT/${TAG}_${v}_$rep.log 2>&1
done
done
