OUT=gpurun_out
TAG=${1:-k4b}
B="python bench.py --config C3 --no-cpu-baseline --e2e-steps 0 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs"
for rep in 1 2; do
for v in base kq8; do
  FLEETPLAN_LIB=tools/libvariants/$v.so timeout 600 $B > $OUT/${TAG}_${v}_$rep.json 2> $OUT/${TAG}_${v}_$rep.err
  FP_K4_BLOCKS_PER_SM=4 FP_K4_BLOCK=256 FLEETPLAN_LIB=tools/libvariants/$v.so timeout 600 $B > $OUT/${TAG}_${v}_b256_$rep.json 2> $OUT/${TAG}_${v}_b256_$rep.err
done
done
