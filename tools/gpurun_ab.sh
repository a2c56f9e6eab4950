# A/B of library builds on the bench's main step (C5): tools/gpurun_ab.sh TAG variant...
# ("new" = the in-tree library; others = tools/libvariants/<name>.so), alternating twice
OUT=gpurun_out
TAG=$1; shift
B="python bench.py --steps 50 --warmup 5 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0"
for rep in 1 2; do
  for v in "$@"; do
    if [ $v = new ]; then unset FLEETPLAN_LIB; else export FLEETPLAN_LIB=tools/libvariants/$v.so; fi
    $B > $OUT/${TAG}_${v}_$rep.json 2> $OUT/${TAG}_${v}_$rep.err
  done
done
unset FLEETPLAN_LIB
