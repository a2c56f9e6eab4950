# the C5 step at several trace sizes (requests per GPU): throughput vs size
OUT=gpurun_out/size_sweep
mkdir -p $OUT
for n in 100000000 300000000 1000000000 4000000000; do
  timeout 900 python bench.py --n $n --no-cpu-baseline --e2e-steps 0 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs > $OUT/c5_$n.json 2> $OUT/c5_$n.err
done
