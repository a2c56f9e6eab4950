OUT=gpurun_out
for st in 1 2 4 8 16; do
  FP_K1_MIN_STEPS=$st python bench.py --config C2 --steps 200 --warmup 10 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/c2g_$st.json 2> $OUT/c2g_$st.err
done
