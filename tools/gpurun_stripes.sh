OUT=gpurun_out
B="python bench.py --steps 50 --warmup 5 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0"
for st in 6 4 3 2 6; do FP_SPEC_STRIPES=$st $B > $OUT/stripes_$st.json 2> $OUT/stripes_$st.err; done
