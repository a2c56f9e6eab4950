set -u
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/r2a_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/r2a_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r2a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r2a_smoke.log
timeout 900 python bench.py > $OUT/r2a_bench.json 2> $OUT/r2a_bench.err; echo "bench rc=$?" >> $OUT/r2a_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/r2a_bench_ref.json 2> $OUT/r2a_bench_ref.err
