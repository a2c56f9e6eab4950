OUT=gpurun_out
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_speculate.py -q -m gpu > $OUT/flaky_$i.log 2>&1; echo "rc=$?" >> $OUT/flaky_$i.log
done
FP_NO_PDL=1 timeout 900 python -m pytest tests/test_gpu_speculate.py -q -m gpu > $OUT/flaky_nopdl.log 2>&1; echo "rc=$?" >> $OUT/flaky_nopdl.log
