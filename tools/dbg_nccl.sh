set -u
T="tests/test_gpu_nccl_one_rank.py::test_sweep_route_through_nccl"
for v in "" "FP_NO_PDL=1" "FP_K3_SHAPE=grid" "NCCL_PDL=0"; do
  echo "=== $v" >> gpurun_out/r2e_dbg.log
  env $v python -m pytest "$T" -q -p no:cacheprovider 2>&1 | tail -3 >> gpurun_out/r2e_dbg.log
done
env python -m pytest tests/test_gpu_nccl_one_rank.py -q -p no:cacheprovider 2>&1 | tail -15 >> gpurun_out/r2e_dbg.log
