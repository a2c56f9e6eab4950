OUT=gpurun_out
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --collectives --steps 20 --warmup 3 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/coll_spec.json 2> $OUT/coll_spec.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --collectives --p2p --steps 20 --warmup 3 --no-next1 --no-next2 --no-next4 --no-k3-grid --no-configs --no-cpu-baseline --e2e-steps 0 > $OUT/coll_p2p.json 2> $OUT/coll_p2p.err
timeout 900 python -m pytest tests -x -q -m gpu -k "multirank or nccl" > $OUT/coll_pytest.log 2>&1; echo "rc=$?" >> $OUT/coll_pytest.log
