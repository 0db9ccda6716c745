# round-1 refresh after the premap / e2e changes (4-GPU box)
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 180 $R2 --master-port 29641 bench.py --gpus 2 > gpurun_out/zl_bench_n2.log 2>&1
timeout 180 $R4 --master-port 29642 bench.py --gpus 4 > gpurun_out/zl_bench_n4.log 2>&1
timeout 180 $R4 --master-port 29643 bench.py --gpus 4 --impl reference > gpurun_out/zl_bench_ref_n4.log 2>&1
for i in 1 2; do
timeout 300 $R4 --master-port 2965$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zl_a2a_n4_$i.log 2>&1
done
timeout 300 $R2 --master-port 29661 bench.py --gpus 2 --workload alltoallv --steps 10 > gpurun_out/zl_a2a_n2.log 2>&1
timeout 300 $R4 --master-port 29662 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zl_moe_iccl_n4.log 2>&1
timeout 300 $R4 --master-port 29663 benchmarks/moe_alltoallv.py --impl nccl > gpurun_out/zl_moe_nccl_n4.log 2>&1
timeout 300 $R4 --master-port 29664 benchmarks/failover.py --chunk-mib 32 > gpurun_out/zl_failover_n4.log 2>&1
timeout 300 $R4 --master-port 29665 benchmarks/failover.py --chunk-mib 32 --backup relay > gpurun_out/zl_failover_n4_relay.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/zl_pytest_gpu4.log 2>&1; echo pytest_rc=$? >> gpurun_out/zl_pytest_gpu4.log
