# round-1 GPU batch H (2 GPUs): debug the single-op LL->CE hang, NCCL MoE comparator, failover phases, LL-256 sweep
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 90 $R --master-port 29661 scripts/debug_sendrecv.py 32768 > gpurun_out/debug_ll32k.log 2>&1
timeout 90 $R --master-port 29662 scripts/debug_sendrecv.py 0 > gpurun_out/debug_ll0.log 2>&1
timeout 300 $R --master-port 29663 benchmarks/moe_alltoallv.py --impl nccl > gpurun_out/moe_nccl_n2.log 2>&1
timeout 300 $R --master-port 29664 benchmarks/failover.py > gpurun_out/failover_n2.log 2>&1
timeout 300 $R --master-port 29665 benchmarks/failover.py --chunk-mib 32 > gpurun_out/failover_n2_c32.log 2>&1
