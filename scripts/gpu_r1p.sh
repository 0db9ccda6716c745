export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
ICCL_DEBUG=1 timeout 300 $R --master-port 29636 benchmarks/failover.py --chunk-mib 32 --steps 2 > gpurun_out/failover_dbg.log 2>&1
