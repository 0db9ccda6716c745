export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
ICCL_DEBUG=1 timeout 300 $R4 --master-port 29681 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zg_a2a_dbg1.log 2>&1
ICCL_DEBUG=1 timeout 300 $R4 --master-port 29682 bench.py --gpus 4 --workload alltoallv --steps 10 --iccl-monitor 0 > gpurun_out/zg_a2a_dbg2.log 2>&1
grep -c 'slow device call' gpurun_out/zg_a2a_dbg*.log
