export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R4 --master-port 29651 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zd_a2a_default.log 2>&1
timeout 300 $R4 --master-port 29652 bench.py --gpus 4 --workload alltoallv --steps 10 --iccl-monitor 0 > gpurun_out/zd_a2a_mon0.log 2>&1
ICCL_BENCH_NO_CLOCKS=1 timeout 300 $R4 --master-port 29653 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zd_a2a_noclk.log 2>&1
ICCL_BENCH_NO_CLOCKS=1 timeout 300 $R4 --master-port 29654 bench.py --gpus 4 --workload alltoallv --steps 10 --iccl-monitor 0 > gpurun_out/zd_a2a_noclk_mon0.log 2>&1
timeout 300 $R4 --master-port 29655 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zd_moe.log 2>&1
