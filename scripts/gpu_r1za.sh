export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R4 --master-port 29646 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/za_bench_a2a_n4.log 2>&1
ICCL_DIRECT_MAX_KIB=0 timeout 300 $R4 --master-port 29647 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/za_bench_a2a_n4_nodirect.log 2>&1
nvidia-smi > gpurun_out/za_nvsmi.txt 2>&1
