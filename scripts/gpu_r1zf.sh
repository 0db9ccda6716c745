export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for i in 1 2; do
timeout 300 $R4 --master-port 2971$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zf_a2a_default_$i.log 2>&1
ICCL_GROUP_SEND_WAIT_US=2000 timeout 300 $R4 --master-port 2972$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zf_a2a_wait2ms_$i.log 2>&1
ICCL_GROUP_SEND_WAIT_US=20000 timeout 300 $R4 --master-port 2974$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zf_a2a_wait20ms_$i.log 2>&1
timeout 300 $R4 --master-port 2973$i benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zf_moe_$i.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/zf_pytest_gpu4.log 2>&1
