# group lanes / group wait experiments (4 GPUs)
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for i in 1 2; do
timeout 300 $R4 --master-port 2971$i benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zp_moe_l1_$i.log 2>&1
ICCL_GROUP_LANES=2 timeout 300 $R4 --master-port 2972$i benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zp_moe_l2_$i.log 2>&1
ICCL_GROUP_LANES=3 timeout 300 $R4 --master-port 2973$i benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zp_moe_l3_$i.log 2>&1
timeout 300 $R4 --master-port 2974$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zp_a2a_l1_$i.log 2>&1
ICCL_GROUP_LANES=2 timeout 300 $R4 --master-port 2975$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zp_a2a_l2_$i.log 2>&1
ICCL_GROUP_SEND_WAIT_US=1000 timeout 300 $R4 --master-port 2976$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zp_a2a_w1000_$i.log 2>&1
done
