export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for i in 1 2 3; do
timeout 300 $R4 --master-port 2965$i benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zc_moe_iccl_n4_$i.log 2>&1
timeout 300 $R4 --master-port 2966$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zc_bench_a2a_n4_$i.log 2>&1
done
ICCL_DEBUG=1 timeout 300 $R4 --master-port 29670 bench.py --gpus 4 --workload alltoallv --steps 4 > gpurun_out/zc_bench_a2a_dbg.log 2>&1
