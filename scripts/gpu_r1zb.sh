# 4 GPUs: hoisted group waits; parity; alltoallv; ring; sweep with SMs used
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R4 --master-port 29645 benchmarks/moe_alltoallv.py --impl iccl --dump-records > gpurun_out/zb_moe_records_n4.log 2>&1
timeout 300 $R4 --master-port 29646 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zb_moe_iccl_n4.log 2>&1
timeout 300 $R4 --master-port 29647 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zb_bench_a2a_n4.log 2>&1
timeout 180 $R4 --master-port 29648 bench.py --gpus 4 > gpurun_out/zb_bench_n4.log 2>&1
timeout 300 $R2 --master-port 29649 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zb_moe_iccl_n2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/zb_pytest_gpu4.log 2>&1; echo pytest_rc=$? >> gpurun_out/zb_pytest_gpu4.log
timeout 500 $R2 --master-port 29650 benchmarks/p2p_sweep.py --impl iccl-auto --max-pow 30 > gpurun_out/zb_sweep_iccl-auto.log 2>&1
