# round-1 GPU batch S (4 GPUs): final-design evidence at N=4
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s_pytest_gpu4.log 2>&1; echo pytest_rc=$? >> gpurun_out/s_pytest_gpu4.log
timeout 180 python bench.py > gpurun_out/s_bench_n1.log 2>&1
timeout 180 $R2 --master-port 29641 bench.py --gpus 2 > gpurun_out/s_bench_n2.log 2>&1
timeout 180 $R4 --master-port 29642 bench.py --gpus 4 > gpurun_out/s_bench_n4.log 2>&1
timeout 300 $R4 --master-port 29643 bench.py --gpus 4 --impl reference > gpurun_out/s_bench_ref_n4.log 2>&1
timeout 300 $R4 --master-port 29644 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/s_bench_a2a_n4.log 2>&1
timeout 300 $R4 --master-port 29645 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/s_moe_iccl_n4.log 2>&1
timeout 300 $R4 --master-port 29646 benchmarks/moe_alltoallv.py --impl nccl > gpurun_out/s_moe_nccl_n4.log 2>&1
timeout 300 $R4 --master-port 29647 benchmarks/failover.py --chunk-mib 32 > gpurun_out/s_failover_n4_sm.log 2>&1
timeout 300 $R4 --master-port 29648 benchmarks/failover.py --chunk-mib 32 --backup relay > gpurun_out/s_failover_n4_relay.log 2>&1
timeout 400 $R4 --master-port 29649 benchmarks/pp_1f1b.py --impl iccl > gpurun_out/s_pp_iccl_n4.log 2>&1
timeout 400 $R4 --master-port 29650 benchmarks/pp_1f1b.py --impl nccl > gpurun_out/s_pp_nccl_n4.log 2>&1
for impl in none iccl-ce nccl; do timeout 300 $R4 --master-port 29651 benchmarks/gemm_interference.py --impl $impl --reps 30 > gpurun_out/s_gemm4_$impl.log 2>&1; done
