# round-1 GPU batch D (2 GPUs): parity tests, kernel rooflines + ncu, sweeps vs NCCL, GEMM interference
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python benchmarks/kernels.py > gpurun_out/kernels.log 2>&1; echo rc=$? >> gpurun_out/kernels.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:iccl_ --csv --log-file gpurun_out/launches_kernels.csv python benchmarks/kernels.py --reps 2 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iccl_ -c 8 -o gpurun_out/kernels_full python benchmarks/kernels.py --reps 1 > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_sm.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --iccl-monitor 0 --transport sm > gpurun_out/ncu_bench_sm.log 2>&1
for impl in iccl-ce iccl-auto nccl; do timeout 400 $R --master-port 29622 benchmarks/p2p_sweep.py --impl $impl --max-pow 30 > gpurun_out/sweep_$impl.log 2>&1; done
timeout 400 $R --master-port 29623 benchmarks/p2p_sweep.py --impl iccl-sm --max-pow 28 > gpurun_out/sweep_iccl-sm.log 2>&1
NCCL_P2P_USE_CUDA_MEMCPY=1 timeout 400 $R --master-port 29624 benchmarks/p2p_sweep.py --impl nccl --max-pow 30 > gpurun_out/sweep_nccl-cemem.log 2>&1
for impl in none iccl-ce iccl-sm nccl; do timeout 300 $R --master-port 29625 benchmarks/gemm_interference.py --impl $impl --reps 20 > gpurun_out/gemm_$impl.log 2>&1; done
