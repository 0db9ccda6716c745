# round-1 GPU batch T (2 GPUs): sweeps vs NCCL, GEMM interference, 1F1B, kernels + ncu, smoke
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t_smoke.log 2>&1; echo rc=$? >> gpurun_out/t_smoke.log
timeout 500 $R --master-port 29622 benchmarks/p2p_sweep.py --impl iccl-auto --max-pow 30 > gpurun_out/t_sweep_iccl-auto.log 2>&1
timeout 500 $R --master-port 29623 benchmarks/p2p_sweep.py --impl nccl --max-pow 30 > gpurun_out/t_sweep_nccl.log 2>&1
NCCL_P2P_USE_CUDA_MEMCPY=1 timeout 500 $R --master-port 29624 benchmarks/p2p_sweep.py --impl nccl --max-pow 26 > gpurun_out/t_sweep_nccl-cemem.log 2>&1
for impl in none iccl-ce nccl; do timeout 300 $R --master-port 29625 benchmarks/gemm_interference.py --impl $impl --reps 30 > gpurun_out/t_gemm_$impl.log 2>&1; done
timeout 300 $R --master-port 29626 benchmarks/pp_1f1b.py --impl iccl > gpurun_out/t_pp_iccl_n2.log 2>&1
timeout 300 $R --master-port 29627 benchmarks/pp_1f1b.py --impl nccl > gpurun_out/t_pp_nccl_n2.log 2>&1
timeout 300 python benchmarks/kernels.py > gpurun_out/t_kernels.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iccl_ -c 4 -o gpurun_out/t_k2k3 python benchmarks/kernels.py --reps 1 --only k2,k3 > gpurun_out/t_ncu_k2k3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t_launches_kernels.csv python benchmarks/kernels.py --reps 2 > gpurun_out/t_ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/t_ncu_bench.log 2>&1
