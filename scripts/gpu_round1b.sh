# round-1 GPU batch B (2 GPUs): parity tests, flag-placement probe, sweeps vs NCCL
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 60 ./probes/p2p_probe5 > gpurun_out/probe5.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 180 $R --master-port 29621 bench.py --gpus 2 --steps 10 --warmup 3 --iccl-monitor 0 > gpurun_out/bench_n2_mon0.log 2>&1
for impl in iccl-ce iccl-sm nccl; do timeout 400 $R --master-port 29622 benchmarks/p2p_sweep.py --impl $impl --max-pow 28 > gpurun_out/sweep2_$impl.log 2>&1; done
timeout 400 $R --master-port 29623 benchmarks/p2p_sweep.py --impl iccl-auto --ll-bytes 32768 --max-pow 20 > gpurun_out/sweep2_iccl-ll.log 2>&1
NCCL_P2P_USE_CUDA_MEMCPY=1 timeout 400 $R --master-port 29624 benchmarks/p2p_sweep.py --impl nccl --max-pow 28 > gpurun_out/sweep2_nccl-cemem.log 2>&1
for impl in none iccl-ce iccl-sm nccl; do timeout 300 $R --master-port 29625 benchmarks/gemm_interference.py --impl $impl --reps 20 > gpurun_out/gemm_$impl.log 2>&1; done
