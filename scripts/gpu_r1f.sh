# round-1 GPU batch F (4 GPUs): parity incl. relay, bench N=1/2/4, alltoallv, failover (sm / relay), GEMM interference, K2/K3 ncu
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu4.log
timeout 180 python bench.py > gpurun_out/bench4_n1.log 2>&1
timeout 180 $R2 --master-port 29641 bench.py --gpus 2 > gpurun_out/bench4_n2.log 2>&1
timeout 180 $R4 --master-port 29642 bench.py --gpus 4 > gpurun_out/bench4_n4.log 2>&1
timeout 180 $R4 --master-port 29643 bench.py --gpus 4 --iccl-monitor 0 > gpurun_out/bench4_n4_mon0.log 2>&1
timeout 300 $R4 --master-port 29644 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/bench4_a2a_n4.log 2>&1
timeout 300 $R4 --master-port 29645 benchmarks/failover.py > gpurun_out/failover_n4_sm.log 2>&1
timeout 300 $R4 --master-port 29646 benchmarks/failover.py --backup relay > gpurun_out/failover_n4_relay.log 2>&1
for impl in none iccl-ce nccl; do timeout 300 $R4 --master-port 29647 benchmarks/gemm_interference.py --impl $impl --reps 30 > gpurun_out/gemm4_$impl.log 2>&1; done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:iccl_ -c 2 -o gpurun_out/k2k3_full python benchmarks/kernels.py --reps 1 --only k2,k3 > gpurun_out/ncu_k2k3.log 2>&1
timeout 200 python benchmarks/kernels.py --only k1_local,k2,k3 > gpurun_out/kernels4.log 2>&1
