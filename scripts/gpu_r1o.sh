# round-1 GPU batch O (2 GPUs): pull kernel, failover, 1F1B both impls, parity
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 200 python benchmarks/kernels.py --only k1_pull,k1_peer > gpurun_out/kernels_pull.log 2>&1
timeout 300 $R --master-port 29636 benchmarks/failover.py --chunk-mib 32 > gpurun_out/failover_n2_c32.log 2>&1
timeout 300 $R --master-port 29637 benchmarks/pp_1f1b.py --impl iccl > gpurun_out/pp_iccl_n2.log 2>&1
timeout 300 $R --master-port 29638 benchmarks/pp_1f1b.py --impl nccl > gpurun_out/pp_nccl_n2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
