# round-1 GPU batch N (2 GPUs): second-arriver issue with senders waiting to come second
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 120 $R --master-port 29671 scripts/diag_ring.py > gpurun_out/diag_ring_mon1.log 2>&1
timeout 70 $R --master-port 29661 scripts/debug_sendrecv.py 32768 > gpurun_out/debug_ll32k.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 180 python bench.py > gpurun_out/bench_n1.log 2>&1
timeout 180 $R --master-port 29631 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1
timeout 180 $R --master-port 29632 bench.py --gpus 2 --iccl-monitor 0 --no-cpu-baseline > gpurun_out/bench_n2_mon0.log 2>&1
timeout 300 $R --master-port 29633 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/moe_iccl_n2.log 2>&1
timeout 300 $R --master-port 29636 benchmarks/failover.py --chunk-mib 32 > gpurun_out/failover_n2_c32.log 2>&1
timeout 300 $R --master-port 29637 benchmarks/pp_1f1b.py --impl iccl > gpurun_out/pp_iccl_n2.log 2>&1
timeout 300 $R --master-port 29638 benchmarks/pp_1f1b.py --impl nccl > gpurun_out/pp_nccl_n2.log 2>&1
timeout 400 $R --master-port 29634 benchmarks/p2p_sweep.py --impl iccl-auto --max-pow 30 > gpurun_out/sweep_iccl-auto.log 2>&1
