export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29636 benchmarks/failover.py --chunk-mib 32 > gpurun_out/failover_n2_c32.log 2>&1
timeout 300 $R --master-port 29637 benchmarks/failover.py --chunk-mib 8 > gpurun_out/failover_n2_c8.log 2>&1
timeout 180 $R --master-port 29631 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1
timeout 180 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
