set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1_mon1.log 2>&1
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --monitor 0 > gpurun_out/bench_n1_mon0.log 2>&1
timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.log 2>&1
timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 10 --warmup 3 --monitor 0 > gpurun_out/bench_n2_mon0.log 2>&1
for impl in iccl-ce iccl-sm nccl; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 benchmarks/p2p_sweep.py --impl $impl --max-pow 28 > gpurun_out/sweep_$impl.log 2>&1; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 2 --workload alltoallv --steps 5 --warmup 3 > gpurun_out/bench_a2a_n2.log 2>&1
