# 2 GPUs: direct K6 path parity + sweep
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/x_pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/x_pytest_gpu.log
timeout 500 $R --master-port 29622 benchmarks/p2p_sweep.py --impl iccl-auto --max-pow 30 > gpurun_out/x_sweep_iccl-auto.log 2>&1
timeout 180 $R --master-port 29631 bench.py --gpus 2 > gpurun_out/x_bench_n2.log 2>&1
