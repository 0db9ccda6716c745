export PYTHONUNBUFFERED=1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R2 --master-port 29671 benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 16 --max-pow 26 > gpurun_out/zn_sweep_auto.log 2>&1
ICCL_KERNEL_WAITS=0 timeout 300 $R2 --master-port 29672 benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 16 --max-pow 26 > gpurun_out/zn_sweep_auto_memop.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/zn_pytest_gpu2.log 2>&1; echo pytest_rc=$? >> gpurun_out/zn_pytest_gpu2.log
