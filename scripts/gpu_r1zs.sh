# K6-class flags in GPU memory vs host-mapped (2 GPUs)
export PYTHONUNBUFFERED=1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/zs_pytest_gpu2.log 2>&1; echo pytest_rc=$? >> gpurun_out/zs_pytest_gpu2.log
for i in 1 2; do
timeout 300 $R2 --master-port 2967$i benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 24 > gpurun_out/zs_sweep_dflags_$i.log 2>&1
ICCL_DEVICE_FLAGS=0 timeout 300 $R2 --master-port 2968$i benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 24 > gpurun_out/zs_sweep_hflags_$i.log 2>&1
done
