# K6-class flags in GPU memory (ICCL_DEVICE_FLAGS=1, default) vs host-mapped (=0), 2 GPUs
export PYTHONUNBUFFERED=1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/zs_pytest_gpu2.log 2>&1; echo pytest_rc=$? >> gpurun_out/zs_pytest_gpu2.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zs_smoke.log 2>&1; echo rc=$? >> gpurun_out/zs_smoke.log
for i in 1 2; do
timeout 150 $R2 --master-port 2967$i benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 24 > gpurun_out/zs_sweep_dflags_$i.log 2>&1
ICCL_DEVICE_FLAGS=0 timeout 150 $R2 --master-port 2968$i benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 24 > gpurun_out/zs_sweep_hflags_$i.log 2>&1
done
