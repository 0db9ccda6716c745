# same-process ready wait as a CUDA event (ICCL_EVENT_READY=1) vs the host-flag memop (=0, the default), 2 GPUs
export PYTHONUNBUFFERED=1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/zv_pytest_gpu2.log 2>&1; echo pytest_rc=$? >> gpurun_out/zv_pytest_gpu2.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zv_smoke.log 2>&1; echo rc=$? >> gpurun_out/zv_smoke.log
for i in 1 2; do
for v in 1 0; do
ICCL_EVENT_READY=$v timeout 200 $R2 --master-port 298$i$v benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 25 --max-pow 28 > gpurun_out/zv_sweep_ev${v}_$i.log 2>&1
done
done
