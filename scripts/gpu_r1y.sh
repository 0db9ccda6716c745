export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
ICCL_DIRECT_MAX_KIB=16384 timeout 500 $R --master-port 29622 benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 25 > gpurun_out/y_sweep_direct.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "direct or ll_small or sendrecv_bytes" > gpurun_out/y_pytest.log 2>&1; echo rc=$? >> gpurun_out/y_pytest.log
