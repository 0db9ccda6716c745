# K6 tile size: adaptive (8/16/32 KiB) vs fixed 32 KiB (2 GPUs)
export PYTHONUNBUFFERED=1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for i in 1 2; do
timeout 300 $R2 --master-port 2967$i benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 24 > gpurun_out/zq_sweep_adaptive_$i.log 2>&1
ICCL_DIRECT_TILE_KIB=32 timeout 300 $R2 --master-port 2968$i benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 24 > gpurun_out/zq_sweep_t32_$i.log 2>&1
done
ICCL_DIRECT_TILE_KIB=4 timeout 300 $R2 --master-port 29691 benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 24 > gpurun_out/zq_sweep_t4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "direct or ll or pair" > gpurun_out/zq_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/zq_pytest.log
