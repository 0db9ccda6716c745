# K6 register copy (ICCL_K6_VEC_KIB) vs the TMA ring, 2 GPUs
export PYTHONUNBUFFERED=1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
ICCL_K6_VEC_KIB=16384 timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/zu_pytest_gpu2_vec.log 2>&1; echo pytest_rc=$? >> gpurun_out/zu_pytest_gpu2_vec.log
for i in 1 2; do
for v in 0 1024 16384; do
ICCL_K6_VEC_KIB=$v timeout 150 $R2 --master-port 297$i$((v % 7)) benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 18 --max-pow 24 > gpurun_out/zu_sweep_vec${v}_$i.log 2>&1
done
done
