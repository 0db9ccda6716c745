# round-1 GPU batch G (2 GPUs): per-file parity runs (hang isolation), multi-CTA LL sweep, kernels
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for t in test_pair_sendrecv_bytes test_pair_ll_small_messages test_pair_bidirectional test_ring_shift_all_gpus test_alltoallv_uneven_vs_oracle test_pair_failover_mid_message; do
  timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k $t > gpurun_out/pt_$t.log 2>&1; echo rc=$? >> gpurun_out/pt_$t.log
  mkdir -p gpurun_out/logs_$t; find /tmp/pytest-of-root -name "rank*.log" -exec cp --backup=numbered {} gpurun_out/logs_$t/ ; 2>/dev/null; rm -rf /tmp/pytest-of-root
done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 400 $R --master-port 29651 benchmarks/p2p_sweep.py --impl iccl-auto --ll-bytes 262144 --max-pow 22 > gpurun_out/sweep_iccl-ll256.log 2>&1
timeout 200 python benchmarks/kernels.py --only k2,k3 > gpurun_out/kernels_k23.log 2>&1
timeout 300 $R --master-port 29652 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/moe_iccl_n2.log 2>&1
timeout 300 $R --master-port 29653 benchmarks/moe_alltoallv.py --impl nccl > gpurun_out/moe_nccl_n2.log 2>&1
timeout 300 $R --master-port 29654 benchmarks/failover.py > gpurun_out/failover_n2.log 2>&1
