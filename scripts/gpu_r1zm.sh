export PYTHONUNBUFFERED=1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R2 --master-port 29671 benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 10 --max-pow 22 > gpurun_out/zm_sweep_auto.log 2>&1
timeout 300 $R2 --master-port 29672 benchmarks/p2p_sweep.py --impl iccl-auto --ll-bytes 0 --min-pow 10 --max-pow 22 > gpurun_out/zm_sweep_k6.log 2>&1
timeout 300 $R2 --master-port 29673 benchmarks/p2p_sweep.py --impl nccl --min-pow 10 --max-pow 22 > gpurun_out/zm_sweep_nccl.log 2>&1
