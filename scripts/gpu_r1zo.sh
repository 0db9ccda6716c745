# regression after K7 (4-GPU box): full GPU suite, bench N=1/4, alltoallv, MoE, full sweep (2 GPUs)
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/zo_pytest_gpu4.log 2>&1; echo pytest_rc=$? >> gpurun_out/zo_pytest_gpu4.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zo_smoke.log 2>&1; echo rc=$? >> gpurun_out/zo_smoke.log
timeout 180 python bench.py > gpurun_out/zo_bench_n1.log 2>&1
timeout 180 $R4 --master-port 29642 bench.py --gpus 4 > gpurun_out/zo_bench_n4.log 2>&1
timeout 300 $R4 --master-port 29646 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zo_a2a_n4.log 2>&1
timeout 300 $R4 --master-port 29644 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zo_moe_iccl_n4.log 2>&1
timeout 500 $R2 --master-port 29643 benchmarks/p2p_sweep.py --impl iccl-auto --max-pow 30 > gpurun_out/zo_sweep_iccl-auto.log 2>&1
