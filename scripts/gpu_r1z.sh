# round-1 final evidence (4-GPU box): parity, bench N=1/2/4 + reference arm, sweep vs NCCL, alltoallv, failover
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/z_pytest_gpu4.log 2>&1; echo pytest_rc=$? >> gpurun_out/z_pytest_gpu4.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo rc=$? >> gpurun_out/z_smoke.log
timeout 180 python bench.py > gpurun_out/z_bench_n1.log 2>&1
timeout 180 python bench.py --impl reference > gpurun_out/z_bench_ref_n1.log 2>&1
timeout 180 $R2 --master-port 29641 bench.py --gpus 2 > gpurun_out/z_bench_n2.log 2>&1
timeout 180 $R4 --master-port 29642 bench.py --gpus 4 > gpurun_out/z_bench_n4.log 2>&1
timeout 500 $R2 --master-port 29643 benchmarks/p2p_sweep.py --impl iccl-auto --max-pow 30 > gpurun_out/z_sweep_iccl-auto.log 2>&1
timeout 300 $R4 --master-port 29644 benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/z_moe_iccl_n4.log 2>&1
timeout 300 $R4 --master-port 29645 benchmarks/failover.py --chunk-mib 32 > gpurun_out/z_failover_n4.log 2>&1
timeout 300 $R4 --master-port 29646 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/z_bench_a2a_n4.log 2>&1
