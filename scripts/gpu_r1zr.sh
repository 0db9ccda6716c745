# final round-1 check of the committed tree (4-GPU box)
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/zr_pytest_gpu4.log 2>&1; echo pytest_rc=$? >> gpurun_out/zr_pytest_gpu4.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zr_smoke.log 2>&1; echo rc=$? >> gpurun_out/zr_smoke.log
timeout 180 python bench.py > gpurun_out/zr_bench_n1.log 2>&1
timeout 180 python bench.py --impl reference > gpurun_out/zr_bench_ref_n1.log 2>&1
timeout 180 $R4 --master-port 29642 bench.py --gpus 4 > gpurun_out/zr_bench_n4.log 2>&1
timeout 300 $R4 --master-port 29646 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zr_a2a_n4.log 2>&1
timeout 300 $R4 --master-port 29647 benchmarks/failover.py --chunk-mib 32 > gpurun_out/zr_failover_n4.log 2>&1
