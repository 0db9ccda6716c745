# round-1 final tree (all experiment knobs at their defaults), 2-GPU box
export PYTHONUNBUFFERED=1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/zw_pytest_gpu2.log 2>&1; echo pytest_rc=$? >> gpurun_out/zw_pytest_gpu2.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zw_smoke.log 2>&1; echo rc=$? >> gpurun_out/zw_smoke.log
timeout 180 python bench.py > gpurun_out/zw_bench_n1.log 2>&1
timeout 180 python bench.py --impl reference > gpurun_out/zw_bench_ref_n1.log 2>&1
timeout 180 $R2 --master-port 29662 bench.py --gpus 2 > gpurun_out/zw_bench_n2.log 2>&1
timeout 200 $R2 --master-port 29663 benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 3 --max-pow 28 > gpurun_out/zw_sweep.log 2>&1
