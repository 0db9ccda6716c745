export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for i in 1 2 3; do
timeout 300 $R4 --master-port 2971$i bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zh_a2a_$i.log 2>&1
timeout 300 $R4 --master-port 2973$i benchmarks/moe_alltoallv.py --impl iccl > gpurun_out/zh_moe_$i.log 2>&1
done
timeout 300 $R4 --master-port 29741 bench.py --gpus 4 > gpurun_out/zh_bench_n4.log 2>&1
ICCL_DEBUG=1 timeout 300 $R4 --master-port 29751 bench.py --gpus 4 --workload alltoallv --steps 10 > gpurun_out/zh_a2a_dbg.log 2>&1
grep -c 'slow device call' gpurun_out/zh_a2a_dbg.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/zh_pytest_gpu4.log 2>&1
tail -2 gpurun_out/zh_pytest_gpu4.log
