# N=4 ring slowness + relay failover hang diagnosis (4 GPUs)
export PYTHONUNBUFFERED=1
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 180 $R4 --master-port 29642 bench.py --gpus 4 --iccl-monitor 0 > gpurun_out/u_bench_n4_mon0.log 2>&1
ICCL_DEBUG=1 timeout 180 $R4 --master-port 29643 bench.py --gpus 4 --steps 4 --warmup 3 > gpurun_out/u_bench_n4_dbg.log 2>&1
ICCL_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k relay_failover > gpurun_out/u_relay.log 2>&1
mkdir -p gpurun_out/u_relay_logs; find /tmp/pytest-of-root -name "rank*.log" | while read f; do cp "$f" gpurun_out/u_relay_logs/$(basename $f); done
timeout 300 $R4 --master-port 29645 benchmarks/moe_alltoallv.py --impl iccl --dump-records > gpurun_out/u_moe_records_n4.log 2>&1
