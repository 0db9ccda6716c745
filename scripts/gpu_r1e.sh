# round-1 GPU batch E (2 GPUs): parity tests after LL credit fix / relay / monitor events, flag-placement probe, benches
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 120 ./probes/p2p_probe5 > gpurun_out/probe5.txt 2>&1
timeout 180 python bench.py > gpurun_out/bench_n1.log 2>&1
timeout 180 python bench.py --iccl-monitor 0 --no-cpu-baseline > gpurun_out/bench_n1_mon0.log 2>&1
timeout 180 python bench.py --impl reference > gpurun_out/bench_ref_n1.log 2>&1
timeout 180 $R --master-port 29631 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1
timeout 180 $R --master-port 29632 bench.py --gpus 2 --iccl-monitor 0 > gpurun_out/bench_n2_mon0.log 2>&1
timeout 300 $R --master-port 29633 benchmarks/failover.py > gpurun_out/failover_n2.log 2>&1
timeout 400 $R --master-port 29634 benchmarks/p2p_sweep.py --impl iccl-auto --ll-bytes 32768 --max-pow 24 > gpurun_out/sweep_iccl-ll.log 2>&1
