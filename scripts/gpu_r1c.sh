# round-1 re-entry GPU batch (2 GPUs): parity tests, smoke, bench N=1/N=2, reference arm, ncu launch list
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 180 python bench.py > gpurun_out/bench_n1.log 2>&1
timeout 180 python bench.py --impl reference > gpurun_out/bench_ref_n1.log 2>&1
timeout 180 $R --master-port 29631 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1
timeout 180 $R --master-port 29632 bench.py --gpus 2 --iccl-monitor 0 > gpurun_out/bench_n2_mon0.log 2>&1
timeout 300 $R --master-port 29633 bench.py --gpus 2 --workload alltoallv --steps 5 > gpurun_out/bench_a2a_n2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_n1.log 2>&1
