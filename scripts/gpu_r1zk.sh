export PYTHONUNBUFFERED=1
for p in 1 2 4; do
timeout 300 python bench.py --e2e-pieces $p --no-cpu-baseline > gpurun_out/zk_bench_n1_p$p.log 2>&1
done
