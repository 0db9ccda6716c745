export PYTHONUNBUFFERED=1
for p in 4 8 16; do
timeout 300 python bench.py --e2e-pieces $p --no-cpu-baseline > gpurun_out/zj_bench_n1_p$p.log 2>&1
done
timeout 300 python bench.py > gpurun_out/zj_bench_n1.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/zj_bench_ref_n1.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zj_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/zj_pytest_gpu1.log 2>&1
tail -2 gpurun_out/zj_pytest_gpu1.log
