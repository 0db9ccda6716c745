export PYTHONUNBUFFERED=1
python probes/pcie_probe.py > gpurun_out/zi_pcie.log 2>&1
for p in 16 32 64; do
timeout 300 python bench.py --e2e-pieces $p --no-cpu-baseline > gpurun_out/zi_bench_n1_p$p.log 2>&1
done
