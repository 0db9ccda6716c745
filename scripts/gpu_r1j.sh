export PYTHONUNBUFFERED=1
timeout 120 ./probes/p2p_probe6 > gpurun_out/probe6.txt 2>&1
