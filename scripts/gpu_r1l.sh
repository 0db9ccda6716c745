timeout 120 ./probes/p2p_probe7 > gpurun_out/probe7.txt 2>&1
