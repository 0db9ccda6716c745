export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
ICCL_DEBUG=1 timeout 70 $R --master-port 29661 scripts/debug_sendrecv.py 32768 > gpurun_out/debug_ll32k.log 2>&1
timeout 70 $R --master-port 29662 scripts/debug_sendrecv.py 32768 pinned > gpurun_out/debug_ll32k_pinned.log 2>&1
timeout 120 ./probes/p2p_probe5 > gpurun_out/probe5b.txt 2>&1
