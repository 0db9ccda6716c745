export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 120 $R --master-port 29671 scripts/diag_ring.py > gpurun_out/diag_ring_mon1.log 2>&1
DIAG_MON=0 timeout 120 $R --master-port 29672 scripts/diag_ring.py > gpurun_out/diag_ring_mon0.log 2>&1
ICCL_DEBUG=1 DIAG_MON=0 timeout 120 $R --master-port 29673 scripts/diag_ring.py > gpurun_out/diag_ring_dbg.log 2>&1
