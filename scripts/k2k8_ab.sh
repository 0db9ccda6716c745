#!/bin/bash
# A/B of the TMA forms of K2 (expand), K8 (fused dispatch) and K10 (fused
# combine) against the warp-copy forms: kernels bench (1 GPU) and the
# dispatch / combine bench (all GPUs).
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $NG"
for V in "ICCL_K10_TMA=1" "ICCL_K10_TMA=0" "ICCL_K2_TMA=1 ICCL_K8_TMA=1" "ICCL_K2_TMA=0 ICCL_K8_TMA=0"; do
  echo "## $V"
  env $V timeout 300 python benchmarks/kernels.py --only k2,k8
  env $V timeout 600 $TR --master-port 29730 benchmarks/moe_dispatch.py --arms fused,unfused 2>&1 | grep "^{"
done
