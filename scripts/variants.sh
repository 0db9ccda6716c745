#!/bin/bash
# p2p_sweep variants on 2 GPUs: one per line of $1 ("ENV=1 ENV2=0 | sweep args"),
# each printed under a "## line" header.  Used for A/B experiments:
#   bash scripts/variants.sh scripts/variants/k7.txt >> log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
P=29690
while IFS= read -r L; do
  [ -z "$L" ] && continue
  case "$L" in \#*) continue ;; esac
  E=${L%%|*}; A=${L#*|}
  echo "## $L"
  P=$((P + 1))
  env $E timeout 600 $TR --master-port $P benchmarks/p2p_sweep.py --impl iccl-auto $A 2>&1 | grep -v "OMP_NUM\|^\*\*\*\|^$"
done < "$1"
