#!/bin/bash
# One parameterised GPU-box runner (replaces round 1's one-off scripts).
#   gpurun -- 'bash scripts/gpu.sh TAG STEP [STEP ...]'
# Every step logs to gpurun_out/TAG_STEP.log and appends its rc; a failing
# step does not stop the next.  Steps:
#   pytest      pytest -m gpu (all tests; ranks share the visible GPUs)
#   pytest:EXPR pytest -m gpu -k EXPR
#   smoke       __graft_entry__.smoke()
#   bench1      bench.py N=1 (+ the reference arm)
#   bench2      bench.py N=2 over torchrun (needs 2 GPUs)
#   sweep       benchmarks/p2p_sweep.py (2 ranks)
#   sweeps      p2p_sweep: iccl-auto, nccl, nccl-zero (zero-CTA), nccl-ce; unidirectional and --bidir
#   gemm        gemm_interference on all GPUs: none, iccl-ce 256 MiB, iccl-auto / nccl at 4 and 16 MiB
#   gemmk7      gemm_interference iccl-ce 256 MiB with memop waits vs K7 waits (parked streams)
#   failover    benchmarks/failover.py on all GPUs (sm backup; relay when >= 3 GPUs)
#   moe         benchmarks/moe_alltoallv.py on all GPUs, iccl and nccl
#   armedexp    p2p_sweep 1-256 MiB: plain / armed (a never-firing fault script) / armed without the
#               backup attempt (attribution), default and 8 MiB chunks, monitor on
#   ncuk        ncu --set full of K2 (expand) and K8 (fused dispatch, 1 rank) + the kernels bench
#   var:NAME    the p2p_sweep variants listed in scripts/variants/NAME.txt (2 GPUs)
#   dispatch    benchmarks/moe_dispatch.py on all GPUs: fused K8 vs K2 + alltoallv vs NCCL
#   launches    ncu launch list of smoke() (gpu__time_duration, no replay of waits)
#   ncuprobe    probes/ncu_xproc under ncu (cross-process serialisation)
#   cmd:...     any command (quoted)
set -u
TAG=$1; shift
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for STEP in "$@"; do
  LOG=gpurun_out/${TAG}_${STEP//[^A-Za-z0-9_.-]/_}.log
  LOG=${LOG:0:120}
  echo "== $STEP (gpus=$NG)" > "$LOG"
  case "$STEP" in
    pytest) timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 300 >> "$LOG" 2>&1 ;;
    pytest:*) timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 300 -k "${STEP#pytest:}" >> "$LOG" 2>&1 ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> "$LOG" 2>&1 ;;
    bench1) timeout 300 python bench.py >> "$LOG" 2>&1; timeout 300 python bench.py --impl reference >> "$LOG" 2>&1 ;;
    bench2) timeout 300 $TR --nproc-per-node 2 --master-port 29671 bench.py --gpus 2 >> "$LOG" 2>&1 ;;
    sweep) timeout 900 $TR --nproc-per-node 2 --master-port 29672 benchmarks/p2p_sweep.py --impl iccl-auto --min-pow 3 --max-pow 28 >> "$LOG" 2>&1 ;;
    sweeps) for I in iccl-auto nccl nccl-zero nccl-ce; do
              for B in "" --bidir; do
                echo "## $I $B" >> "$LOG"
                timeout 900 $TR --nproc-per-node 2 --master-port 29673 benchmarks/p2p_sweep.py --impl $I $B --min-pow 3 --max-pow 30 >> "$LOG" 2>&1
              done; done ;;
    gemm) echo "## none" >> "$LOG"; timeout 600 $TR --nproc-per-node $NG --master-port 29674 benchmarks/gemm_interference.py --impl none >> "$LOG" 2>&1
          echo "## iccl-ce 256" >> "$LOG"; timeout 600 $TR --nproc-per-node $NG --master-port 29675 benchmarks/gemm_interference.py --impl iccl-ce >> "$LOG" 2>&1
          for M in 4 16; do for I in iccl-auto nccl; do
            echo "## $I $M" >> "$LOG"
            timeout 600 $TR --nproc-per-node $NG --master-port 29676 benchmarks/gemm_interference.py --impl $I --msg-mib $M >> "$LOG" 2>&1
          done; done ;;
    failover) timeout 600 $TR --nproc-per-node $NG --master-port 29677 benchmarks/failover.py >> "$LOG" 2>&1
              [ "$NG" -ge 3 ] && timeout 600 $TR --nproc-per-node $NG --master-port 29678 benchmarks/failover.py --backup relay >> "$LOG" 2>&1 || true ;;
    armedexp) for V in "" "--armed" "--armed ICCL_ARMED_BACKUP=0" "--chunk-bytes 8388608" "--chunk-bytes 8388608 --armed" \
                    "--chunk-bytes 8388608 --armed ICCL_ARMED_BACKUP=0" "--chunk-bytes 8388608 --records" "--chunk-bytes 33554432" "--chunk-bytes 33554432 --armed" "--chunk-bytes 33554432 --records"; do
                A=$(echo "$V" | sed 's/ICCL_ARMED_BACKUP=0//'); E=$(echo "$V" | grep -o 'ICCL_ARMED_BACKUP=0')
                echo "## $V" >> "$LOG"
                env $E timeout 600 $TR --nproc-per-node 2 --master-port 29681 benchmarks/p2p_sweep.py --impl iccl-auto \
                  --min-pow 20 --max-pow 28 --step 2 $A >> "$LOG" 2>&1
              done ;;
    ncuk) timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:iccl_(expand|dispatch)' -c 4 \
            -f -o gpurun_out/${TAG}_k2k8 python benchmarks/kernels.py --only k2,k8 --reps 1 >> "$LOG" 2>&1
          timeout 300 python benchmarks/kernels.py --only k1_local,k1_peer,k2,k3,k8 >> "$LOG" 2>&1 ;;
    var:*) timeout 3000 bash scripts/variants.sh "scripts/variants/${STEP#var:}.txt" >> "$LOG" 2>&1 ;;
    dispatch) timeout 600 $TR --nproc-per-node $NG --master-port 29680 benchmarks/moe_dispatch.py >> "$LOG" 2>&1 ;;
    gemmk7) for V in "X=0" "ICCL_K7_CE=1" "ICCL_K7_CE=1 ICCL_K7_READY=1" "X=0"; do echo "## $V" >> "$LOG"
              env $V timeout 600 $TR --nproc-per-node $NG --master-port 29720 benchmarks/gemm_interference.py --impl iccl-ce >> "$LOG" 2>&1
            done ;;
    gemm1) for I in iccl-auto nccl; do for M in 0.25 1; do echo "## $I $M" >> "$LOG"
             timeout 600 $TR --nproc-per-node $NG --master-port 29750 benchmarks/gemm_interference.py --impl $I --msg-mib $M >> "$LOG" 2>&1
           done; done ;;
    failcaps) for C in 16 32 64; do echo "## sm_cap $C" >> "$LOG"
                ICCL_SM_CAP=$C timeout 600 $TR --nproc-per-node $NG --master-port 2969$((C % 7)) benchmarks/failover.py >> "$LOG" 2>&1
                ICCL_SM_CAP=$C timeout 600 $TR --nproc-per-node $NG --master-port 2969$((C % 7 + 1)) benchmarks/failover.py --chunk-mib 32 >> "$LOG" 2>&1
              done ;;
    a2apieces) for P in 1 2 4 1; do echo "## ICCL_A2A_PIECES=$P" >> "$LOG"
                ICCL_A2A_PIECES=$P timeout 600 $TR --nproc-per-node $NG --master-port 29740 benchmarks/moe_alltoallv.py --impl iccl >> "$LOG" 2>&1
              done ;;
    a2aorder) for O in 0 1 0 1; do echo "## ICCL_A2A_ORDER=$O" >> "$LOG"
                ICCL_A2A_ORDER=$O timeout 600 $TR --nproc-per-node $NG --master-port 29741 benchmarks/moe_alltoallv.py --impl iccl >> "$LOG" 2>&1
              done ;;
    moe) for I in iccl nccl; do timeout 600 $TR --nproc-per-node $NG --master-port 29679 benchmarks/moe_alltoallv.py --impl $I >> "$LOG" 2>&1; done ;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 2000 --csv \
                --log-file gpurun_out/${TAG}_launches.csv python -c "import __graft_entry__ as g; g.smoke()" >> "$LOG" 2>&1 ;;
    ncuprobe) ./probes/ncu_xproc >> "$LOG" 2>&1; timeout 120 ncu --target-processes all --metrics gpu__time_duration.sum \
                ./probes/ncu_xproc >> "$LOG" 2>&1 ;;
    cmd:*) timeout 1800 bash -c "${STEP#cmd:}" >> "$LOG" 2>&1 ;;
    *) echo "unknown step $STEP" >> "$LOG" ;;
  esac
  echo "rc=$?" >> "$LOG"
  tail -3 "$LOG"
done
