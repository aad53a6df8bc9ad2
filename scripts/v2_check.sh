#!/usr/bin/env bash
# Interleaved (v=2) step parity on 2 GPUs, unbuffered logs per case.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1 SP_STEP_TIMEOUT=150
for c in "2 4 selective" "1 4 full" "2 8 selective"; do
  set -- $c
  SP_M=$1 SP_N=$2 SP_RC=$3 SP_V=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) tests/mp_step_check.py \
    > gpurun_out/r02_v2_m$1_n$2_$3.log 2>&1
  echo "m=$1 n=$2 $3 rc=$?"
done
