#!/usr/bin/env bash
# Multi-GPU measurement batch (4 GPUs):
#   M: c2 (Llama-7B shapes x8 layers) 128K, n=8, m=4 at PP=4 and PP=2: base,
#      vocabulary parallelism, interleaved v=2
#   A: the north-star shape at one box's depth: c2 x8, 256K, n=16, m=4, PP=4 / 2
#   B: c3 (Llama-13B shapes x8), 256K, n=16, m=4, PP=4, exchange off / on / early
# Every run writes its bench JSON line, the calibrated simulate() prediction
# and the measured Gantt under gpurun_out/.
#   gpurun --gpus 4 --timeout 6000 -- bash scripts/north_star_runs.sh [M][A][B]
set -u
mkdir -p gpurun_out
which=${1:-MAB}
tr() {  # nproc, tag, args...
  local n=$1 tag=$2; shift 2
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 2 --warmup 3 "$@" \
    --calibrate gpurun_out/r02_ms_${tag}.calib.json --gantt gpurun_out/r02_ms_${tag}.gantt.json \
    > gpurun_out/r02_ms_${tag}.json 2> gpurun_out/r02_ms_${tag}.err
  echo "$tag rc=$? $(tail -c 400 gpurun_out/r02_ms_${tag}.json)"
}
if [[ $which == *M* ]]; then
  tr 4 c2_128k_pp4 --model c2 --no-e2e
  tr 4 c2_128k_pp4_vp --model c2 --vocab-parallel --no-e2e
  tr 4 c2_128k_pp4_v2 --model c2 --interleave 2 --no-e2e
  tr 2 c2_128k_pp2 --model c2 --no-e2e
  tr 2 c2_128k_pp2_vp --model c2 --vocab-parallel --no-e2e
fi
S="--seq-len 262144 --slices 16 --microbatches 4"
if [[ $which == *A* ]]; then
  tr 4 c2_256k_pp4 --model c2 --layers 8 $S
  tr 2 c2_256k_pp2 --model c2 --layers 8 $S --no-e2e
fi
if [[ $which == *B* ]]; then
  for x in off on early; do
    tr 4 c3_256k_pp4_$x --model c3 --layers 8 $S --exchange $x --no-e2e
  done
fi
