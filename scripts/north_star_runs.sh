#!/usr/bin/env bash
# The north-star shapes at the depths one box can hold:
#   A: Llama-7B layer shapes, 256K context, n=16 slices, m=4, PP = 1 / 2 / 4
#   B: Llama-13B layer shapes (c3), 256K, n=16, m=4, PP=4, exchange off / on / early
# Every run writes its bench JSON line, the calibrated simulate() prediction
# and the measured Gantt under gpurun_out/.
#   gpurun --gpus 4 --timeout 5400 -- bash scripts/north_star_runs.sh [A|B|AB]
set -u
mkdir -p gpurun_out
which=${1:-AB}
tr() {  # nproc, tag, args...
  local n=$1 tag=$2; shift 2
  if [ "$n" = 1 ]; then
    timeout 1500 python bench.py --gpus 1 "$@" --calibrate gpurun_out/r02_ns_${tag}.calib.json \
      > gpurun_out/r02_ns_${tag}.json 2> gpurun_out/r02_ns_${tag}.err
  else
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@" \
      --calibrate gpurun_out/r02_ns_${tag}.calib.json --gantt gpurun_out/r02_ns_${tag}.gantt.json \
      > gpurun_out/r02_ns_${tag}.json 2> gpurun_out/r02_ns_${tag}.err
  fi
  echo "$tag rc=$? $(tail -c 300 gpurun_out/r02_ns_${tag}.json)"
}
S="--seq-len 262144 --slices 16 --microbatches 4 --steps 2 --warmup 3"
if [[ $which == *A* ]]; then
  tr 4 c2_256k_pp4 --model c2 --layers 8 $S --no-cpu-baseline
  tr 2 c2_256k_pp2 --model c2 --layers 8 $S --no-cpu-baseline
  tr 1 c2_256k_pp1 --model c2 --layers 8 $S --no-cpu-baseline --no-e2e
fi
if [[ $which == *B* ]]; then
  for x in off on early; do
    tr 4 c3_256k_pp4_$x --model c3 --layers 8 $S --exchange $x --no-cpu-baseline --no-e2e
  done
fi
