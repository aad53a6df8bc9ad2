#!/usr/bin/env bash
# Activation offload: parity, and what it buys (one GPU).
set -u
mkdir -p gpurun_out
PYTHONUNBUFFERED=1 timeout 900 python -m pytest tests/test_step_gpu.py -q -s -k offload > gpurun_out/r02_offload_parity.log 2>&1
echo "parity rc=$?"
timeout 900 python bench.py --offload --no-cpu-baseline > gpurun_out/r02_bench_n1_offload.json 2> gpurun_out/r02_bench_n1_offload.err
echo "c2 offload rc=$?"
for o in "--offload" ""; do
  tag=$([ -n "$o" ] && echo offload || echo base)
  timeout 1500 python bench.py --model c4 --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $o \
    > gpurun_out/r02_bench_c4_1M_$tag.json 2> gpurun_out/r02_bench_c4_1M_$tag.err
  echo "c4 1M $tag rc=$?"
done
