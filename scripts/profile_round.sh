#!/usr/bin/env bash
# One-GPU measurement batch for profiles/: the default bench line (with the
# cost calibration), the ncu launch list of the same command (kernel time
# shares), full ncu captures of the layer GEMMs (cuBLASLt nvjet) and of K1/K2.
#   gpurun --timeout 3000 -- bash scripts/profile_round.sh
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 --calibrate gpurun_out/r02_n1.calib.json \
  > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv \
  --log-file gpurun_out/r02_launches_n1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02_ncu_launches.log 2>&1
echo "launch list rc=$?"
python scripts/launch_shares.py gpurun_out/r02_launches_n1.csv "ncu launch list, bench.py --steps 1 --warmup 3 (N=1 default c2 x8, 128K, n8, m4)" \
  > gpurun_out/r02_launch_shares.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nvjet -s 60 -c 8 \
  -o gpurun_out/r02_gemm_full -f python bench.py --steps 1 --warmup 1 --layers 2 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02_ncu_gemm.log 2>&1
echo "gemm full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:attn_(fwd_ps|bwd_d128)" -c 2 \
  -o gpurun_out/r02_attn_full -f python scripts/prof_attn.py > gpurun_out/r02_ncu_attn.log 2>&1
echo "attn full rc=$?"
# K2 variants (SP_BWD_VARIANT 0/1/2, scripts/k2_ab.py)
timeout 600 python scripts/k2_ab.py > gpurun_out/r02_k2ab2.log 2>&1
echo "k2 a/b rc=$?"
# (compute-sanitizer is closed on this GPU pool: runs under it left GPUs needing a reset)
