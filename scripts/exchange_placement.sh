#!/usr/bin/env bash
# Exchange placement A/B on one 4-GPU box (same box, back to back):
#   C: c2 (Llama-7B shapes x8) 128K, n=8, m=4, PP=4: off, early (every plan
#      transfer), early without transfers into the last stage, early with
#      >= 2-chunk transfers only, both filters
#   D: c3 (Llama-13B shapes x8) 256K, n=16, m=4, PP=4: off and the filtered
#      early exchange
# Each run writes its bench line and the measured Gantt under gpurun_out/.
#   E: c2 PP=4 posting A/B (the switches as measured; just-in-time stage
#      receives have since become the default): stage receives posted
#      early (SP_JIT_RECV=0) or just in time (=1), exchange serves posted at
#      the receiving pass (SP_XSERVE_JIT=1, default), NCCL CTAs capped
#      (SP_NCCL_MAX_CTAS=4); then c3 off / filtered early when the best c2
#      exchange variant beats c2 off
#   gpurun --gpus 4 --timeout 3000 -- bash scripts/exchange_placement.sh [C][D][E]
set -u
mkdir -p gpurun_out
which=${1:-CD}
ENVX=${ENVX:-SP_JIT_RECV=0}
tr() {  # tag, args...   (env: per-run NCCL / posting switches)
  local tag=$1; shift
  timeout 900 env $ENVX python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 2 --warmup 3 --no-e2e "$@" \
    --gantt gpurun_out/r02_xp_${tag}.gantt.json > gpurun_out/r02_xp_${tag}.json 2> gpurun_out/r02_xp_${tag}.err
  echo "$tag rc=$? $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['value']), d['bubble_fraction'], d.get('exchange_passes_sending'))" gpurun_out/r02_xp_${tag}.json 2>&1 | tail -1)"
}
if [[ $which == *C* ]]; then
  tr c2_off --model c2
  tr c2_early --model c2 --exchange early
  tr c2_early_nolast --model c2 --exchange early --exchange-skip-last
  tr c2_early_min2 --model c2 --exchange early --exchange-min-chunks 2
  tr c2_early_min2_nolast --model c2 --exchange early --exchange-min-chunks 2 --exchange-skip-last
fi
S="--seq-len 262144 --slices 16 --microbatches 4"
if [[ $which == *D* ]]; then
  tr c3_off --model c3 --layers 8 $S
  tr c3_early_min3_nolast --model c3 --layers 8 $S --exchange early --exchange-min-chunks 3 --exchange-skip-last
fi
if [[ $which == *E* ]]; then
  ENVX=SP_JIT_RECV=0 tr e_c2_off --model c2
  ENVX="SP_JIT_RECV=1" tr e_c2_off_jitrecv --model c2
  ENVX="SP_JIT_RECV=0 SP_XSERVE_JIT=1" tr e_c2_early_min2_nolast --model c2 --exchange early --exchange-min-chunks 2 --exchange-skip-last
  ENVX="SP_XSERVE_JIT=1 SP_JIT_RECV=1 SP_NCCL_MAX_CTAS=4" tr e_c2_early_min2_nolast_all --model c2 --exchange early \
    --exchange-min-chunks 2 --exchange-skip-last
  best=$(python - <<'PY'
import json, glob
v = {}
for f in glob.glob("gpurun_out/r02_xp_e_c2_*.json"):
    try:
        v[f.split("r02_xp_e_c2_")[1][:-5]] = json.loads(open(f).read().strip().splitlines()[-1])["value"]
    except Exception:
        pass
off = max(v.get("off", 0), v.get("off_jitrecv", 0), v.get("off_cta4", 0))
xs = {k: x for k, x in v.items() if k.startswith("early")}
print(max(xs, key=xs.get) if xs and max(xs.values()) > off else "none")
PY
)
  echo "best exchange variant over off: $best"
  if [[ $best != none ]]; then
    S="--seq-len 262144 --slices 16 --microbatches 4"
    ENVX=SP_JIT_RECV=0 tr e_c3_off --model c3 --layers 8 $S
    ENVX=SP_JIT_RECV=0 tr e_c3_early_min3_nolast --model c3 --layers 8 $S --exchange early --exchange-min-chunks 3 \
      --exchange-skip-last
  fi
fi
