#!/bin/bash
# Thomas (K1) configuration sweep at C3: W,CP,D x occupancy x math.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e ${BARGS} > gpurun_out/th_$tag.json 2> gpurun_out/th_$tag.err
  python - "$tag" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/th_{t}.json")); r=d["roofline"]
    print(f"{t:26s} it/s={d['value']:7.1f} K1={r['fused_prec_ms']:.3f}ms ({r['fused_prec_gbs']:5.0f} GB/s) K2={r['fused_spmv_ms']:.3f}ms ({r['fused_spmv_gbs']:5.0f})")
except Exception as e:
    print(t, "FAILED", e, open(f"gpurun_out/th_{t}.err").read()[-300:])
PY
}
for cfg in "2,2,12" "2,4,12" "2,4,8" "4,4,8" "2,8,8" "4,2,8"; do
  run "ex_$cfg" ACG_THOMAS=$cfg
done
BARGS="--math fast"
for cfg in "2,2,12" "2,4,8" "2,8,8"; do
  run "fast_$cfg" ACG_THOMAS=$cfg
done
BARGS=""
run "ex_2,4,8_occ6" ACG_THOMAS=2,4,8 ACG_THOMAS_OCC=6
run "ex_2,4,8_occ5" ACG_THOMAS=2,4,8 ACG_THOMAS_OCC=5
run "ex_2,8,8_occ8" ACG_THOMAS=2,8,8 ACG_THOMAS_OCC=8
