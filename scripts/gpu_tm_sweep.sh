#!/bin/bash
# TMEM Thomas (K1) sweep at C3 + GPU parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_tm.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_tm.log)"
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e ${BARGS} > gpurun_out/tm_$tag.json 2> gpurun_out/tm_$tag.err
  python - "$tag" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/tm_{t}.json")); r=d["roofline"]
    print(f"{t:26s} it/s={d['value']:7.1f} K1={r['fused_prec_ms']:.3f}ms ({r['fused_prec_gbs']:5.0f} GB/s) K2={r['fused_spmv_ms']:.3f}ms ({r['fused_spmv_gbs']:5.0f})")
except Exception as e:
    print(t, "FAILED", e, open(f"gpurun_out/tm_{t}.err").read()[-600:])
PY
}
for cfg in 0 "2,7,8" "4,7,8" "2,12,16" "4,12,16" "2,15,16" "4,15,16"; do
  run "tm_$cfg" ACG_THOMAS_TM=$cfg
done
BARGS="--math fast" run "fast_2,7,8" ACG_THOMAS_TM=2,7,8
BARGS="--config c4" run "c4_2,7,8" ACG_THOMAS_TM=2,7,8
BARGS="--config c4" run "c4_0" ACG_THOMAS_TM=0
