#!/bin/bash
# Quick loop: GPU parity tests + C3 bench lines for the given ACG_THOMAS_TM configs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_q.log)"
grep -E "FAIL|Error|assert" gpurun_out/pytest_q.log | head -20
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e ${BARGS} > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err
  python - "$tag" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/q_{t}.json")); r=d["roofline"]
    print(f"{t:26s} it/s={d['value']:7.1f} K1={r['fused_prec_ms']:.3f}ms ({r['fused_prec_gbs']:5.0f} GB/s) K2={r['fused_spmv_ms']:.3f}ms ({r['fused_spmv_gbs']:5.0f})")
except Exception as e:
    print(t, "FAILED", e, open(f"gpurun_out/q_{t}.err").read()[-600:])
PY
}
for cfg in ${TM_CFGS:-"2,7"}; do run "tm_$cfg" ACG_THOMAS_TM=$cfg; done
for cfg in ${TM_FAST:-}; do BARGS="--math fast" run "fast_$cfg" ACG_THOMAS_TM=$cfg; done
for cfg in ${TM_C4:-}; do BARGS="--config c4" run "c4_$cfg" ACG_THOMAS_TM=$cfg; done
