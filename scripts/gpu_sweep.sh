#!/bin/bash
# Parity + configuration sweep of the fused sweeps at C3 (no CPU baseline).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=5 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
run() { # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/sw_$tag.json 2> gpurun_out/sw_$tag.err
  python - "$tag" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/sw_{t}.json"))
    r=d["roofline"]
    print(f"{t:22s} it/s={d['value']:8.1f} iter_GB/s={d['achieved_gbs_iteration']:7.0f} K1={r['fused_prec_ms']:.3f}ms ({r['fused_prec_gbs']:.0f} GB/s) K2={r['fused_spmv_ms']:.3f}ms ({r['fused_spmv_gbs']:.0f} GB/s)")
except Exception as e:
    print(t, "FAILED", e, open(f"gpurun_out/sw_{t}.err").read()[-500:])
PY
}
run default
run spmv_plain ACG_SPMV=plain
run occ2 ACG_THOMAS_OCC=2
run occ3 ACG_THOMAS_OCC=3

timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --math fast > gpurun_out/sw_fast.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/sw_fast.json')); r=d['roofline']; print('fast', d['value'], r['fused_prec_ms'], r['fused_spmv_ms'])"
