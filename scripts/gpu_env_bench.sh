#!/bin/bash
# Usage: gpu_env_bench.sh "TAG:ENV=.. ENV2=..;TAG2:..." [bench args]; prints one line per config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IFS=';' read -ra CFGS <<< "$1"; shift
for c in "${CFGS[@]}"; do
  tag=${c%%:*}; envs=${c#*:}
  env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/e_$tag.json 2> gpurun_out/e_$tag.err
  python - "$tag" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/e_{t}.json")); r=d["roofline"]
    print(f"{t:22s} it/s={d['value']:7.1f} K1={r['fused_prec_ms']:.3f}ms ({r['fused_prec_gbs']:5.0f} GB/s) K2={r['fused_spmv_ms']:.3f}ms ({r['fused_spmv_gbs']:5.0f}) step={d['ms_per_step']:.3f}")
except Exception as e:
    print(t, "FAILED", e, open(f"gpurun_out/e_{t}.err").read()[-600:])
PY
done
