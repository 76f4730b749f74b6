#!/bin/bash
# Usage: gpu_env_steps.sh "TAG:ENV=..;TAG2:.." STEPS [bench args]  (long runs: power-capped steady state)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IFS=';' read -ra CFGS <<< "$1"; shift; N=$1; shift
for c in "${CFGS[@]}"; do
  tag=${c%%:*}; envs=${c#*:}
  env $envs timeout 600 python bench.py --steps $N --warmup 5 --no-cpu --no-e2e "$@" > gpurun_out/es_$tag.json 2> gpurun_out/es_$tag.err
  python - "$tag" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/es_{t}.json")); r=d["roofline"]; c=d["clocks"]
    print(f"{t:16s} it/s={d['value']:7.1f} K1={r['fused_prec_ms']:.3f} K2={r['fused_spmv_ms']:.3f} step={d['ms_per_step']:.3f} mhz={c['sm_mhz']}")
except Exception as e:
    print(t, "FAILED", e, open(f"gpurun_out/es_{t}.err").read()[-600:])
PY
done
