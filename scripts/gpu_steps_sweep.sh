#!/bin/bash
# it/s and SM clocks vs. timed-region length (power-cap behaviour).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for n in ${STEPS:-20 100 300 1000}; do
  env $ENVS timeout 600 python bench.py --steps $n --warmup 5 --no-cpu --no-e2e "$@" > gpurun_out/st_$n.json 2> gpurun_out/st_$n.err
  python - "$n" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/st_{n}.json")); r = d["roofline"]; c = d["clocks"]
print(f"steps={n:5s} it/s={d['value']:7.1f} K1={r['fused_prec_ms']:.3f} K2={r['fused_spmv_ms']:.3f} sm_mhz={c['sm_mhz']} reasons={c['reasons']} samples={c.get('samples')}")
PY
done
