#!/bin/bash
# All BASELINE configs on one GPU (device it/s, short runs) + GPU parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-100} --warmup 20 --no-cpu --sustain-steps 0 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/cfg_{c}.json")); r = d["roofline"]
    print(f"{c} it/s={d['value']:9.1f} ms/it={d['ms_per_step']:.4f} iter={d['achieved_gbs_iteration']:.0f} GB/s "
          f"({d['frac_of_peak_iteration']*100:.1f}%) K1={r['fused_prec_ms']:.3f} K2={r['fused_spmv_ms']:.3f} e2e={d['e2e']['value']:.1f} launches/it={d['gpu_launches']/d['steps']:.1f}")
except Exception as e:
    print(c, "FAILED", e, open(f"gpurun_out/cfg_{c}.err").read()[-800:])
PY
done
[ -n "$SKIP_TESTS" ] || timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
