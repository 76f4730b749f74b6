#!/bin/bash
# BASELINE config 2: fused (interleaved) vs unfused (standard) loop at 512^2 x 128 fp64.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in interleaved standard; do
  timeout 300 python bench.py --config c2 --variant $v --steps 100 --warmup 5 --no-cpu > gpurun_out/c2_$v.json 2> gpurun_out/c2_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.load(open(f"gpurun_out/c2_{v}.json"))
print(f"{v:12s} it/s={d['value']:8.1f} ms/it={d['ms_per_step']:.4f} bytes/it={d['algorithmic_bytes_iteration']/1e9:.3f} GB "
      f"achieved={d['achieved_gbs_iteration']:.0f} GB/s e2e={d['e2e']['value']:.1f} it/s launches/it={d['gpu_launches']/d['steps']:.1f}")
PY
done
