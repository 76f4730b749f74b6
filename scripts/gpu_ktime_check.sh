#!/bin/bash
# Overhead of per-launch K1/K2 events: headline pass with them (--ktime-inline)
# vs without (default; the kernel roofline then comes from a second pass).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
for a in "--ktime-inline" ""; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e $a 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('${a:-default}', round(d['value'],1), round(d['ms_per_step'],4))"
done; done
