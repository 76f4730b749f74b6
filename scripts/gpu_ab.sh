#!/bin/bash
# A/B of the in-tree library (new) against paper_1302_7193_b200/alt_libacg_cuda.so (old),
# alternated: K1/K2 per-launch times (ktime pass) and it/s. Usage: gpu_ab.sh [config] [steps]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
A=$PWD/paper_1302_7193_b200/alt_libacg_cuda.so
C=${1:-c3}; S=${2:-50}
for i in 1 2 3; do
for v in new old; do
  if [ $v = old ]; then export ACG_LIB_OVERRIDE=$A; else unset ACG_LIB_OVERRIDE; fi
  timeout 300 python bench.py --config $C --steps $S --warmup 5 --no-cpu --no-e2e --sustain-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$v', round(d['value'],1), 'it/s K1', round(r['fused_prec_ms']*1e3,1), 'us K2', round(r['fused_spmv_ms']*1e3,1), 'us', d['clocks']['sm_mhz'], 'MHz')"
done; done
