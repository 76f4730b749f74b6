#!/bin/bash
# A/B of the in-tree library (new) against paper_1302_7193_b200/alt_libacg_cuda.so (old)
# over several configs, alternated, it/s only (no ktime pass). Usage: gpu_ab_cfgs.sh "c1 c2 c3"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
A=$PWD/paper_1302_7193_b200/alt_libacg_cuda.so
for C in ${1:-c1 c2 c3}; do
  case $C in c1) S=1000;; c2) S=300;; *) S=100;; esac
  for i in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export ACG_LIB_OVERRIDE=$A; else unset ACG_LIB_OVERRIDE; fi
    timeout 300 python bench.py --config $C --steps $S --warmup 20 --no-cpu --no-e2e --no-ktime --sustain-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$C $v', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us/it', d['clocks']['sm_mhz'], 'MHz')"
  done; done
done
