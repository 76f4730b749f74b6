#!/bin/bash
# Env-toggle A/B, alternated, it/s only: gpu_env_ab.sh VAR "c1 c2" [values, default "0 1"]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
V=$1; CFGS=${2:-c1}; VALS=${3:-0 1}
for C in $CFGS; do
  case $C in c1) S=1000;; c2) S=300;; *) S=100;; esac
  for i in 1 2; do
  for x in $VALS; do
    env $V=$x timeout 300 python bench.py --config $C --steps $S --warmup 20 --no-cpu --no-e2e --no-ktime --sustain-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$C $V=$x', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us/it', d['clocks']['sm_mhz'], 'MHz')"
  done; done
done
