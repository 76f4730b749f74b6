#!/bin/bash
# Current tree vs the round-1 tree (_r1/, git archive e2ede89, built in place), alternated at C3.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for i in 1 2 3; do
  for v in new r1; do
    d=.; [ $v = r1 ] && d=_r1
    (cd $d && timeout 300 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$v', round(d['value'],1), 'it/s K1', round(r['fused_prec_ms']*1e3,1), 'us K2', round(r['fused_spmv_ms']*1e3,1), 'us', d['clocks']['sm_mhz'], 'MHz')"
  done
done
