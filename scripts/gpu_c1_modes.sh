#!/bin/bash
# C1 (and C2) launch-mode study: default vs the sweep's last CTA finishing the reduction.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in c1 c2; do
for v in "base:" "ctafin:ACG_CTA_FINISH=1" "base2:" "ctafin2:ACG_CTA_FINISH=1"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 300 python bench.py --config $c --steps 2000 --warmup 32 --no-cpu --no-e2e --no-ktime \
      --sustain-steps 0 > gpurun_out/m_$c_$tag.json 2> gpurun_out/m_$c_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/m_$c_$tag.json'));print('$c $tag', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us/it', round(d['frac_of_peak_iteration']*100,1), '% launches/it', d['gpu_launches']/d['steps'])" || tail -3 gpurun_out/m_$c_$tag.err
done; done
