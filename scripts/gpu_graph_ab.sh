#!/bin/bash
# A/B: CUDA-graph chunks of 16 iterations (ACG_GRAPH=1) vs stream launches, per config.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ACG_GRAPH=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_runtime_contract.py \
    tests/test_csr_backend.py -m gpu -q -x 2>&1 | tail -2
for c in c1 c2 c3; do
  for g in 0 1; do
    ACG_GRAPH=$g timeout 300 python bench.py --config $c --steps ${STEPS:-500} --warmup 20 --no-cpu --no-e2e \
        --no-ktime --sustain-steps 0 > gpurun_out/g_${c}_$g.json 2> gpurun_out/g_${c}_$g.err
    python -c "import json;d=json.load(open('gpurun_out/g_${c}_$g.json'));print('$c graph=$g', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us/it host', round(d['host_enqueue_ms']*1e3/d['steps'],2), 'us/it launches', d['gpu_launches'])" || tail -3 gpurun_out/g_${c}_$g.err
  done
done
