#!/bin/bash
# Consumed-reduction mode (ACG_CONSUME=1, default) vs a reduction kernel after
# each sweep (ACG_CONSUME=0): parity tests, sanitizers, then per-config A/B.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_runtime_contract.py tests/test_convergence.py \
    tests/test_dropin.py tests/test_acceptance.py tests/test_variants.py -m gpu -q -x 2>&1 | tail -4
timeout 900 python -m pytest tests/test_sanitizers.py -m gpu -q -x -k "single_process and (memcheck or racecheck or initcheck)" 2>&1 | tail -2
for c in ${CONFIGS:-c1 c1 c3}; do
  for g in 0 1; do
    ACG_CONSUME=$g timeout 300 python bench.py --config $c --steps ${STEPS:-1000} --warmup 20 --no-cpu --no-e2e \
        --no-ktime --sustain-steps 0 > gpurun_out/cs_${c}_$g.json 2> gpurun_out/cs_${c}_$g.err
    python -c "import json;d=json.load(open('gpurun_out/cs_${c}_$g.json'));print('$c consume=$g', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us/it launches', d['gpu_launches'], 'frac', d['roofline']['frac'])" || tail -3 gpurun_out/cs_${c}_$g.err
  done
done
