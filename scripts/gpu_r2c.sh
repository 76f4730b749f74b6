#!/bin/bash
# Round-2 check 3: whole GPU suite, C1/C2/C3 bench lines (graph chunks on small grids,
# fused K2 reduction for m < 512).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "gpu suite rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/pytest_gpu.log | tail -15
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-500} --warmup 20 --no-cpu --no-e2e \
      --sustain-steps 0 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b_$c.json'));r=d['roofline'];print('$c', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us/it', round(d['frac_of_peak_iteration']*100,1), '% iter; K1', round(r['fused_prec_ms']*1e3,1), 'K2', round(r['fused_spmv_ms']*1e3,1), 'us; launches/it', d['gpu_launches']/d['steps'], 'host us/it', round(d['host_enqueue_ms']*1e3/d['steps'],2))" || tail -3 gpurun_out/b_$c.err
done
