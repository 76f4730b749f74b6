#!/bin/bash
# Round-end numbers: default bench line (all legs), the reference arm, every
# config, and the C1 small-grid line at 1000 steps.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
cat gpurun_out/final_bench_ref.json
SKIP_TESTS=1 bash scripts/gpu_configs.sh
timeout 300 python bench.py --config c1 --steps 1000 --warmup 20 --no-cpu --no-ktime --sustain-steps 0 > gpurun_out/final_c1.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/final_c1.json')); print('c1 1000 steps', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us', round(d['frac_of_peak_iteration'],3), 'e2e', round(d['e2e']['value'],1))"
