#!/bin/bash
# Round-2 check: whole GPU suite (timed), smoke, default bench line, all configs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
s0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1
echo "gpu suite rc=$? in $(( $(date +%s) - s0 )) s"; grep -E "^FAILED|passed|failed" gpurun_out/pytest_gpu.log | tail -12
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench.json
SKIP_TESTS=1 bash scripts/gpu_configs.sh
