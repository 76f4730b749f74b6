#!/bin/bash
# Round-2 check: new contract/convergence/sanitizer tests, then the whole GPU suite, then bench.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 2400 python -m pytest tests/test_runtime_contract.py tests/test_convergence.py \
    tests/test_sanitizers.py tests/test_bench_contract.py -m gpu -q --durations=40 \
    > gpurun_out/pytest_new.log 2>&1
echo "new tests rc=$?"
tail -5 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q --durations=25 \
    --deselect tests/test_sanitizers.py > gpurun_out/pytest_gpu.log 2>&1
echo "gpu suite rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.json
