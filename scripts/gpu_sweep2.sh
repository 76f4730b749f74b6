#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=3 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for cfg in "2,8,7" "2,2,7"; do
  ACG_THOMAS=$cfg timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "solve_bit_exact or operators_bit_exact or config1 or slab" > gpurun_out/pytest_$cfg.log 2>&1; echo "cfg $cfg: $(tail -1 gpurun_out/pytest_$cfg.log)"
done
source scripts/sweep_lib.sh
for cfg in "2,4,7" "4,4,7" "2,8,7" "4,8,7" "2,2,7" "4,4,5" "8,4,7"; do run "ex_$cfg" ACG_THOMAS=$cfg; done
BARGS="--math fast"
for cfg in "4,4,7" "2,8,7" "4,8,7"; do run "fast_$cfg" ACG_THOMAS=$cfg; done
