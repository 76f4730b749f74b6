#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.log)"
source scripts/sweep_lib.sh
for spec in "4,4,7:1:4" "4,4,7:0:4" "4,4,7:1:3" "4,2,7:1:2" "4,2,7:1:3"; do
  IFS=: read cfg h occ <<< "$spec"
  run "h${h}_${cfg}_o${occ}" ACG_THOMAS=$cfg ACG_L2_HINTS=$h ACG_THOMAS_OCC=$occ
  ACG_THOMAS=$cfg ACG_L2_HINTS=$h ACG_THOMAS_OCC=$occ timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_thomas -s 2 -c 1 --csv --log-file gpurun_out/hint_${h}_${cfg}_${occ}.csv python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
done
BARGS="--math fast"
for spec in "4,4,7:1:4" "4,4,7:1:3" "4,2,7:1:2"; do
  IFS=: read cfg h occ <<< "$spec"
  run "fast_h${h}_${cfg}_o${occ}" ACG_THOMAS=$cfg ACG_L2_HINTS=$h ACG_THOMAS_OCC=$occ
done
