#!/bin/bash
# ncu --set full captures of the two fused sweeps at C3 (one launch each).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r1}
for K in k_fused_prec k_fused_spmv; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/prof_${TAG}_$K python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e ${EXTRA} > gpurun_out/ncu_${TAG}_$K.log 2>&1
  echo "$K rc=$?"
done
ls -la gpurun_out/
