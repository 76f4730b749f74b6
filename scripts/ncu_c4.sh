#!/bin/bash
# ncu --set full of the fp32 sweeps at C4 (k_thomas_tm2, k_fused_spmv_pair), summarised.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for K in k_thomas_tm2 k_fused_spmv_pair; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K}" -s 2 -c 1 \
    -o gpurun_out/prof_c4_$K python bench.py --config c4 --steps 3 --warmup 2 --no-cpu --no-e2e \
    --sustain-steps 0 > /dev/null 2>&1; echo "$K rc=$?"
  python scripts/ncu_summary.py gpurun_out/prof_c4_$K.ncu-rep --hot > gpurun_out/prof_c4_$K.txt 2>&1
  rm -f gpurun_out/prof_c4_$K.ncu-rep
done
