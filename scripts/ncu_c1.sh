#!/bin/bash
# Full ncu captures of K1 and K2 at C1 (128^2 x 64, L2-resident): where the
# small-grid iteration goes.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for k in k_thomas_tm k_fused_spmv_pair2; do
  timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:$k -s 20 -c 1 \
      -o gpurun_out/c1_$k python bench.py --config c1 --steps 30 --warmup 3 --no-cpu --no-e2e --no-ktime \
      --sustain-steps 0 > gpurun_out/ncu_c1_$k.log 2>&1
  echo "$k rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -c 200 --csv \
    --log-file gpurun_out/c1_launches2.csv python bench.py --config c1 --steps 40 --warmup 3 --no-cpu --no-e2e \
    --no-ktime --sustain-steps 0 > /dev/null 2>&1
echo "launches rc=$?"
