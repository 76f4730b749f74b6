#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for spec in "4,4,7:2" "4,4,7:3" "4,4,7:4" "4,2,7:2" "4,2,7:3" "8,4,7:1" "8,2,7:1"; do
  cfg=${spec%%:*}; occ=${spec##*:}
  ACG_THOMAS=$cfg ACG_THOMAS_OCC=$occ timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_thomas -s 2 -c 1 --csv --log-file gpurun_out/occ_${cfg}_${occ}.csv python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
done
