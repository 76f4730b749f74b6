#!/bin/bash
# ncu full capture of one kernel (regex $1) at C3 + launch list; tag $2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
K=${1:-k_thomas_tm}; TAG=${2:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_${TAG}_$K python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/prof_${TAG}.log 2>&1; echo "$K full rc=$?"
