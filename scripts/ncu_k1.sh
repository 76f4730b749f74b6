#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1; shift
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_thomas -s 2 -c 1 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ncu_${TAG}.log 2>&1
echo "$TAG rc=$?"
