#!/bin/bash
# Full round-end style measurement: tests, smoke, bench (with CPU baseline + e2e),
# reference arm, ncu launch list + full captures of the two fused sweeps
# (summarised on the box; the .ncu-rep files are kept only while under 60 MiB total).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r1}
nproc > gpurun_out/host_nproc.txt; lscpu | head -20 > gpurun_out/host_cpu.txt; free -g >> gpurun_out/host_cpu.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu_$TAG.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke: $(tail -1 gpurun_out/smoke_$TAG.log)"
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 10 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
for K in k_thomas_tm k_fused_spmv_pair2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_${TAG}_$K python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1; echo "$K full rc=$?"
  python scripts/ncu_summary.py gpurun_out/prof_${TAG}_$K.ncu-rep --hot > gpurun_out/prof_${TAG}_$K.txt 2>&1
done
total=$(du -cm gpurun_out/*.ncu-rep 2>/dev/null | tail -1 | cut -f1)
if [ "${total:-0}" -gt 60 ]; then rm -f gpurun_out/prof_${TAG}_k_fused_spmv_pair2.ncu-rep; fi
total=$(du -cm gpurun_out/*.ncu-rep 2>/dev/null | tail -1 | cut -f1)
if [ "${total:-0}" -gt 60 ]; then rm -f gpurun_out/*.ncu-rep; fi
