#!/bin/bash
# Round-2 check 2: pruned library, CSR backend, drop-in smoke, sanitizers; C1 launch-mode
# study; C2 fused / standard / CSR comparison with an ncu dram__bytes capture per launch.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/pytest_gpu.log 2>&1
echo "gpu suite rc=$?"; tail -8 gpurun_out/pytest_gpu.log
for v in "base:" "nopdl:ACG_PDL=0"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 300 python bench.py --config c1 --steps 2000 --warmup 20 --no-cpu --no-e2e \
      --sustain-steps 0 > gpurun_out/c1_$tag.json 2> gpurun_out/c1_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/c1_$tag.json'));r=d['roofline'];print('c1 $tag', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us/it K1', round(r['fused_prec_ms']*1e3,2), 'K2', round(r['fused_spmv_ms']*1e3,2))" || tail -5 gpurun_out/c1_$tag.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 8 --warmup 3 \
    --no-cpu --no-e2e --no-ktime --sustain-steps 0 > /dev/null 2>&1; echo "ncu c1 rc=$?"
for b in "il:--variant interleaved" "std:--variant standard" "csr:--backend csr"; do
  tag=${b%%:*}; args=${b#*:}
  timeout 300 python bench.py --config c2 --steps 100 --warmup 5 --no-cpu --sustain-steps 0 $args \
      > gpurun_out/c2_$tag.json 2> gpurun_out/c2_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/c2_$tag.json'));print('c2 $tag', round(d['value'],1), 'it/s', round(d['achieved_gbs_iteration']), 'GB/s model', d['algorithmic_bytes_iteration'], 'launches/it', d['gpu_launches']/d['steps'])" || tail -5 gpurun_out/c2_$tag.err
  # one iteration's launches with DRAM bytes (warmup 3 + 2 steps; kernels of the last iterations)
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/ncu_c2_$tag.csv \
      python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-ktime \
      --sustain-steps 0 $args > /dev/null 2>&1; echo "ncu c2 $tag rc=$?"
done
