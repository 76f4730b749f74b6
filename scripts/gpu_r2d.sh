#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
./scripts/micro/fp64_latency | tee gpurun_out/fp64_latency.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_variants.py tests/test_csr_backend.py -m gpu -q -x 2>&1 | tail -2
for c in c1 c2; do
  timeout 300 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu --no-e2e \
      --sustain-steps 0 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b_$c.json'));r=d['roofline'];print('$c', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,2), 'us/it', round(d['frac_of_peak_iteration']*100,1), '% iter; K1', round(r['fused_prec_ms']*1e3,1), 'K2', round(r['fused_spmv_ms']*1e3,1), 'us; launches/it', d['gpu_launches']/d['steps'])" || tail -3 gpurun_out/b_$c.err
done
timeout 300 python bench.py --config c2 --backend csr --steps 50 --warmup 5 --no-cpu --sustain-steps 0 > gpurun_out/c2_csr.json 2> gpurun_out/c2_csr.err
python -c "import json;d=json.load(open('gpurun_out/c2_csr.json'));print('c2 csr', round(d['value'],1), 'it/s', round(d['achieved_gbs_iteration']), 'GB/s model; e2e', round(d['e2e']['value'],1))" || tail -5 gpurun_out/c2_csr.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/ncu_c2_csr.csv \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-ktime \
    --sustain-steps 0 --backend csr > /dev/null 2>&1; echo "ncu c2 csr rc=$?"
