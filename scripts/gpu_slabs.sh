#!/bin/bash
# Decomposition cost on one GPU: p virtual slabs in one process (device-copy halos), and
# N rank processes sharing the GPU through the peer-memory transport (ACG_SAME_GPU=1).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in c3 c5; do
  st=50; [ $c = c5 ] && st=10
  for p in 1 2 4 8; do
    timeout 600 python bench.py --config $c --slabs $p --steps $st --warmup 5 --no-cpu --no-e2e \
        --sustain-steps 0 > gpurun_out/sl_${c}_$p.json 2> gpurun_out/sl_${c}_$p.err
    python -c "import json;d=json.load(open('gpurun_out/sl_${c}_$p.json'));print('$c slabs=$p', round(d['value'],2), 'it/s', round(d['ms_per_step'],3), 'ms/it launches/it', d['gpu_launches']/d['steps'], 'exact', d['exact_tree'])" || tail -3 gpurun_out/sl_${c}_$p.err
  done
  for n in 2 4 8; do
    ACG_SAME_GPU=1 timeout 900 python bench.py --gpus $n --config $c --steps $st --warmup 5 --no-cpu \
        --no-e2e --sustain-steps 0 > gpurun_out/rk_${c}_$n.json 2> gpurun_out/rk_${c}_$n.err
    python -c "import json;d=[json.loads(l) for l in open('gpurun_out/rk_${c}_$n.json') if l.startswith('{')][-1];print('$c ranks=$n (one GPU)', round(d['value'],2), 'it/s', round(d['ms_per_step'],3), 'ms/it launches/it', d['gpu_launches']/d['steps'], 'verified', d['verified_vs_1gpu']['ok'])" || tail -3 gpurun_out/rk_${c}_$n.err
  done
done
