#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_variants.py tests/test_multirank_ipc.py tests/test_convergence.py -m gpu -q -x -k "float32 or f32 or c4 or variant or ipc" 2>&1 | tail -2
bash scripts/gpu_ab.sh c4 30
ACG_QUAD_D=2 bash scripts/gpu_ab.sh c4 30 | grep new
