#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 900 python -m pytest tests/test_variants.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
bash scripts/gpu_ab.sh tall 30
