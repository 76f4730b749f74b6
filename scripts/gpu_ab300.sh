cd "${GRAFT_REPO_ROOT:-/root/repo}"
A=$PWD/paper_1302_7193_b200/alt_libacg_cuda.so
for i in 1 2 3; do
for v in base pre; do
  if [ $v = pre ]; then export ACG_LIB_OVERRIDE=$A; else unset ACG_LIB_OVERRIDE; fi
  timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-ktime 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
