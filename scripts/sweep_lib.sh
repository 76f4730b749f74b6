# run TAG ENV... : one bench line summarised (C3 unless BARGS says otherwise)
run() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e ${BARGS} > gpurun_out/sw_$tag.json 2> gpurun_out/sw_$tag.err
  python - "$tag" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/sw_{t}.json")); r=d["roofline"]
    print(f"{t:22s} it/s={d['value']:7.1f} K1={r['fused_prec_ms']:.3f}ms ({r['fused_prec_gbs']:5.0f} GB/s) K2={r['fused_spmv_ms']:.3f}ms ({r['fused_spmv_gbs']:5.0f})")
except Exception as e:
    print(t, "FAILED", e, open(f"gpurun_out/sw_{t}.err").read()[-300:])
PY
}
