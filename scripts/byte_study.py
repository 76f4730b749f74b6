"""Fused vs unfused (and matrix-explicit) per-iteration DRAM bytes at C2 from ncu
launch lists (scripts/gpu_r2b.sh: ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum on bench.py --config c2 --steps 2
--warmup 3 [--variant standard | --backend csr]).

Per-launch DRAM bytes are averaged per kernel and multiplied by the launches one
loop iteration makes (acg_runtime.cu iterate_interleaved / iterate_standard):
  interleaved: K1 k_thomas_tm<Fused>, K2 k_fused_spmv_pair2, 2 x k_tree2_wide
  standard:    k_apply, 3 x k_dot_partials, 3 x k_axpy, k_thomas_tm<!Fused>,
               k_scal, 3 x (k_tree1 + k_tree2_wide)
  csr:         k_csr_spmv, 3 x k_dot_partials, 3 x k_axpy, k_csr_tridiag, k_scal,
               3 x (k_tree1 + k_tree2_wide)
and compared with the algorithmic byte models of bench.py.
usage: python scripts/byte_study.py gpurun_out/ncu_c2_{il,std,csr}.csv
"""
import csv
import sys
from collections import defaultdict

M, NZ, S = 512, 128, 8
N = M * M * NZ
NNZ = N + 4 * (M - 1) * M * NZ + 2 * (NZ - 1) * M * M
MODEL = {"il": S * (11 * N + 8 * M * M), "std": S * (20 * N + 8 * M * M),
         "csr": 8 * N + NNZ * (S + 4) + S * (2 * N + 5 * N + 16 * N)}
PER_IT = {
    "il": {"k_thomas_tm<double, 0, 1": 1, "k_fused_spmv_pair2": 1, "k_tree2_wide": 2},
    "std": {"k_apply": 1, "k_dot_partials": 3, "k_axpy": 3, "k_thomas_tm<double, 0, 0": 1,
            "k_scal": 1, "k_tree1": 3, "k_tree2_wide": 3},
    "csr": {"k_csr_spmv": 1, "k_dot_partials": 3, "k_axpy": 3, "k_csr_tridiag": 1, "k_scal": 1,
            "k_tree1": 3, "k_tree2_wide": 3},
}


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = [i for i, r in enumerate(rows) if r[0] == "ID"][0]
    idx = {k: i for i, k in enumerate(rows[hi])}
    per = defaultdict(dict)
    for r in rows[hi + 1:]:
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        if r[idx["Metric Name"]] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        else:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per[r[idx["ID"]]][r[idx["Metric Name"]]] = v
        per[r[idx["ID"]]]["name"] = r[idx["Kernel Name"]]
    return per


def main(paths):
    print("| loop | kernel | launches/it | DRAM read (MB) | DRAM write (MB) | us/launch (ncu) |")
    print("|---|---|---|---|---|---|")
    totals = {}
    for path in paths:
        tag = path.rsplit("_", 1)[-1].split(".")[0]
        per = load(path)
        tot_b, tot_t = 0.0, 0.0
        for key, n in PER_IT[tag].items():
            ls = [m for m in per.values() if key in m["name"]]
            if not ls:
                continue
            rd = sum(m.get("dram__bytes_read.sum", 0) for m in ls) / len(ls)
            wr = sum(m.get("dram__bytes_write.sum", 0) for m in ls) / len(ls)
            t = sum(m.get("gpu__time_duration.sum", 0) for m in ls) / len(ls)
            tot_b += n * (rd + wr)
            tot_t += n * t
            print(f"| {tag} | `{key.split('<')[0]}` | {n} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {t:.1f} |")
        totals[tag] = (tot_b, tot_t)
    print()
    print("| loop | DRAM bytes / iteration (ncu) | model | ncu / model | kernel time / iteration (ncu, serialised) |")
    print("|---|---|---|---|---|")
    for tag, (b, t) in totals.items():
        print(f"| {tag} | {b / 1e9:.3f} GB | {MODEL[tag] / 1e9:.3f} GB | {b / MODEL[tag]:.3f} | {t:.0f} us |")


if __name__ == "__main__":
    main(sys.argv[1:])
