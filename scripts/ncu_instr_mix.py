"""Instruction mix and stall reasons per SASS opcode from an ncu source page.

usage: ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
       python scripts/ncu_instr_mix.py src.csv <points>   (points = columns * levels)
"""
import collections
import csv
import re
import sys


def main(path, points):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    inst = collections.Counter()
    wait = collections.Counter()
    stalls = collections.Counter()
    total = 0
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        op = re.sub(r"^@!?U?P\w+\s+", "", r[ix["Source"]].strip()).split(" ")[0].split(".")[0]
        n = int(r[ix["Instructions Executed"]] or 0)
        total += n
        inst[op] += n
        wait[op] += int(r[ix["stall_wait"]] or 0)
        for k in hdr:
            if k.startswith("stall_") and "Not Issued" not in k:
                stalls[k] += int(r[ix[k]] or 0)
    per = 32.0 / points
    print(f"warp instructions {total}, thread instructions per point {total * per:.1f}")
    print("per point:", ", ".join(f"{k} {v * per:.1f}" for k, v in inst.most_common(20)))
    print("stall samples:", ", ".join(f"{k[6:]} {v}" for k, v in stalls.most_common(12) if v))
    print("stall_wait by opcode:", ", ".join(f"{k} {v}" for k, v in wait.most_common(10)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
