"""Static checks on the built SASS: wide uniform descriptors must be even-aligned
(an odd desc[URn] traps with an illegal-instruction error on sm_100)."""
import re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1302_7193_b200/libacg_cuda.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
bad = 0
fn = "?"
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
    for d in re.findall(r"desc\[UR(\d+)\]", line):
        if int(d) % 2:
            bad += 1
            print(fn[:90], line.strip()[:110])
print(f"odd descriptors: {bad}")
sys.exit(1 if bad else 0)
