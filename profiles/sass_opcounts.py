"""Static SASS op counts per kernel of libgdwd_b200.so (cuobjdump -sass):
python profiles/sass_opcounts.py > profiles/r02/sass_opcounts.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2305_12019_b200" / "libgdwd_b200.so"
OPS = re.compile(r"\b(DMMA\.8x8x4|LDTM\.x\d+|STTM\.x\d+|UBLKCP\.S|SYNCS|UCGABAR\w*|LDGSTS(?:\.\w+)*|DFMA|REDG|LDS\.128)\b")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    counts, name = collections.OrderedDict(), None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            counts[name] = collections.Counter()
            continue
        if name:
            m = OPS.search(line.split("/*")[1] if line.count("/*") >= 2 else line)
            if m:
                op = m.group(1)
                op = "LDGSTS" if op.startswith("LDGSTS") else op
                counts[name][op] += 1
    names = list(counts)
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    print("# Static SASS op counts per kernel (cuobjdump -sass of libgdwd_b200.so, sm_100a).")
    print("# DMMA = FP64 tensor-core MMA; LDTM/STTM = tensor-memory load/store (tcgen05.ld/st);")
    print("# UBLKCP = bulk copy (TMA engine, cp.async.bulk); SYNCS = mbarrier ops; UCGABAR = cluster barrier;")
    print("# LDGSTS = cp.async; DFMA = FP64 FMA (CUDA cores); REDG = global reduction (grid barrier arrive).")
    keep = ("DMMA", "LDTM", "STTM", "UBLKCP", "SYNCS", "UCGABAR", "LDGSTS")
    for n, d in sorted(zip(dem, (counts[k] for k in names))):
        if any(op.startswith(keep) for op in d):
            print(n[:150])
            print("    " + ", ".join(f"{k} {v}" for k, v in sorted(d.items())))


if __name__ == "__main__":
    main()
