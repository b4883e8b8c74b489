"""Per-opcode executed instructions and stall samples of an ncu report's SASS page
(run here, no GPU):  python tools/ncu_sass.py report.ncu-rep [--top N]"""
import csv
import subprocess
import sys
from collections import Counter


def main(path, top=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = rows[2:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    samples = sum(int(r[iS] or 0) for r in data)
    ex = sum(int(r[iE] or 0) for r in data)
    op, opex = Counter(), Counter()
    for r in data:
        t = r[1].split()
        if not t:
            continue
        m = t[1] if t[0].startswith("@") else t[0]
        m = m.split(".")[0]
        op[m] += int(r[iS] or 0)
        opex[m] += int(r[iE] or 0)
    print(f"{path}: {samples} stall samples, {ex} warp instructions")
    for k, v in opex.most_common(18):
        print(f"  {k:10s} exec {v:11d} ({100 * v / ex:5.1f}%)  stall samples {100 * op[k] / samples:5.1f}%")
    if top:
        for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:top]:
            print("   ", r[0][-5:], r[1][:64].ljust(64), r[iS], r[iE])


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 0
    for p in args:
        if p.endswith(".ncu-rep"):
            main(p, top)
