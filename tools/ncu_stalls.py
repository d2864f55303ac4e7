"""Stall-reason breakdown per SASS region of one kernel in an ncu report.
usage: ncu_stalls.py report kernel_index [topN]"""
import csv, subprocess, sys, collections
path, kid = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-id", f"::regex:gemm:{kid}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
st = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
iS, iN, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
tot = collections.Counter()
for r in data:
    for c in st:
        tot[c] += int(r[h.index(c)] or 0)
print("kernel stalls:", ", ".join(f"{k[6:]}={v}" for k, v in tot.most_common(10)))
idx = sorted(range(len(data)), key=lambda i: -int(data[i][iN] or 0))[:top]
for i in sorted(idx):
    r = data[i]
    reasons = sorted(((int(r[h.index(c)] or 0), c[6:]) for c in st), reverse=True)[:3]
    print(f"{i:5d} {r[iN]:>6s} exec={r[iE]:>8s} {r[iS].strip()[:60]:60s} {reasons}")
