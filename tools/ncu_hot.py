"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iS, iN, iA, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Address"), h.index("Instructions Executed")
data = [(int(r[iN] or 0), r[iA], r[iS].strip(), r[iE]) for r in rows[2:] if len(r) > iN]
tot = sum(d[0] for d in data)
print("total samples", tot)
for i, d in enumerate(data):
    pass
idx = sorted(range(len(data)), key=lambda i: -data[i][0])[:top]
for i in sorted(idx):
    s, a, src, ex = data[i]
    print(f"{i:5d} {s:7d} {100*s/tot:5.1f}%  exec={ex:>8s}  {src}")
if len(sys.argv) > 3:
    # region sums: comma list of a-b index ranges
    for rg in sys.argv[3].split(","):
        a, b = map(int, rg.split("-"))
        print(f"region {a}-{b}: {sum(d[0] for d in data[a:b+1])} samples")
    for i in range(int(sys.argv[4]), int(sys.argv[5])):
        print(i, data[i][0], data[i][3], data[i][2])
