"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X.csv)
into per-kernel totals and shares, plus the per-launch list.
usage: launch_summary.py launches.csv [header line ...]"""
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name)            # drop the argument list
    name = name.replace("void ", "").replace("srl::", "")
    return name.strip()


def main(path, header):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    seq = [(short(r[iK]), float(r[iV].replace(",", ""))) for r in rows[1:] if r[iM] == "gpu__time_duration.sum"]
    tot = {}
    for k, ns in seq:
        c, t = tot.get(k, (0, 0.0))
        tot[k] = (c + 1, t + ns)
    all_us = sum(t for _, t in tot.values()) / 1e3
    for line in header:
        print("# " + line)
    print("# per-launch times are cold-cache and serialised: compare SHARES with bench.py's breakdown, not absolutes\n")
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>7s}")
    for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {c:8d} {t / 1e3:10.1f} {t / 1e3 / c:9.2f} {100 * t / 1e3 / all_us:6.1f}%")
    print(f"{'TOTAL':40s} {len(seq):8d} {all_us:10.1f}\n")
    print("# per-launch list (kernel, ns)")
    for k, ns in seq:
        print(f"{k}\t{int(ns)}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
