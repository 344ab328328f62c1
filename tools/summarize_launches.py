"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel
mean time and share of the step (ncu times are cold-cache and serialised:
compare shares, not absolutes)."""
import csv
import sys
from collections import OrderedDict


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[h + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in agg.items():
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / total:.1f}% |")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
