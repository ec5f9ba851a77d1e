"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` log into a per-kernel launch list."""
import collections
import csv
import sys

src, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr, data = rows[0], rows[1:]
iN, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in data:
    if r[iM] != "gpu__time_duration.sum":
        continue
    name = r[iN].split("(")[0].replace("void ", "").replace("lmra_dev::", "")
    name = name.replace("(int)", "")
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + float(r[iV].replace(",", "")) / 1000.0)
total = sum(t for _, t in agg.values())
print(f"# ncu launch list{', ' + title if title else ''}")
print("# `ncu --metrics gpu__time_duration.sum --clock-control none`; serialised, cold-cache")
print("# per-launch times: compare SHARES, not absolutes.\n")
print(f"{'kernel':55s} {'launches':>9s} {'total_us':>10s} {'share':>7s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:55]:55s} {c:9d} {t:10.1f} {t / total:7.3f}")
