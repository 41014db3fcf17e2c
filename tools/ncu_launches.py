"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel as markdown.
Usage: python tools/ncu_launches.py launches.csv > launches.md"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ix = {k: i for i, k in enumerate(h)}
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[start + 1:]:
    if len(r) != len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    us = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3 if unit == "ms" else v / 1e3)
    name = r[ix["Kernel Name"]].split("(")[0][:70]
    tot[name] += us
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
print("| share | total us | launches | mean us | kernel |")
print("|---|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"| {100 * v / T:.1f}% | {v:.1f} | {cnt[k]} | {v / cnt[k]:.2f} | {k} |")
