"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0, []])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][:70]
        v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
        agg[k][0] += 1
        agg[k][1] += v
        agg[k][2].append(v)
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
    print("| share | total us | launches | mean us | kernel |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| {100 * v[1] / tot:.1f}% | {v[1]:.1f} | {v[0]} | {v[1] / v[0]:.2f} | {k} |")


if __name__ == "__main__":
    main(sys.argv[1])
