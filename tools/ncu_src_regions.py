"""Stall samples of one kernel per source line / region, from an ncu `--page source --csv` export (SASS
view) and the line table of the same build (nvdisasm -g of the kernel's cubin):
   python tools/ncu_src_regions.py SRC_CSV SASS_TXT KERNEL_MANGLED [top]
SASS_TXT: `nvdisasm -g -c obj.cubin` of the object the library was built from (same flags)."""
import collections
import csv
import re
import sys

src_csv, sass_txt, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
lines = open(sass_txt).read().split("\n")
start = next(i for i, l in enumerate(lines) if ".text." + kname in l and l.startswith("//"))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//") and ".text." in lines[i]), len(lines))
cur, offmap = None, {}
for l in lines[start:end]:
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m2 = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m2 and cur:
        offmap[int(m2.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
h, data = rows[hi], rows[hi + 1:]
base = int(data[0][0], 16)
i_all = h.index("Warp Stall Sampling (All Samples)")
cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
per = collections.defaultdict(collections.Counter)
for r in data:
    c = offmap.get(int(r[0], 16) - base, ("?", 0))
    per[c]["all"] += int(r[i_all] or 0)
    for i in cols:
        per[c][h[i][6:]] += int(r[i] or 0)
tot = sum(v["all"] for v in per.values())
print(f"{kname}: {tot} stall samples")
for c, v in sorted(per.items(), key=lambda kv: -kv[1]["all"])[:top]:
    st = sorted(((k, x) for k, x in v.items() if k != "all"), key=lambda kv: -kv[1])[:3]
    print(f"{c[0]}:{c[1]:<5d} {v['all'] / tot * 100:5.1f}%  " + " ".join(f"{k}={x / tot * 100:.1f}" for k, x in st))
