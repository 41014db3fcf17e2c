"""Summarise an .ncu-rep: key metrics per launch + top stall reasons + hottest source lines."""
import csv
import io
import subprocess
import sys

KEYS = ['Duration', 'Elapsed Cycles', 'Registers Per Thread', 'Achieved Occupancy', 'Executed Ipc Active',
        'Issue Slots Busy', 'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'Block Size',
        'Grid Size', 'DRAM Throughput', 'Compute (SM) Throughput', 'L2 Hit Rate', 'L1/TEX Hit Rate']


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, src_lines=25):
    r = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = r[0]
    for row in r[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in KEYS:
            print(d["ID"], d["Kernel Name"][:40], "|", d["Metric Name"], d["Metric Value"], d["Metric Unit"])
    r = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h = r[0]
    for v in r[2:]:
        st = []
        for i, k in enumerate(h):
            if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(v[i].replace(",", "")), k.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        fp = [v[i] for i, k in enumerate(h) if k == "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
        dr = [v[i] for i, k in enumerate(h) if k in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
        print("stalls:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:6]), "| fp64 pipe %:", fp,
              "| dram r/w:", dr)
    if src_lines:
        out = run([rep, "--page", "source", "--csv", "--print-source", "sass"])
        rows = list(csv.reader(io.StringIO(out)))
        if rows:
            hh = rows[0]
            try:
                ci = hh.index("Warp Stall Sampling (All Samples)")
            except ValueError:
                ci = None
            if ci is not None:
                data = []
                for rr in rows[1:]:
                    if len(rr) == len(hh):
                        try:
                            data.append((float(rr[ci] or 0), rr))
                        except ValueError:
                            pass
                tot = sum(x for x, _ in data) or 1
                si = hh.index("Source") if "Source" in hh else 1
                for x, rr in sorted(data, key=lambda t: -t[0])[:src_lines]:
                    print(f"{100 * x / tot:5.1f}%  {rr[si][:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
