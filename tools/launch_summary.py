"""Summarise an ncu launch list of bench.py (cfg2 key-only step) into the
per-kernel table of profiles/*_summary.md and profiles/traffic.json.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --clock-control none --csv --log-file launches.csv \\
        python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-kv --no-clock-window
    python tools/launch_summary.py launches.csv [--traffic profiles/traffic.json]
"""
import argparse
import collections
import csv
import json

UNIT = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
# bench.py pass names of the kernels whose traffic feeds roofline.traffic
PASS_OF = {"k_page_partition": "partition", "k_page_count": "count", "k_emit": "emit"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic", default="")
    ap.add_argument("--step-kernels", type=int, default=9, help="launches per bench step")
    ap.add_argument("--aggregate", type=int, default=0,
                    help="per-kernel totals over the whole list divided by this many iterations")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ik, im, iv, iu, iid = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        v = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1.0)
        per.setdefault(int(r[iid]), {"name": r[ik]})[r[im]] = v
    if args.aggregate:
        agg = collections.OrderedDict()
        for d in per.values():
            name = d["name"].split("(")[0].replace("void ", "").replace("rsb::", "")
            a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
            a[0] += 1
            a[1] += d.get("gpu__time_duration.sum", 0.0)
            a[2] += d.get("dram__bytes_read.sum", 0.0)
            a[3] += d.get("dram__bytes_write.sum", 0.0)
        total = sum(a[1] for a in agg.values())
        print("| kernel | launches/iter | us/iter | share | DRAM read MB/iter | DRAM write MB/iter |")
        print("|---|---|---|---|---|---|")
        k = args.aggregate
        for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            print(f"| {name} | {a[0] / k:g} | {a[1] / k / 1e3:.1f} | {100 * a[1] / total:.1f}% | "
                  f"{a[2] / k / 1e6:.1f} | {a[3] / k / 1e6:.1f} |")
        print(f"\ntotal {total / k / 1e3:.1f} us per iteration under ncu (serialised, cold caches)")
        return
    last = list(per)[-args.step_kernels:]
    total = sum(per[i]["gpu__time_duration.sum"] for i in last)
    print("| kernel | us | share | DRAM read MB | DRAM write MB |")
    print("|---|---|---|---|---|")
    traffic = {}
    for i in last:
        d = per[i]
        name = d["name"].split("(")[0].replace("void ", "").replace("rsb::", "")
        t = d["gpu__time_duration.sum"]
        rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        print(f"| {name} | {t / 1e3:.1f} | {100 * t / total:.1f}% | {rd / 1e6:.1f} | {wr / 1e6:.1f} |")
        for prefix, pas in PASS_OF.items():
            if name.startswith(prefix):
                traffic[pas] = rd + wr
    print(f"\nstep total {total / 1e3:.1f} us under ncu (serialised, cold caches)")
    if args.traffic:
        json.dump(traffic, open(args.traffic, "w"), indent=1)
        print("traffic ->", args.traffic, traffic)


if __name__ == "__main__":
    main()
