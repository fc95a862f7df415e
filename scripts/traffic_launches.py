"""DRAM bytes per limb-product of each kernel of the fused product step, from
an ncu launch list (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv`) of `bench.py` at one configuration.

    python scripts/traffic_launches.py launches.csv LOG_N [--update profiles/traffic.json]

Products per launch come from each launch's grid size: the fused row kernel
runs N1 = n / 4096 CTAs per limb-product; the forward column kernel covers
a and b (2 x 4096 columns per product, SPAN columns per CTA), the inverse
one c only.  Only the fused-product instantiations (LB = 32 rows with the
Karatsuba middle, LB = 32 columns) are counted."""
from __future__ import annotations

import argparse
import csv
import json
import re
from collections import defaultdict


def span(log_n1: int) -> int:  # ColGeom<..>::SPAN for 4096-word rows
    want = 1 if log_n1 >= 4 else 16 >> log_n1
    return 256 * want


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("log_n", type=int)
    ap.add_argument("--update", default=None)
    args = ap.parse_args()
    log_n1 = args.log_n - 12
    lines = [ln for ln in open(args.csv) if ln.startswith('"')]
    launches = defaultdict(dict)
    for r in csv.DictReader(lines):
        launches[int(r["ID"])]["name"] = r["Kernel Name"]
        launches[int(r["ID"])]["grid"] = int(r["Grid Size"].strip("()").split(",")[0])
        launches[int(r["ID"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    acc = defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0])  # read, write, ns, products, launches
    for L in launches.values():
        nm = L["name"]
        m = re.match(r"void (col|row)_kernel<([^>]*)>", nm)
        if not m:
            continue
        t = [x.strip() for x in m.group(2).split(",")]
        if m.group(1) == "row":
            if not (t[0] == "12" and t[2] == "1" and t[-1] == "32"):
                continue
            kind, prods = "row_fused", L["grid"] / (1 << log_n1)
        else:
            if not (int(t[0]) == log_n1 and t[2] == "32"):
                continue
            inv = t[1] == "1"
            kind = "col_inv" if inv else "col_fwd"
            prods = L["grid"] * span(log_n1) / ((1 if inv else 2) * 4096)
        a = acc[kind]
        a[0] += L.get("dram__bytes_read.sum", 0)
        a[1] += L.get("dram__bytes_write.sum", 0)
        a[2] += L.get("gpu__time_duration.sum", 0)
        a[3] += prods
        a[4] += 1
    out = {}
    for k, (rd, wr, ns, prods, cnt) in acc.items():
        out[k] = {"n": 1 << args.log_n, "bytes_per_product": int((rd + wr) / prods),
                  "dram_read_per_product": int(rd / prods),
                  "dram_write_per_product": int(wr / prods),
                  "ncu_us_per_launch": round(ns / cnt / 1e3, 2), "launches": cnt}
    tot = sum(v["bytes_per_product"] for v in out.values())
    print(json.dumps({"log_n": args.log_n, "kernels": out, "total_per_product": tot,
                      "ratio_to_24n": round(tot / (24 << args.log_n), 3)}, indent=1))
    if args.update:
        with open(args.update) as fh:
            rec = json.load(fh)
        rec.setdefault("by_n", {})[str(1 << args.log_n)] = {**out, "source": args.csv}
        with open(args.update, "w") as fh:
            json.dump(rec, fh, indent=1)
            fh.write("\n")


if __name__ == "__main__":
    main()
