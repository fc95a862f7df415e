"""Map an ncu launch list of `ntt_sweep.py --ncu-plan` back to its
configurations (BASELINE cfg5 radix-split sweep, ncu evidence).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\\
sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none \\
        -k regex:"row_kernel|col_kernel|small_kernel" --csv --log-file L.csv \\
        python scripts/ntt_sweep.py --ncu-plan --out P.jsonl
    python scripts/cfg5_ncu.py P.jsonl L.csv > cfg5_ncu.jsonl

Per configuration: summed kernel time, DRAM bytes and their ratio to the
16n algorithmic bytes of a forward transform (read + write), the time-weighted
fmaheavy-pipe utilisation; then one line per N naming the fastest split.
(ncu replays serialise launches with cold caches: times are relative.)"""
from __future__ import annotations

import collections
import csv
import json
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out, cur = None, [], None
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if cur is None or cur["id"] != d["ID"]:
            cur = {"id": d["ID"], "kernel": d["Kernel Name"], "grid": d["Grid Size"], "m": {}}
            out.append(cur)
        cur["m"][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return out


def main(plan_path, csv_path):
    plan = [json.loads(x) for x in open(plan_path) if x.strip()]
    ls = launches(csv_path)
    i = 0
    best = {}
    for p in plan:
        k = ls[i:i + p["ncu_launches"]]
        i += p["ncu_launches"]
        n = 1 << p["log_n"]
        t = sum(x["m"]["gpu__time_duration.sum"] for x in k) / 1e3  # us
        by = sum(x["m"]["dram__bytes_read.sum"] + x["m"]["dram__bytes_write.sum"] for x in k)
        fh = sum(x["m"]["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"] *
                 x["m"]["gpu__time_duration.sum"] for x in k) / max(t * 1e3, 1e-9)
        rec = {"log_n": p["log_n"], "split": p["split"], "batch": p["batch"],
               "kernels": [x["kernel"].split("(")[0] for x in k],
               "ncu_us": round(t, 2), "ncu_us_per_poly": round(t / p["batch"], 4),
               "dram_bytes_per_poly": int(by / p["batch"]),
               "dram_over_16n": round(by / p["batch"] / (16 * n), 2),
               "fmaheavy_pct": round(fh, 1)}
        print(json.dumps(rec))
        if p["log_n"] not in best or rec["ncu_us"] < best[p["log_n"]]["ncu_us"]:
            best[p["log_n"]] = rec
    for log_n, r in sorted(best.items()):
        print(json.dumps({"log_n": log_n, "best_split": r["split"], "ncu_us_per_poly":
                          r["ncu_us_per_poly"], "dram_over_16n": r["dram_over_16n"],
                          "fmaheavy_pct": r["fmaheavy_pct"]}))


if __name__ == "__main__":
    main(*sys.argv[1:3])
