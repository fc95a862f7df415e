"""Summarise an `ncu --page raw --csv` export: per kernel, duration, pipe
utilisation, issue activity, top stall reasons and DRAM bytes."""
import csv
import sys

KEYS = [
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sass__inst_executed_register_spilling",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        dur = d.get("gpu__time_duration.sum", "?")
        print(f"== {name} dur {dur} {u.get('gpu__time_duration.sum', '')}")
        stalls = {k.split("stalled_")[1].split("_per_issue")[0]: float(v)
                  for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and
                  k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        print("  stalls/issue: " + ", ".join(f"{k}={v:.2f}" for k, v in top))
        for k in KEYS:
            if k in d:
                print(f"   {k} {d[k]} {u.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1])
