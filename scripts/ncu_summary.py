"""Summaries of ncu output for profiles/: (1) a launch list (--csv
--metrics gpu__time_duration.sum) -> per-kernel count, total and share;
(2) a --page raw --csv export of a --set full capture -> selected metrics per
launch as JSON (the traffic figure bench.py reports)."""
import csv
import json
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        v = v / 1000.0 if r[iu] == "ns" else (v * 1000.0 if r[iu] == "ms" else v)
        name = r[ik].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(x[1] for x in agg.values())
    out = sorted(([k, v[0], v[1], v[1] / tot] for k, v in agg.items()), key=lambda x: -x[2])
    print("kernel,launches,total_us,share")
    for k, c, t, f in out:
        print(f"{k},{c},{t:.1f},{f:.4f}")


def full(path, kernel, algorithmic):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    recs = []
    for r in rows[2:]:
        if kernel not in r[h.index("Kernel Name")]:
            continue
        recs.append({k: [r[h.index(k)], rows[1][h.index(k)]] for k in KEYS if k in h})
    def byt(rec, k):
        v, u = rec[k]
        v = float(v.replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    per = [byt(x, "dram__bytes_read.sum") + byt(x, "dram__bytes_write.sum") for x in recs]
    print(json.dumps({"kernel": kernel, "bytes_per_launch": sum(per) / max(1, len(per)),
                      "algorithmic_bytes": algorithmic, "per_launch": recs}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]))
