"""Summaries of ncu evidence for profiles/: launch-list shares and key metrics of full captures."""
import csv
import json
import subprocess
import sys
from collections import defaultdict


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    K, M, V = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > V and r[M] == "gpu__time_duration.sum":
            name = r[K].split("(")[0].replace("void vinp::", "").replace("vinp::", "")
            agg[name][0] += 1
            agg[name][1] += float(r[V].replace(",", ""))
    unit = "ns"
    tot = sum(v[1] for v in agg.values())
    return {k: {"launches": v[0], "total_ms": round(v[1] / 1e6, 3), "share": round(v[1] / tot, 4)}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}, round(tot / 1e6, 3)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")][:80]}
    for w in WANT:
        if w in h:
            res[w] = f"{v[h.index(w)]} {u[h.index(w)]}".strip()
    return res


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        shares, tot = launch_shares(sys.argv[2])
        print(json.dumps({"total_ms": tot, "kernels": shares}, indent=1))
    else:
        for rep in sys.argv[2:]:
            print(json.dumps(full_metrics(rep), indent=1))
