"""Write profiles/ncu_summary.json: the headline counters of each --set full capture of a round
(DRAM rate, L2 hit rate of the gather, L2 throughput, issue activity, RED traffic), keyed like
bench.py's workload key so the bench line can cite the evidence behind its roofline."""
import csv
import json
import os
import sys

KEYS = {
    "time_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_GB": ("dram__bytes_read.sum", 1e-9),
    "dram_write_GB": ("dram__bytes_write.sum", 1e-9),
    "dram_TBps": ("dram__bytes.sum.per_second", 1e-12),
    "l2_read_hit_pct": ("lts__t_sector_op_read_hit_rate.pct", 1),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "l2_red_requests": ("lts__t_requests_srcunit_tex_op_red.sum", 1),
}
UNIT = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "byte": 1,
        "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6, "%": 1, "": 1,
        "request": 1, "sector": 1}
WORKLOADS = {  # capture -> bench workload key
    "full_reddit_mean": "reddit-mean-segment-cb21179-n1",
    "full_rmat_sum": "rmat-sum-segment-cb0-n1",
    "full_rmat_max": "rmat-max-segment-cb0-n1",
    "full_rmat_sum_atomic": "rmat-sum-atomic-cb0-n1",
    "full_reddit_mean_atomic": "reddit-mean-atomic-cb0-n1",
    "full_reddit_max": "reddit-max-segment-cb21179-n1",
    "full_gat_rmat": "rmat-gat-segment-cb0-n1-gat",
}


def summary(path, row=2):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[row]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name", "")[:80]}
    for k, (m, scale) in KEYS.items():
        if d.get(m, "") == "":
            continue
        v = float(d[m].replace(",", "")) * UNIT.get(u.get(m, ""), 1)
        if k == "time_ms":
            v *= 1e3
        elif scale != 1:
            v *= scale
        out[k] = round(v, 4)
    return out


if __name__ == "__main__":
    tag = sys.argv[1]
    res = {"_note": "headline ncu counters of one launch of each workload's dominant kernel (--set full, "
                    f"--clock-control none), from profiles/{tag}_full_*.raw.csv"}
    for cap, key in WORKLOADS.items():
        p = os.path.join("profiles", f"{tag}_{cap}.raw.csv")
        if os.path.exists(p):
            res[key] = summary(p)
            res[key]["source"] = p
            n_rows = len(list(csv.reader(open(p))))
            for extra in range(3, n_rows):  # captures of several kernels (GAT: forward, backward)
                res[f"{key}#{extra - 2}"] = dict(summary(p, extra), source=p)
    json.dump(res, open("profiles/ncu_summary.json", "w"), indent=1)
    print(json.dumps(res, indent=1))
