"""Write profiles/traffic.json from ncu launch lists: DRAM bytes (read + write) summed over the
launches of ONE propagate call (the last call in the list), keyed like bench.py's roofline key."""
import csv
import gzip
import io
import json
import os
import sys


SEG = ("seg_kernel", "seg_tma", "combine_kernel", "empty_rows")
COO = ("coo_", "pack_cols", "unpack_cols", "degree_kernel", "hub_assign", "zero_slots", "hub_combine", "mean_div")


def call_traffic(path, n_last, names=SEG):
    f = io.TextIOWrapper(gzip.open(path)) if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    hdr = [r for r in rows if r and r[0] == "ID"][0]
    K, M, V, U = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    d = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
    for r in rows:
        if r and r[0].isdigit():
            d.setdefault(int(r[0]), {"name": r[K]})[r[M]] = float(r[V].replace(",", "")) * scale.get(r[U], 1)
    ours = [i for i in sorted(d) if any(k in d[i]["name"] for k in names)]
    sel = ours[-n_last:]
    b = sum(d[i].get("dram__bytes_read.sum", 0) + d[i].get("dram__bytes_write.sum", 0) for i in sel)
    t = sum(d[i].get("gpu__time_duration.sum", 0) for i in sel)
    return int(b), t / 1e6, [d[i]["name"][:60] for i in sel]


if __name__ == "__main__":
    tag = sys.argv[1]
    out = {"_note": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) summed over the launches of one "
                    "propagate call, from the ncu launch lists in profiles/; bench.py divides by launches_per_call."}
    specs = [("reddit-mean-segment-cb21179-n1", f"launches_reddit_mean.csv", 11),
             ("rmat-sum-segment-cb0-n1", "launches_rmat_sum.csv", 3),
             ("rmat-max-segment-cb0-n1", "launches_rmat_max.csv", 3),
             ("reddit-max-segment-cb21179-n1", "launches_reddit_max.csv", 11),
             # atomic: degree + hub setup (2) + 19 L2 column tiles x (pack, tile kernel, unpack) + hub combine
             ("reddit-mean-atomic-cb0-n1", "launches_reddit_mean_atomic.csv", 61, COO)]
    for spec in specs:
        key, f, n = spec[:3]
        names = spec[3] if len(spec) > 3 else SEG
        p = os.path.join("profiles", f"{tag}_{f}")
        if not os.path.exists(p) and os.path.exists(p + ".gz"):
            p += ".gz"
        if os.path.exists(p):
            b, ms, names = call_traffic(p, n, names)
            out[key] = b
            out[key + "_source"] = f"profiles/{tag}_{f} (last {n} launches: {sorted(set(names))}; {ms:.3f} ms serialized)"
    json.dump(out, open("profiles/traffic.json", "w"), indent=1)
    print(json.dumps(out, indent=1))
