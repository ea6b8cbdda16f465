"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) for the LAST propagate
call: the launches of our kernels after the last warm-up.  Usage: launch_summary.py file.csv [n_last]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if r and r[0] == "ID"][0]
K, M, V, U = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
launch = {}
order = []
for r in rows:
    if not r or not r[0].isdigit():
        continue
    i = int(r[0])
    if i not in launch:
        launch[i] = {"name": r[K]}
        order.append(i)
    v = float(r[V].replace(",", ""))
    unit = r[U]
    if unit in ("Mbyte", "MB"):
        v *= 1e6
    elif unit in ("Gbyte", "GB"):
        v *= 1e9
    elif unit in ("Kbyte", "KB"):
        v *= 1e3
    elif unit == "usecond":
        v *= 1e3
    elif unit == "msecond":
        v *= 1e6
    launch[i][r[M]] = v
n_last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
OURS = ("pyg", "seg::", "seg_kernel", "seg_tma", "coo_kernel", "combine", "degree_kernel", "hub_", "zero_slots",
        "mean_div", "max_decode", "softmax", "gat_", "tf32_gemm", "pool_kernel", "gather_rows", "halo_", "empty_rows",
        "dist_", "xi_kernel", "edge_", "fill_")
ours = [i for i in order if any(k in launch[i]["name"] for k in OURS)]
sel = ours[-n_last:] if n_last else ours
tot_t = sum(launch[i].get("gpu__time_duration.sum", 0) for i in sel)
tot_b = sum(launch[i].get("dram__bytes_read.sum", 0) + launch[i].get("dram__bytes_write.sum", 0) for i in sel)
for i in sel:
    L = launch[i]
    print(f"{i:5d} {L['name'][:70]:70s} {L.get('gpu__time_duration.sum', 0) / 1e6:9.3f} ms "
          f"{(L.get('dram__bytes_read.sum', 0) + L.get('dram__bytes_write.sum', 0)) / 1e9:8.2f} GB")
print(f"TOTAL {len(sel)} launches {tot_t / 1e6:.3f} ms, DRAM {tot_b / 1e9:.2f} GB ({tot_b:.0f} bytes)")
