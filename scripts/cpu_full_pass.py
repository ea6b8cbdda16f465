"""One FULL pass of the CPU oracle (single-threaded C, fp64 accumulation) over a whole large workload,
timed on the host it runs on (SURVEY 8(d) "the final report uses full passes"; the bench's
cpu_baseline times a fixed row sample to stay within minutes and reports this record beside it).

    python scripts/cpu_full_pass.py [reddit-mean] [rmat-sum] ...   -> profiles/cpu_full_pass.json

The workload is bench.py's (same generators, seeds and shapes), built on the CPU.
"""
from __future__ import annotations

import datetime
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(keys):
    import bench
    import oracle

    oracle.build()
    out_path = os.path.join(ROOT, "profiles", "cpu_full_pass.json")
    try:
        rec = json.load(open(out_path))
    except Exception:
        rec = {}
    for key in keys:
        cfg, red = key.split("-")
        t0 = time.perf_counter()
        # drawn on the GPU when there is one (the identical graph bench times), then copied to the host
        w = bench.make_workload(cfg, torch.device("cuda" if torch.cuda.is_available() else "cpu"), 0)
        ei = w["ei"].cpu().numpy()
        x = np.ascontiguousarray(w["x"].cpu().numpy())
        gen = time.perf_counter() - t0
        E, F, N = w["E"], w["F"], w["N"]
        t0 = time.perf_counter()
        oracle.propagate(x, ei, reduce=red)
        dt = time.perf_counter() - t0
        rec[key] = {"value": E * F / dt, "unit": "edges*F/s", "seconds": dt, "N": N, "E": E, "F": F,
                    "cores": 1, "kind": "oracle", "what": f"oracle.propagate {red} over the whole graph, one pass",
                    "host": bench.host_info(), "gen_s": gen,
                    "when": datetime.datetime.now(datetime.timezone.utc).isoformat(timespec="seconds")}
        print(key, json.dumps(rec[key]), flush=True)
        json.dump(rec, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["reddit-mean"])
