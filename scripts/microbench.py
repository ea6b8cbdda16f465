#!/usr/bin/env python
"""Device time and bandwidth of the per-row building blocks of the path that bench.py does not time on
their own (SURVEY 8(a) rows a1 plan, a2 degree, a3 GCN normalisation, a9 collate, a10 halo build /
pack), on the configs' shapes.  CUDA events around each call (median of R calls after warm-up),
algorithmic bytes = what the step must read + write once.  Synchronous calls (plan build, gcn_norm,
halo build) include their host read-back.  One JSON object per line; --out writes a list."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1903_02428_b200 as pg  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=10, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def row(name, ms, nbytes, **kw):
    gbs = nbytes / (ms * 1e-3) / 1e9
    r = {"op": name, "ms": ms, "alg_bytes": int(nbytes), "GB/s": gbs, "frac_of_hbm_peak": gbs / peak()}
    r.update(kw)
    print(json.dumps(r), flush=True)
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    res = []
    # ---- Reddit-shaped graph (config 4) ----
    ei, x = synth.reddit_like_torch(dev, ld=608)
    N, E = x.shape[0], ei.shape[1]
    res.append(row("degree (a2), Reddit", timed(lambda: pg.pyg_degree(ei[1], N)), E * 8 + N * 4, E=E, N=N))
    res.append(row("plan build (a1), Reddit, unblocked", timed(lambda: pg.pyg_plan_build(ei[1], ei[0], N, N), 3, 1),
                   E * 16 + E * 4 * 3 + (N + 1) * 8, E=E, N=N,
                   note="reads the edge list, writes col + perm + pos_row + rowptr; radix sort passes extra"))
    res.append(row("gcn_norm (a3), Reddit", timed(lambda: pg.pyg_gcn_norm(ei, N), 3, 1),
                   E * 16 + (E + N) * (16 + 4) + N * 8, E=E, N=N,
                   note="self-loops appended, D^-1/2 (A+I) D^-1/2 weights; synchronous (reads E' back)"))
    del ei, x
    torch.cuda.empty_cache()
    # ---- R-MAT (config 5): halo of a 1/8 slice (a10) ----
    ei = synth.rmat_torch(dev)
    N, E = synth.RMAT["N"], ei.shape[1]
    plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
    per = (N + 7) // 8
    sl = plan.slice(0, per)
    res.append(row("halo build (a10), R-MAT rank 0 of 8", timed(lambda: pg.pyg_halo_build(sl, N, 0, per, per), 3, 1),
                   (E // 8) * 8 + N * 16, E=E, N=N, note="mark + scan + remap over the slice; synchronous"))
    _, hids = pg.pyg_halo_build(sl, N, 0, per, per)
    xr = torch.rand((N, 128), device=dev)
    res.append(row("halo pack / gather_rows (a10), R-MAT rank 0 of 8", timed(lambda: pg.pyg_gather_rows(xr, hids)),
                   hids.numel() * (128 * 4 * 2 + 8), rows=int(hids.numel())))
    del ei, plan, sl, xr
    torch.cuda.empty_cache()
    # ---- point-cloud collate (a9) ----
    nn, eptr, local, _ = synth.clouds_like()
    args = (torch.from_numpy(nn).to(dev), torch.from_numpy(eptr).to(dev), torch.from_numpy(local).to(dev))
    Et, Nt = local.shape[1], int(nn.sum())
    res.append(row("collate (a9), 64 point clouds", timed(lambda: pg.pyg_collate(*args, N_total=Nt), 20, 3),
                   2 * (2 * Et * 8) + Nt * 8 + (nn.size + 1) * 16, E=Et, N=Nt))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
