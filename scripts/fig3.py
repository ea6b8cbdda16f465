#!/usr/bin/env python
"""NEXT-4: the paper's Fig. 3 study on B200 (Appendix A): forward and backward runtime of
1,000 runs of gather/scatter aggregation (GS) versus sparse-matrix multiplication (SpMM) on
Erdos-Renyi graphs with 10,000 nodes and average degree 2..128, for coalesced (target-sorted) and
non-coalesced (shuffled) edge order.

  GS atomic   pyg_propagate / pyg_propagate_backward without a plan (the paper's scheme: gather +
              red.global scatter; no preprocessing, order-agnostic)
  GS segment  the same calls with CSR plans (built once, outside the timing, as P:276 advises)
  SpMM        torch.sparse CSR x dense (cuSPARSE) -- the paper's comparator, a library call.  Its
              forward needs CSR (coalesced) input: for the non-coalesced layout the COO -> CSR
              conversion is part of every call; its backward multiplies by the transpose, whose CSR
              is rebuilt every call ("coalescing is performed in any case").

Sum aggregation, F = 16 by default (the paper does not state F; reading Q20).  Times are CUDA-event
measurements of 1,000 back-to-back runs, reported in ms for the 1,000 runs like Fig. 3.
Writes one JSON object per (degree, layout) to stdout and, with --out, a JSON list.
"""
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


def timed(fn, runs):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(runs):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)  # ms for `runs` runs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=10000)
    ap.add_argument("--degrees", default="2,4,8,16,32,64,128")
    ap.add_argument("--features", type=int, default=16)
    ap.add_argument("--runs", type=int, default=1000)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    N, F = a.nodes, a.features
    res = []
    for d in [int(v) for v in a.degrees.split(",")]:
        ei_np = synth.erdos_renyi(N, d, seed=d)
        x = torch.from_numpy(synth.features(N, F, 100 + d)).to(dev)
        g = torch.from_numpy(synth.features(N, F, 200 + d, signed=True)).to(dev)
        order = np.lexsort((ei_np[0], ei_np[1]))
        for layout, ei_l in (("coalesced", ei_np[:, order]), ("non-coalesced", ei_np)):
            ei = torch.from_numpy(np.ascontiguousarray(ei_l)).to(dev)
            E = ei.shape[1]
            plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
            planT = pg.pyg_plan_build(ei[0], ei[1], N, N)
            out = torch.empty((N, F), device=dev)
            gx = torch.empty((N, F), device=dev)
            ws = torch.empty(max(1, pg.pyg_workspace_size(None, N, F, "sum", E=ei.shape[1])), dtype=torch.uint8, device=dev)
            wsp = torch.empty(max(1, pg.pyg_workspace_size(plan, N, F, "sum")), dtype=torch.uint8, device=dev)
            row = {"degree": d, "layout": layout, "N": N, "E": E, "F": F, "runs": a.runs}
            row["gs_atomic_fwd_ms"] = timed(lambda: pg.pyg_propagate(x, ei, reduce="sum", out=out, workspace=ws),
                                            a.runs)
            row["gs_atomic_bwd_ms"] = timed(lambda: pg.pyg_propagate_backward(None, ei, g, n_src=N, F=F,
                                                                              grad_x_src=gx), a.runs)
            row["gs_segment_fwd_ms"] = timed(lambda: pg.pyg_propagate(x, None, reduce="sum", plan=plan, out=out, E=E,
                                                                      workspace=wsp), a.runs)
            row["gs_segment_bwd_ms"] = timed(lambda: pg.pyg_propagate_backward(None, ei, g, n_src=N, F=F, plan_T=planT,
                                                                               grad_x_src=gx), a.runs)
            vals = torch.ones(E, device=dev)
            if layout == "coalesced":
                A = torch.sparse_coo_tensor(ei[[1, 0]], vals, (N, N)).coalesce().to_sparse_csr()
                row["spmm_fwd_ms"] = timed(lambda: torch.sparse.mm(A, x), a.runs)
            else:
                row["spmm_fwd_ms"] = timed(
                    lambda: torch.sparse.mm(torch.sparse_coo_tensor(ei[[1, 0]], vals, (N, N)).coalesce().to_sparse_csr(),
                                            x), a.runs)
            # backward of out = A x w.r.t. x: A^T g; the transpose is re-coalesced every call
            row["spmm_bwd_ms"] = timed(
                lambda: torch.sparse.mm(torch.sparse_coo_tensor(ei, vals, (N, N)).coalesce().to_sparse_csr(), g),
                a.runs)
            # correctness of the comparison: both compute A x
            ref = torch.sparse.mm(torch.sparse_coo_tensor(ei[[1, 0]], vals, (N, N)).coalesce().to_sparse_csr(), x)
            got = pg.pyg_propagate(x, None, reduce="sum", plan=plan, E=E)
            row["max_abs_diff_vs_spmm"] = float((got - ref).abs().max())
            print(json.dumps(row), flush=True)
            res.append(row)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
