"""Debug check: the GAT forward on the Reddit-shaped graph (H = 8, C = 75, the bench's --op gat
setup) against the oracle on the in-edges of the first R target rows, for the plain and the factored
form, printing the worst element against the tolerance |got - ref| <= 1e-5 * S + 1e-6.
Usage (GPU): python scripts/gat_reddit_check.py [R] [C]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1903_02428_b200 as pg  # noqa: E402
import synth  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
C = int(sys.argv[2]) if len(sys.argv) > 2 else 75
dev = torch.device("cuda:0")
ei, x = synth.reddit_like_torch(dev)
N, E = x.shape[0], ei.shape[1]
H = 8
F = H * C
plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
gg = torch.Generator(device=dev)
gg.manual_seed(107)
s_src = torch.randn((N, H), generator=gg, device=dev) * 2
s_dst = torch.randn((N, H), generator=gg, device=dev) * 2
z = torch.randn((N, F), generator=gg, device=dev)
ei_c = ei.cpu().numpy()
m = ei_c[1] < R
sub = ei_c[:, m]
ref_out, ref_alpha, ref_abs = oracle.gat(z.cpu().numpy(), s_src.cpu().numpy(), s_dst[:R].cpu().numpy(), sub, H,
                                         n_dst=R, with_abs=True)[:3]
for factored in (False, True):
    rs = torch.empty((N, H), device=dev) if factored else None
    out, alpha = pg.pyg_gat_propagate(z, s_src, s_dst, H, plan, row_sums=rs)
    got = out[:R].cpu().numpy()
    err = np.abs(got - ref_out)
    tol = 1e-5 * ref_abs + 1e-6
    bad = err > tol
    i = np.unravel_index(np.argmax(err - tol), err.shape)
    print(f"factored={factored} C={C} R={R} E_sub={sub.shape[1]}: bad={int(bad.sum())} of {bad.size}; worst row {i[0]} "
          f"col {i[1]}: got {got[i]:.8g} ref {ref_out[i]:.8g} err {err[i]:.3g} tol {tol[i]:.3g}; "
          f"bad rows {np.unique(np.nonzero(bad)[0])[:10].tolist()}; bad cols of row 0 {np.nonzero(bad[0])[0].tolist()}")
